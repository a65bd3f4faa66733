"""How sparse is the fused union the e2e cycle ships to the host?  (GPU)

Runs the bench scene's cycle (production mode, float64 union) and reports, per step and in
total, the nonzero cells and the nonzero 32 x 32 tiles of the (T, H, W) union -- the bytes
a tile-sparse D2H would move instead of the dense 8 T H W.

    python tools/union_sparsity.py [--config cfg3] [--goal-radius R]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2603_01122_b200.engine import CycleEngine, EngineConfig  # noqa: E402
from paper_2603_01122_b200.scenario import make_scene  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--goal-radius", type=float, default=None)
    ap.add_argument("--mode", default="production")
    a = ap.parse_args()
    sc = make_scene(a.config, cycles=4, goal_radius=a.goal_radius)
    cfg = EngineConfig(n=sc.n, steps=sc.steps, dt=sc.dt, mode=a.mode, union_dtype="float64")
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, cfg)
    eng.prime(sc.warmup_track[0])
    for k in range(1, 11):
        eng.stage(sc.warmup_track[k], buf=k % 2)
        u = eng.run_cycle(buf=k % 2)
    torch.cuda.synchronize()
    T, H, W = u.shape
    E = 32
    Hp, Wp = -(-H // E) * E, -(-W // E) * E
    pad = torch.zeros((T, Hp, Wp), dtype=u.dtype, device=u.device)
    pad[:, :H, :W] = u
    nzc = (u > 0).sum(dim=(1, 2))
    tiles = (pad.view(T, Hp // E, E, Wp // E, E) > 0).any(dim=4).any(dim=2).sum(dim=(1, 2))
    tot_tiles = (Hp // E) * (Wp // E)
    print(f"{a.config} goal radius {sc.goal_radius:g} m: union {T}x{H}x{W} f64 = {u.numel() * 8 / 1e6:.0f} MB dense")
    for t in (0, T // 10, T // 4, T // 2, 3 * T // 4, T - 1):
        print(f"  step {t + 1:4d}: nonzero cells {int(nzc[t]):7d} ({float(nzc[t]) / (H * W):.3f}), "
              f"nonzero 32x32 tiles {int(tiles[t]):4d} of {tot_tiles}")
    nt = int(tiles.sum())
    print(f"total: nonzero cells {int(nzc.sum())} ({float(nzc.sum()) / u.numel():.4f} of the stack), nonzero tiles "
          f"{nt} of {T * tot_tiles} ({nt / (T * tot_tiles):.3f}) -> {nt * E * E * 8 / 1e6:.1f} MB as f64 tiles")


if __name__ == "__main__":
    main()
