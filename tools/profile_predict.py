"""Run one k_predict launch of a cfg3-shaped workload (for ncu captures).

    python tools/profile_predict.py [--mode production|reference] [--steps T] [--humans H] [--n N]
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
    ap.add_argument("--mode", default="production")
    ap.add_argument("--steps", type=int, default=250)
    ap.add_argument("--humans", type=int, default=8)
    ap.add_argument("--n", type=int, default=262144)
    ap.add_argument("--cycles", type=int, default=2)
    ap.add_argument("--summary", action="store_true", help="one line: mean K2 ms over cycles 1..")
    ap.add_argument("--uniform", action="store_true", help="keep the uniform prior (no belief updates)")
    ap.add_argument("--betas", default=None, help="comma-separated rationality set (default log_spaced(5))")
    ap.add_argument("--goal-radius", type=float, default=None)
    ap.add_argument("--ref-exact", action="store_true", help="reference mode: numpy exp everywhere (no filter)")
    a = ap.parse_args()
    sc = make_scene("cfg3", cycles=4, humans=a.humans, goal_radius=a.goal_radius)
    if a.betas:
        from paper_2603_01122_b200.agents import RationalitySet
        from paper_2603_01122_b200.belief import HypothesisSpace
        rs = RationalitySet(tuple(float(b) for b in a.betas.split(",")))
        sc.spaces = [HypothesisSpace(rs, sp.goals) for sp in sc.spaces]
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec,
                      EngineConfig(n=a.n, steps=a.steps, dt=sc.dt, mode=a.mode, ref_filter=not a.ref_exact))
    eng.prime(sc.warmup_track[0])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    k2 = []
    for k in range(a.cycles):
        eng.stage(sc.warmup_track[1 + k], buf=0)
        eng.run_cycle(buf=0, events=ev, with_update=not a.uniform)
        torch.cuda.synchronize()
        k2.append(ev[0].elapsed_time(ev[1]))
        if not a.summary:
            print(f"cycle {k}: k_predict {k2[-1]:.3f} ms, epilogue {ev[1].elapsed_time(ev[2]):.3f} ms")
    if a.summary:
        print(f"k_predict mean {sum(k2[1:]) / max(1, len(k2) - 1):.4f} ms  " + " ".join(f"{v:.3f}" for v in k2[1:]))
    eng.check_errors()


if __name__ == "__main__":
    main()
