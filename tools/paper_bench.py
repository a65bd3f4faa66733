"""The paper's / reference's own prediction benchmark through the drop-in API.

    python tools/paper_bench.py

`gridcast bench` (cli.py:100-115, :172-230): one human in a 10 m room, 50 x 50 grid,
|B| = 5 rationality values x |G| = 10 goals on a 3.5 m circle, the 4 x 24 control grid,
n = 8192 particles, dt 0.5, sigma 0, T in {2, 4, 6, 8, 10}; 1 warm-up + 5 timed runs per
T.  Each run is one call of the drop-in `predict()` (the call a reference user makes) with
the layers read back as a host float64 (T, H, W) array -- wall clock around the whole
call, so Python, launch and copy overheads are included -- in the deterministic reference
mode (bit-exact counts) and in production mode.  The paper's JAX implementation reports
7 / 7 / 7 / 7 / 8 ms for this configuration on an RTX 2080 Ti (PAPER.md:304-335,
BASELINE.md section 1); the reference CPU path 21-81 ms on 8 threads.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_01122_b200 as G  # noqa: E402

PAPER_MS = {2: 7.0, 4: 7.0, 6: 7.0, 8: 7.0, 10: 8.0}


def problem():
    room, grid = 10.0, 50
    spec = G.GridSpec(grid, grid, room / grid)
    ang = 2.0 * np.pi * np.arange(10) / 10
    goals = np.stack([room / 2 + 3.5 * np.cos(ang), room / 2 + 3.5 * np.sin(ang)], axis=1)
    space = G.HypothesisSpace(G.RationalitySet.log_spaced(5), G.GoalSet(goals))
    return (G.HumanState(room / 2, room / 2), G.init_belief(space), G.ControlSet.grid(4, 24, 1.4),
            G.q_goal_progress(0.5), space, spec)


def main():
    z0, belief, cs, q, space, spec = problem()
    print(f"{'T':>3} {'mode':>10} {'mean ms':>9} {'min ms':>8}   paper JAX 2080 Ti")
    for mode in ("reference", "production"):
        for T in (2, 4, 6, 8, 10):
            cfg = G.PredictionConfig(n=8192, steps=T, dt=0.5, smoothing_sigma=0.0, seed=0, mode=mode)
            ts = []
            for it in range(6):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                st = G.predict(z0, belief, cfg, cs, q, space, spec)
                layers = st.layers  # host float64 (T, H, W), the reference's layout
                assert layers.shape == (T, spec.height, spec.width)
                ts.append((time.perf_counter() - t0) * 1e3)
            run = ts[1:]
            print(f"{T:>3} {mode:>10} {np.mean(run):9.3f} {np.min(run):8.3f}   {PAPER_MS[T]:.0f} ms")


if __name__ == "__main__":
    main()
