"""Time the per-GPU shard of BASELINE cfg4 (8 humans x 1,048,576 particles x 500 steps,
400x400 shared grid): K2/K3 events of eager cycles + graph-replayed full cycles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2603_01122_b200.engine import CycleEngine, EngineConfig  # noqa: E402
from paper_2603_01122_b200.scenario import make_scene  # noqa: E402


def main(budget_kb=0.0, steps=None):
    sc = make_scene("cfg4_rank", cycles=4, humans=8)
    if steps:
        sc.steps = steps
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec,
                      EngineConfig(n=sc.n, steps=sc.steps, dt=sc.dt, smoothing_sigma=0.1, mode="production",
                                   window_budget_kb=budget_kb))
    eng.prime(sc.warmup_track[0])
    for k in range(1, 11):
        eng.stage(sc.warmup_track[k], buf=0)
        eng.run_cycle(buf=0)
    s = torch.cuda.Stream()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(3)]
    for e in ev:
        eng.run_cycle(buf=0, with_h2d=False, stream=s, events=e)
    s.synchronize()
    g = eng.capture(buf=0, with_h2d=False)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g.replay()
        a.record(s)
        for _ in range(5):
            g.replay()
        b.record(s)
    s.synchronize()
    eng.check_errors()
    cyc = a.elapsed_time(b) / 5
    ps = 8 * sc.n * sc.steps
    print(f"cfg4_rank T={sc.steps} (window budget {budget_kb} KB, launches {eng.window_bounds()}, "
          f"GC_PREDICT_GLOBAL_HIST={os.environ.get('GC_PREDICT_GLOBAL_HIST', '0')}): K2 {sum(e[0].elapsed_time(e[1]) for e in ev) / 3:.2f} ms, "
          f"K3 {sum(e[1].elapsed_time(e[2]) for e in ev) / 3:.3f} ms, cycle {cyc:.2f} ms "
          f"({1000 / cyc:.1f} Hz, {ps / cyc / 1e6:.1f} G particle-steps/s)")


if __name__ == "__main__":
    main(float(sys.argv[1]) if len(sys.argv) > 1 else 0.0, int(sys.argv[2]) if len(sys.argv) > 2 else None)
