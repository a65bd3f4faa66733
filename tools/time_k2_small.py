"""K2 / K3 event times of the single-human configurations (cfg1, cfg2) over eager cycles."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2603_01122_b200.engine import CycleEngine, EngineConfig  # noqa: E402
from paper_2603_01122_b200.scenario import make_scene  # noqa: E402

for name in ("cfg1", "cfg2"):
    sc = make_scene(name, cycles=4)
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec,
                      EngineConfig(n=sc.n, steps=sc.steps, dt=sc.dt, mode="production"))
    eng.prime(sc.warmup_track[0])
    eng.stage(sc.warmup_track[1], buf=0)
    s = torch.cuda.Stream()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(20)]
    for e in ev:
        eng.run_cycle(buf=0, with_h2d=False, stream=s, events=e)
    s.synchronize()
    k2 = sorted(e[0].elapsed_time(e[1]) for e in ev[5:])
    k3 = sorted(e[1].elapsed_time(e[2]) for e in ev[5:])
    print(f"{name}: K2 {k2[len(k2) // 2] * 1e3:.1f} us, K3 {k3[len(k3) // 2] * 1e3:.1f} us (medians)")
