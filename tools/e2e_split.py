"""Where the e2e cycle's time above the device-resident cycle goes (cfg3, one GPU).

Replays CUDA graphs of one cycle back to back and times each on the stream:
  chunks=1, no D2H     (the device-resident cycle bench.py reports as ms_per_step)
  chunks=C, no D2H     (cost of splitting the horizon into C launches)
  chunks=C, D2H tiles  (the e2e graph: + tile-sparse publication on a copy stream)
    python tools/e2e_split.py [--chunks 4] [--dtype float64]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_01122_b200.engine import CycleEngine, EngineConfig  # noqa: E402
from paper_2603_01122_b200.scenario import make_scene  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", type=int, default=4)
    ap.add_argument("--taper", type=float, default=0.5)
    ap.add_argument("--dtype", default="float64")
    ap.add_argument("--cycles", type=int, default=30)
    a = ap.parse_args()
    sc = make_scene("cfg3", cycles=64)
    cfg = EngineConfig(n=sc.n, steps=sc.steps, dt=sc.dt, mode="production", union_dtype=a.dtype,
                       chunk_taper=a.taper)
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, cfg)
    eng.prime(sc.warmup_track[0])
    for k in range(1, 11):
        eng.stage(sc.warmup_track[k], buf=0)
        eng.run_cycle(buf=0)
    torch.cuda.synchronize()
    dt = torch.float64 if a.dtype == "float64" else torch.float32
    ushape = (sc.steps, sc.spec.height, sc.spec.width)
    h_out = torch.empty(ushape, dtype=dt).pin_memory()
    s = torch.cuda.Stream()
    variants = [("chunks=1 no-d2h", dict(chunks=1, d2h=None)),
                (f"chunks={a.chunks} no-d2h", dict(chunks=a.chunks, d2h=None)),
                (f"chunks={a.chunks} d2h-tiles", dict(chunks=a.chunks, d2h=h_out))]
    with torch.cuda.stream(s):
        graphs = [(name, eng.capture(buf=0, with_h2d=True, **kw)) for name, kw in variants]
    for rep in range(2):
        for name, g in graphs:
            times = []
            with torch.cuda.stream(s):
                for i in range(a.cycles):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(s)
                    g.replay()
                    e1.record(s)
                    times.append((e0, e1))
            s.synchronize()
            ms = np.array([x.elapsed_time(y) for x, y in times[3:]])
            print(f"{name:24s} mean {ms.mean():.3f} ms  p50 {np.median(ms):.3f}  max {ms.max():.3f}")
    # the same cycle eagerly (no graph): chunked with the publication on a copy stream
    cp = torch.cuda.Stream(priority=0)
    s = torch.cuda.Stream(priority=-1)
    for d2 in (None, h_out):
        times = []
        with torch.cuda.stream(s):
            for i in range(a.cycles):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                eng.run_cycle(buf=0, chunks=a.chunks, d2h=d2, copy_stream=cp if d2 is not None else None, stream=s)
                e1.record(s)
                times.append((e0, e1))
        s.synchronize()
        ms = np.array([x.elapsed_time(y) for x, y in times[3:]])
        print(f"eager chunks={a.chunks} {'d2h' if d2 is not None else 'no-d2h':8s} mean {ms.mean():.3f} ms")
    # each chunk's publication alone (the union of the last cycle; host stack already equal,
    # so this is the steady-state work: changed tiles only)
    import ctypes
    from paper_2603_01122_b200 import _lib
    for (t0, t1) in eng.chunk_bounds(a.chunks):
        pa = eng._publish_args(0, eng.unions[0], h_out)
        pa.t_begin, pa.t_end = t0 - 1, t1 - 1
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            _lib.check(_lib.lib().gc_publish_tiles(ctypes.byref(pa), ctypes.c_void_p(s.cuda_stream)), "publish")
            e1.record(s)
        s.synchronize()
        fl = eng.utile[0][t0 - 1:t1 - 1]
        print(f"publish layers [{t0 - 1},{t1 - 1}): {e0.elapsed_time(e1):.3f} ms, {int(fl.sum())} live tiles "
              f"({int(fl.sum()) * 32 * 32 * h_out.element_size() / 1e6:.1f} MB)")
    print("chunk sizes", [b - a_ for a_, b in eng.chunk_bounds(a.chunks)])


if __name__ == "__main__":
    main()
