"""Roofline sweep of the update+predict cycle (BASELINE.json config 5, one GPU).

    python tools/sweep.py [--humans 1] [--out gpurun_out/sweep.json]

Grid of particles n = 2^10 .. 2^24 (every 2 powers) x horizon T in {20, 100, 250, 1000}
(dt 0.02) x grid {100^2, 400^2, 1000^2} @ 0.1 m, one human with |H| = 20 (4 goals x 5
betas) after 10 observations, production mode.  Per point: K2 time (event-record nodes
inside the replayed cycle graph: the last of 5 back-to-back replays, mean of 3 such runs), full
cycle time (the same back-to-back CUDA graph replays, mean of the last 5),
particle-steps/s, and the issue-rate roofline fraction of the whole cycle (K1+K2+K3 time)
using the lane-instructions per particle-step of the cfg3 ncu capture
(profiles/ncu_summary.json; an approximation away from cfg3, where the histogram share
differs, and a lower bound since the cycle time includes K1/K3).  Horizons whose
reachable window exceeds 64 KB of shared memory (T=1000) take K2's global-atomics path.
--table re-renders a saved sweep with the current ncu summary.  Multi-GPU points are the driver's
scaling run (bench.py --gpus N), not this tool: gpurun exposes one GPU.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2603_01122_b200 import scenario  # noqa: E402
from paper_2603_01122_b200.engine import CycleEngine, EngineConfig  # noqa: E402


def point(n, T, cells, humans):
    scenario.CONFIGS["sweep"] = dict(humans=humans, goals=4, n=n, steps=T, dt=0.02, cells=cells)
    sc = scenario.make_scene("sweep", cycles=4, humans=humans)
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec,
                      EngineConfig(n=n, steps=T, dt=sc.dt, smoothing_sigma=0.1, mode="production"))
    eng.prime(sc.warmup_track[0])
    for k in range(1, 11):
        eng.stage(sc.warmup_track[k], buf=0)
        eng.run_cycle(buf=0)
    s = torch.cuda.Stream()
    # K2 timed by event-record nodes inside the replayed cycle graph (the clock of the cycle
    # time itself, as bench.py does): eager events would include host launch gaps
    kev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(3)]
    g = eng.capture(buf=0, with_h2d=False, events=kev)
    reps = 5
    k2s = []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        g.replay()
        s.synchronize()
        for _ in range(3):  # K2 of the last of back-to-back replays (the cycle's own regime)
            a.record(s)
            for _ in range(reps):
                g.replay()
            b.record(s)
            s.synchronize()
            k2s.append(kev[0].elapsed_time(kev[1]))
    k2 = sum(k2s) / len(k2s)
    eng.check_errors()
    cyc = a.elapsed_time(b) / reps
    del eng, g
    torch.cuda.empty_cache()
    return k2, cyc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--humans", type=int, default=1)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--table", action="store_true", help="print the table of a saved sweep (--out)")
    a = ap.parse_args()
    summ = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary.json")))["production"]["k_predict"]
    ipp = summ["lane_instr_per_particle_step"]
    mhz = 1965.0
    issue_peak = 148 * 4 * 32 * mhz * 1e6
    ns = [1 << p for p in range(10, 25, 2)]
    Ts = [20, 100, 250, 1000]
    grids = [100, 400, 1000]
    if a.quick:
        ns, Ts, grids = [1 << 10, 1 << 18], [20, 250], [400]
    hdr = (f"{'n':>9} {'T':>5} {'grid':>5} {'K2 ms':>9} {'cycle ms':>9} {'Hz':>8} {'G psteps/s':>11} "
           f"{'issue frac':>10}")
    if a.table:
        rows = json.load(open(a.out))["rows"]
        print(f"# cycle roofline fraction at {ipp} lane-instr/particle-step (cfg3 ncu), {mhz:.0f} MHz")
        print(hdr)
        for r in rows:
            ps = r["humans"] * r["n"] * r["T"]
            frac = ps * ipp / (r["cycle_ms"] * 1e-3) / issue_peak
            print(f"{r['n']:>9} {r['T']:>5} {r['grid']:>5} {r['k2_ms']:9.3f} {r['cycle_ms']:9.3f} {r['hz']:8.1f} "
                  f"{r['psteps_per_s'] / 1e9:11.2f} {frac:10.2f}")
        return
    rows = []
    print(f"{'n':>9} {'T':>5} {'grid':>5} {'K2 ms':>9} {'cycle ms':>9} {'Hz':>8} {'G psteps/s':>11} {'issue frac':>10}")
    for cells in grids:
        for T in Ts:
            for n in ns:
                k2, cyc = point(n, T, cells, a.humans)
                ps = a.humans * n * T
                rate = ps / (cyc * 1e-3)
                frac = ps * ipp / (cyc * 1e-3) / issue_peak
                rows.append(dict(n=n, T=T, grid=cells, humans=a.humans, k2_ms=k2, cycle_ms=cyc, hz=1000 / cyc,
                                 psteps_per_s=rate))
                print(f"{n:>9} {T:>5} {cells:>5} {k2:9.3f} {cyc:9.3f} {1000 / cyc:8.1f} {rate / 1e9:11.2f} {frac:10.2f}",
                      flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump({"ipp_cfg3": ipp, "sm_mhz_assumed": mhz, "rows": rows}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
