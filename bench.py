#!/usr/bin/env python
"""Benchmark: the full predict+update cycle of BASELINE.json configs[2] (cfg3) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one prediction cycle: belief update of every human (K1) + prediction of
every human (K2: 262,144 particles x 250 steps, dt 0.02) + smoothing and max-union into
the shared 400x400 grid (K3).  N GPUs: weak scaling, 8 humans per rank; with N > 1 the
per-rank unions are merged into one fused grid by an NCCL max-reduce each cycle.

``value``  -- particle-steps/s of the whole job, inputs resident in HBM (CUDA graph
              replay, CUDA events, max over ranks);  ``hz`` = cycles/s, ``p99_ms``.
``e2e``    -- the same metric with the cycle's observations copied from pinned host
              memory and the fused float32 (T, H, W) union read back to pinned host
              memory every cycle (double-buffered on a copy stream).
``--impl reference`` times the reference CPU implementation (oracle/port.py, a
restatement pinned bit-exact to the reference) on the host cores on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")  # fair CPU timing

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "particle-steps/s"
# reference-algorithm work per particle-step: 9m+10 FP32 ops, m = 96
REF_OPS_PER_PSTEP = 9 * 96 + 10
LAT_CYCLES = 1000  # p50/p99 latencies are taken over at least this many cycles


def peaks():
    p = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback"}
    f = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(f):
        d = json.load(open(f))
        p.update({k: d[k] for k in ("hbm_gbs", "sm_max_mhz") if k in d})
        p["source"] = "measured"
    return p


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------------------
# CPU baseline: the reference CPU cycle (oracle/port.py) on a bounded sample of cfg3
# ---------------------------------------------------------------------------------------
def cpu_sample(scene, t_steps=10, reps=3, workers=None):
    """Time 1 human x n particles x t_steps (+ one belief update) with the reference CPU
    path; extrapolate linearly in T and in humans (predict is linear in both,
    cli.py:135-146) to one full cycle."""
    from oracle import model, port
    from oracle.predict import Grid, belief_update
    workers = workers or (os.cpu_count() or 1)
    t_steps = min(t_steps, scene.steps)
    cs = scene.control_set
    tb = model.make_tables(cs.v, cs.theta, scene.dt, model.QSpec("goal_progress", 0.5))
    sp = scene.spaces[0]
    beta_of, goal_of = sp.beta_of, sp.goal_xy_of
    lw = np.full(len(beta_of), -np.log(len(beta_of)))
    grid = Grid(scene.spec.width, scene.spec.height, scene.spec.resolution)
    prev, obs = scene.prev_xy[0], scene.track[0][0]
    t_upd, t_pred = [], []
    for r in range(reps + 1):
        t0 = time.perf_counter()
        post, _ = belief_update(lw, prev, obs, 0.1, cs.v, cs.theta, model.QSpec("goal_progress", 0.5),
                                beta_of, goal_of, 0.0, snap_tol=float("inf"))
        t1 = time.perf_counter()
        port.predict(obs, post, scene.n, t_steps, scene.dt, 0.1, 0, tb, beta_of, goal_of, grid,
                     prefix=(2, 0), workers=workers)
        t2 = time.perf_counter()
        if r > 0:
            t_upd.append(t1 - t0)
            t_pred.append(t2 - t1)
    H = len(scene.spaces)
    cycle_s = H * (float(np.median(t_upd)) + float(np.median(t_pred)) * scene.steps / t_steps)
    psteps = H * scene.n * scene.steps
    return {
        "value": psteps / cycle_s, "unit": UNIT, "cores": workers, "kind": "port",
        "hz": 1.0 / cycle_s, "cycle_s": cycle_s,
        "sample": (f"1 human x {scene.n} particles x {t_steps} steps + 1 belief update, median of {reps}; "
                   f"extrapolated x{H} humans x{scene.steps / t_steps:g} in T (reference CPU path restated "
                   f"in oracle/port.py, ThreadPool {workers} workers, OPENBLAS_NUM_THREADS=1)"),
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_2603_01122_b200.scenario import make_scene
    scene = make_scene(args.config, cycles=2)
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(scene, t_steps=args.ref_t, reps=1)
        if i >= args.warmup:
            vals.append(r)
    v = float(np.median([r["value"] for r in vals]))
    cycle_s = float(np.median([r["cycle_s"] for r in vals]))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cycle_s * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "hz": 1.0 / cycle_s,
        "config": {"workload": (f"{args.config}: {len(scene.spaces)} humans x {scene.n} particles x {scene.steps} "
                                f"steps dt {scene.dt}, {scene.spec.width}x{scene.spec.height} union"),
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": vals[0]["cores"], "kind": "port",
                         "sample": vals[0]["sample"]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    # --force-dist: run the multi-GPU code path (NCCL process group, fused reduce) even
    # at world size 1 -- a one-rank smoke test of the N > 1 branch on a single GPU
    distributed = world > 1 or args.force_dist
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2603_01122_b200 import _lib
    from paper_2603_01122_b200.engine import CycleEngine, EngineConfig, fused_reduce
    from paper_2603_01122_b200.scenario import make_scene

    K, W = args.steps, args.warmup
    from paper_2603_01122_b200.scenario import CONFIGS
    hpg = CONFIGS[args.config]["humans"]  # humans per GPU (weak scaling): cfg3 8, cfg1/cfg2 1
    scene = make_scene(args.config, cycles=W + K + 4, humans=hpg, human_offset=hpg * rank)
    cfg = EngineConfig(n=scene.n, steps=scene.steps, dt=scene.dt, smoothing_sigma=0.1, seed=0,
                       mode=args.mode, time_union=False, chunk_taper=args.chunk_taper)
    fused = distributed and not args.no_fused
    # fused grid: NCCL max-reduce of the per-rank unions (engine.fused_reduce), or every
    # rank's K3 writing rank 0's grid over NVLink peer memory (peer.PeerUnion)
    peer = None
    if fused and args.fused_path == "peer":
        from paper_2603_01122_b200.peer import PeerUnion
        peer = PeerUnion((scene.steps, scene.spec.height, scene.spec.width), torch.float32)
    eng = CycleEngine(scene.control_set, scene.q, scene.spaces, scene.spec, cfg,
                      human_ids=list(range(hpg * rank, hpg * rank + len(scene.spaces))), peer=peer)
    # posterior after 10 observations (also warms every kernel)
    eng.prime(scene.warmup_track[0])
    for k in range(1, 11):
        eng.stage(scene.warmup_track[k], buf=k % 2)
        eng.run_cycle(buf=k % 2)
    torch.cuda.synchronize()
    eng.check_errors()

    def device_cycle(g, b=0):
        """One graph-replayed cycle plus the fused-grid merge (on the current stream)."""
        if peer is not None:
            peer.zero(b)
            peer.barrier()
            g.replay()
            peer.barrier()
        else:
            g.replay()
            if fused:
                fused_reduce(eng.unions[b], dst=0)

    def barrier():
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if not distributed:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    stream = torch.cuda.Stream()
    # ---- kernel timing (eager cycles, events on the launching stream) ----
    n_k = max(3, min(K, 10))
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(n_k)]
    for i in range(n_k):
        eng.run_cycle(buf=0, with_h2d=False, stream=stream, events=ev[i])
    stream.synchronize()
    barrier()
    k2_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in ev]))
    k3_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in ev]))

    # ---- value: device-resident cycle (CUDA graph replay) ----
    g = eng.capture(buf=0, with_h2d=False)
    cyc_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with torch.cuda.stream(stream):
        for _ in range(W):
            device_cycle(g)
    launches0 = _lib.lib().gc_launch_count()
    barrier()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local).__enter__()
    if True:
        with torch.cuda.stream(stream):
            t_start.record(stream)
            for i in range(K):
                cyc_ev[i][0].record(stream)
                device_cycle(g)
                cyc_ev[i][1].record(stream)
            t_end.record(stream)
        barrier()
    ms = t_start.elapsed_time(t_end) / K
    ms = max_over_ranks(ms)
    per_cycle = [a.elapsed_time(b) for a, b in cyc_ev]
    # latency percentiles over >= LAT_CYCLES cycles: extra untimed-for-value replays
    n_lat = max(args.lat_cycles, K)
    extra = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_lat - K)]
    with torch.cuda.stream(stream):
        for a_, b_ in extra:
            a_.record(stream)
            device_cycle(g)
            b_.record(stream)
    barrier()
    per_cycle += [a.elapsed_time(b) for a, b in extra]
    p99 = max_over_ranks(float(np.percentile(per_cycle, 99)))
    p50 = max_over_ranks(float(np.percentile(per_cycle, 50)))
    # graph replays do not pass through the C ABI launch counter: 3 kernels per cycle
    # (K1 belief, K2 predict, K3 epilogue) are captured in the graph
    gpu_launches = 3 * K
    assert _lib.lib().gc_launch_count() == launches0  # nothing eager snuck in

    # ---- e2e: pinned H2D of observations + D2H of the fused union every cycle ----
    ushape = (scene.steps, scene.spec.height, scene.spec.width)  # float32 fused union
    h2d = eng._nb
    d2h = math.prod(ushape) * 4
    tr = scene.track
    h_out = [torch.empty(ushape, dtype=torch.float32).pin_memory() for _ in range(2)]
    if not fused:
        # one CUDA graph per cycle: H2D of the observations, update, predict in
        # args.chunks horizon chunks whose layers stream to pinned host memory on a
        # copy stream while the next chunk computes; cycles run strictly one after
        # another, so the per-cycle time is the host-in -> host-out latency
        ga = [eng.capture(buf=b, with_h2d=True, chunks=args.chunks, d2h=h_out[b]) for b in (0, 1)]
        done = [torch.cuda.Event() for _ in range(2)]

        def e2e_loop(n_cycles, base):
            evs = []
            for i in range(n_cycles):
                b = i % 2
                done[b].synchronize()           # pinned input/output b free again
                eng.stage(tr[(base + i) % len(tr)], buf=b)
                with torch.cuda.stream(stream):
                    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s_ev.record(stream)
                    ga[b].replay()
                    e_ev.record(stream)
                    done[b].record(stream)
                evs.append((s_ev, e_ev))
            return evs

        e2e_loop(W, 0)
        barrier()
        e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_start.record(stream)
        evs = e2e_loop(K, W)
        e_end.record(stream)
        barrier()
        evs += e2e_loop(n_lat - K, W + K)  # latency samples only
        barrier()
        e2e_note = (f"per cycle: pinned obs H2D + update + predict in {args.chunks} horizon chunks "
                    f"(sizes {[b - a for a, b in eng.chunk_bounds(args.chunks)]}), each "
                    f"chunk's f32 union layers D2H on a copy stream while the next computes; cycles strictly "
                    f"sequential (latency = cycle time), one CUDA graph")
    else:
        # N > 1: the fused grid is merged by the NCCL max-reduce (or written in place over
        # peer memory); rank 0 reads it back, D2H of cycle k overlapped with cycle k+1
        # (double-buffered unions; with peer memory rank 0 re-zeroes buffer b after its
        # D2H, and every rank's next write of b follows the barrier that waits for that)
        ga = [eng.capture(buf=b, with_h2d=True) for b in (0, 1)]
        copy = torch.cuda.Stream()
        done = [torch.cuda.Event() for _ in range(2)]
        copied = [torch.cuda.Event() for _ in range(2)]
        staged_ok = [torch.cuda.Event() for _ in range(2)]

        def e2e_loop(n_cycles, base):
            evs = []
            for i in range(n_cycles):
                b = i % 2
                staged_ok[b].synchronize()
                eng.stage(tr[(base + i) % len(tr)], buf=b)
                with torch.cuda.stream(stream):
                    stream.wait_event(copied[b])
                    s_ev = torch.cuda.Event(enable_timing=True)
                    s_ev.record(stream)
                    if peer is not None:
                        peer.barrier()      # rank 0's zero of b precedes every rank's writes
                    ga[b].replay()
                    staged_ok[b].record(stream)
                    if peer is not None:
                        peer.barrier()      # every rank's K3 writes precede rank 0's read
                    else:
                        fused_reduce(eng.unions[b], dst=0)
                    done[b].record(stream)
                with torch.cuda.stream(copy):
                    copy.wait_event(done[b])
                    if rank == 0:
                        src = peer.tensor(b) if peer is not None else eng.unions[b]
                        h_out[b].copy_(src, non_blocking=True)
                        if peer is not None:
                            src.zero_()
                    e_ev = torch.cuda.Event(enable_timing=True)
                    e_ev.record(copy)
                    copied[b].record(copy)
                evs.append((s_ev, e_ev))
            return evs

        e2e_loop(W, 0)
        barrier()
        copy.synchronize()
        e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_start.record(stream)
        evs = e2e_loop(K, W)
        stream.wait_stream(copy)
        e_end.record(stream)
        barrier()
        evs += e2e_loop(n_lat - K, W + K)  # latency samples only
        stream.wait_stream(copy)
        barrier()
        e2e_note = ("pinned obs H2D + " + ("peer-memory fused union (K3 atomicMax into rank 0's grid over "
                    "NVLink)" if peer is not None else "NCCL fused union") +
                    " + rank-0 f32 D2H each cycle, D2H overlapped with the next cycle")
    clocks.__exit__(None, None, None)
    e2e_ms = max_over_ranks(e_start.elapsed_time(e_end) / K)
    lat = [a_.elapsed_time(b_) for a_, b_ in evs]
    e2e_p99 = max_over_ranks(float(np.percentile(lat, 99)))
    e2e_p50 = max_over_ranks(float(np.percentile(lat, 50)))
    eng.check_errors()

    psteps_rank = len(scene.spaces) * scene.n * scene.steps
    psteps = psteps_rank * world
    value = psteps / (ms * 1e-3)
    pk = peaks()
    clk = clocks.summary()
    sm_mhz = pk["sm_max_mhz"]
    issue_peak = 148 * 4 * 32 * sm_mhz * 1e6 / 1e12  # T lane-instr/s: 4 schedulers x 1 warp-instr/clk
    fp32_peak = 148 * 128 * sm_mhz * 1e6 / 1e12      # T FP32 lane-ops/s
    xu_peak = 148 * 16 * sm_mhz * 1e6 / 1e12         # T MUFU lane-ops/s (16 per SM per clock)
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    ncu = None
    if os.path.exists(prof):
        try:
            ncu = json.load(open(prof)).get(args.mode, {}).get("k_predict")
        except (ValueError, AttributeError):
            ncu = None
    ipp = (ncu or {}).get("lane_instr_per_particle_step")
    mpp = (ncu or {}).get("mufu_per_particle_step")
    traffic = (ncu or {}).get("dram_bytes_per_launch")
    k2_s = k2_ms * 1e-3
    # K2 is bound by SM instruction issue (no dense contraction, ~1 GB/s of HBM): the
    # roofline is executed lane-instructions per particle-step (ncu, static for this code
    # and workload) x particle-steps of the launch / the live launch time
    roof = {"bound": "issue", "kernel": "k_predict", "achieved": None, "peak": issue_peak,
            "unit": "T lane-instr/s", "frac": None, "traffic": traffic, "work": None,
            "peak_source": f"148 SM x 4 schedulers x 32 lanes x {sm_mhz:.0f} MHz ({pk['source']} sm_max_mhz)"}
    if ipp:
        ach = psteps_rank * ipp / k2_s / 1e12
        roof.update(achieved=ach, frac=ach / issue_peak,
                    work=f"{ipp} lane-instructions per particle-step (ncu) x {psteps_rank} particle-steps per launch")
    if mpp:
        xa = psteps_rank * mpp / k2_s / 1e12
        roof["xu"] = {"achieved": xa, "peak": xu_peak, "unit": "T MUFU lane-ops/s", "frac": xa / xu_peak,
                      "mufu_per_particle_step": mpp,
                      "note": "second bound: 24 heading + 1 speed-weight (2^-kr) + 1 chosen-heading ex2 and 1 rsqrt per particle-step"}
    if traffic:
        ga = traffic / k2_s / 1e9
        roof["hbm"] = {"achieved": ga, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": ga / pk["hbm_gbs"],
                       "note": "particles live in registers; HBM sees only the count reductions"}
    ref_ach = psteps_rank * REF_OPS_PER_PSTEP / k2_s / 1e12
    roof["reference_equivalent"] = {
        "achieved": ref_ach, "peak": fp32_peak, "unit": "T FP32 ops/s", "frac": ref_ach / fp32_peak,
        "work": (f"the reference's per-action softmax step: {REF_OPS_PER_PSTEP} FP32 ops per particle-step "
                 f"(9m+10, m=96, SURVEY 8d); the factorised sampler needs fewer, so frac > 1 is possible")}
    roof["ncu"] = ncu
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "hz": 1000.0 / ms, "p50_ms": p50, "p99_ms": p99, "latency_cycles": n_lat,
        "config": {
            "workload": (f"{args.config}: {len(scene.spaces)} humans/GPU x {scene.n} particles x {scene.steps} "
                         f"steps dt {scene.dt}, |H|={scene.spaces[0].size}, |U|={len(scene.control_set)}, "
                         f"{scene.spec.width}x{scene.spec.height} @{scene.spec.resolution} m union, sigma 0.1 m, "
                         f"update+predict per cycle"),
            "mode": args.mode, "humans": len(scene.spaces) * world, "particles": scene.n,
            "horizon": scene.steps, "grid": [scene.spec.width, scene.spec.height],
            "fused_grid": (args.fused_path if fused else None), "parallelism": f"humans sharded over {world} GPU(s)",
            "l2": (f"per-cycle working set: {d2h / 1e6:.0f} MB f32 union + counts rewritten each cycle, "
                   f"{'above' if d2h > 126e6 else 'below'} the 126 MB L2 (no explicit flush)"),
        },
        "e2e": {"value": psteps / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h if (rank == 0 or not fused) else 0,
                "hz": 1000.0 / e2e_ms, "p50_latency_ms": e2e_p50, "p99_latency_ms": e2e_p99,
                "note": e2e_note},
        "gpu_launches": gpu_launches,
        "kernels_ms": {"k_predict": k2_ms, "k_epilogue": k3_ms},
        "roofline": roof,
        "clocks": clk,
    }
    if args.mode == "production" and not args.no_ref_mode:
        # the same cycle in deterministic (reference-RNG, bit-exact arithmetic) mode
        import dataclasses
        eng_r = CycleEngine(scene.control_set, scene.q, scene.spaces, scene.spec,
                            dataclasses.replace(cfg, mode="reference"),
                            human_ids=list(range(hpg * rank, hpg * rank + len(scene.spaces))))
        eng_r.prime(scene.warmup_track[0])
        eng_r.stage(scene.warmup_track[1], buf=0)
        eng_r.run_cycle(buf=0)
        torch.cuda.synchronize()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record()
        for _ in range(2):
            eng_r.run_cycle(buf=0, with_h2d=False)
        r1.record()
        torch.cuda.synchronize()
        rms = max_over_ranks(r0.elapsed_time(r1) / 2)
        line["reference_rng_mode"] = {"ms_per_step": rms, "hz": 1000.0 / rms, "value": psteps / (rms * 1e-3),
                                      "note": "same cycle with the reference's Philox4x64 streams regenerated "
                                              "in-register and its float32 step op for op (bit-exact counts)"}
        del eng_r
    if world == 1 and not args.no_cpu_baseline and rank == 0:
        line["cpu_baseline"] = cpu_sample(scene, t_steps=args.cpu_t, reps=3)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if peer is not None:
        peer.close()
    if distributed:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg3")
    ap.add_argument("--mode", default="production", choices=["production", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fused", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="take the multi-GPU path (NCCL group, fused reduce) even with one rank")
    ap.add_argument("--fused-path", default="nccl", choices=["nccl", "peer"],
                    help="N > 1 fused grid: NCCL max-reduce, or K3 writes over NVLink peer memory")
    ap.add_argument("--no-ref-mode", action="store_true")
    ap.add_argument("--lat-cycles", type=int, default=LAT_CYCLES,
                    help="cycles the p50/p99 latencies are taken over (at least --steps)")
    ap.add_argument("--chunks", type=int, default=7, help="horizon chunks of the e2e cycle (D2H overlap)")
    ap.add_argument("--chunk-taper", type=float, default=0.5, help="chunk size ratio (1.0 = uniform chunks)")
    ap.add_argument("--cpu-t", type=int, default=25)
    ap.add_argument("--ref-t", type=int, default=10)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
