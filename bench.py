#!/usr/bin/env python
"""Benchmark: the full predict+update cycle of BASELINE.json configs[2] (cfg3) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is one prediction cycle: belief update of every human (K1) + prediction of
every human (K2: 262,144 particles x 250 steps, dt 0.02) + smoothing and max-union into
the shared 400x400 grid (K3).  N GPUs: weak scaling, 8 humans per rank (one process per
GPU; ``--gpus N`` without torchrun re-launches itself under torch.distributed.run); with
N > 1 the per-rank unions are merged into one fused grid each cycle, by an NCCL
max-reduce of the nonzero 32 x 32 tiles only (``--fused-path nccl``: the ranks' tile flags
OR-ed, the flagged tiles packed, reduced and scattered back; ``nccl-dense`` reduces the
whole grid) or by every rank's K3 writing rank 0's grid over NVLink peer memory
(``--fused-path peer``).

``value``  -- particle-steps/s of the whole job, inputs resident in HBM (CUDA graph
              replay, CUDA events, max over ranks);  ``hz`` = cycles/s, ``p99_ms``.
``e2e``    -- the same metric end to end: the cycle's observations copied from pinned
              host memory and the fused (T, H, W) union read back to pinned host memory
              every cycle, in the reference's float64 layout (prediction.py:98-106,
              occupancy.py:176-187) -- the drop-in contract; ``e2e_f32`` is the same with
              a float32 union (half the D2H bytes).
``--impl reference`` times the reference CPU implementation (oracle/port.py, a
restatement pinned bit-exact to the reference) on the host cores on a bounded sample.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import platform
import socket
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
L2_BYTES = 126e6  # B200 L2; smaller per-cycle working sets get an L2 flush between timed cycles


def union_bytes(scene):
    """The per-cycle f64 (T, H, W) union every cycle rewrites (the dominant working set)."""
    return scene.steps * scene.spec.width * scene.spec.height * 8


def l2_flushed(scene):
    return union_bytes(scene) < L2_BYTES


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
# the workload (shared by both arms: their `config` dicts are identical)
# ---------------------------------------------------------------------------------------
def workload_config(args, scene, world):
    H = len(scene.spaces) * world
    return {
        "workload": (f"{args.config}: {H} humans ({len(scene.spaces)}/GPU) x {scene.n} particles x {scene.steps} "
                     f"steps dt {scene.dt}, |H|={scene.spaces[0].size}, |U|={len(scene.control_set)}, "
                     f"{scene.spec.width}x{scene.spec.height} @{scene.spec.resolution} m union, sigma 0.1 m, "
                     f"goals {scene.goal_radius:g} m from each start, update+predict per cycle"),
        "humans": H, "particles": scene.n, "horizon": scene.steps, "dt": scene.dt,
        "grid": [scene.spec.width, scene.spec.height], "resolution_m": scene.spec.resolution,
        "goal_radius_m": scene.goal_radius, "sigma_m": 0.1,
        "union": "max over humans, (T, H, W) on the host each cycle (e2e)",
        "parallelism": f"humans sharded over {world} GPU(s)" if world > 1 else "1 GPU",
        "l2": (f"per-cycle working set: {union_bytes(scene) / 1e6:.0f} MB f64 union + count windows rewritten "
               f"each cycle, " + ("below the 126 MB L2: a 256 MB buffer is written before every timed cycle and the "
                                  "writes' own event-timed durations are subtracted from the timed span"
                                  if l2_flushed(scene) else "above the 126 MB L2 (no explicit flush)")),
    }


def scene_for(args, rank=0, cycles=8):
    from paper_2603_01122_b200.scenario import CONFIGS, make_scene
    hpg = CONFIGS[args.config]["humans"]  # humans per GPU (weak scaling): cfg3 8, cfg1/cfg2 1
    return make_scene(args.config, cycles=cycles, humans=hpg, human_offset=hpg * rank,
                      goal_radius=args.goal_radius)


# ---------------------------------------------------------------------------------------
# CPU baseline: the reference CPU cycle (oracle/port.py) on a bounded sample of the workload
# ---------------------------------------------------------------------------------------
def host_info():
    info = {"cpu_model": platform.processor() or "unknown", "nproc": os.cpu_count(),
            "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None,
            "numpy": np.__version__, "python": platform.python_version()}
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    info["cpu_model"] = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        import scipy
        info["scipy"] = scipy.__version__
    except ImportError:
        pass
    try:
        import threadpoolctl
        blas = [d for d in threadpoolctl.threadpool_info() if d.get("internal_api") in ("openblas", "mkl", "blis")]
        if blas:
            info["blas"] = f"{blas[0]['internal_api']} {blas[0].get('version')} ({blas[0].get('architecture')})"
    except Exception:  # noqa: BLE001
        pass
    info["OPENBLAS_NUM_THREADS"] = os.environ.get("OPENBLAS_NUM_THREADS")
    return info


class CpuCycle:
    """One human's reference CPU cycle (belief update + predict of t_steps steps) on the
    scene; humans are taken round robin so every human's posterior is sampled."""

    def __init__(self, scene, t_steps):
        from oracle import model
        from oracle.predict import Grid, belief_update
        self.scene, self.t = scene, min(t_steps, scene.steps)
        cs = scene.control_set
        self.qs = model.QSpec("goal_progress", 0.5)
        self.tb = model.make_tables(cs.v, cs.theta, scene.dt, self.qs)
        self.grid = Grid(scene.spec.width, scene.spec.height, scene.spec.resolution)
        self.belief_update = belief_update
        # the posterior after the 10 warm-up observations (the bench's belief), per human
        self.lw = []
        for i, sp in enumerate(scene.spaces):
            lw = np.full(sp.size, -np.log(sp.size))
            for k in range(1, 11):
                lw, _ = belief_update(lw, scene.warmup_track[k - 1][i], scene.warmup_track[k][i], 0.1, cs.v, cs.theta,
                                      self.qs, sp.beta_of, sp.goal_xy_of, 0.0, snap_tol=float("inf"))
            self.lw.append(lw)
        self.k = 0

    def run(self, workers):
        from oracle import port
        sc, i = self.scene, self.k % len(self.scene.spaces)
        self.k += 1
        sp = sc.spaces[i]
        cs = sc.control_set
        t0 = time.perf_counter()
        post, _ = self.belief_update(self.lw[i], sc.warmup_track[10][i], sc.track[0][i], 0.1, cs.v, cs.theta,
                                     self.qs, sp.beta_of, sp.goal_xy_of, 0.0, snap_tol=float("inf"))
        t1 = time.perf_counter()
        port.predict(sc.track[0][i], post, sc.n, self.t, sc.dt, 0.1, 0, self.tb, sp.beta_of, sp.goal_xy_of,
                     self.grid, prefix=(2, i), workers=workers)
        t2 = time.perf_counter()
        return t1 - t0, t2 - t1

    def cycle_s(self, upd_s, pred_s, humans):
        """Extrapolate one sampled human x t steps to the whole cycle: predict is linear in
        T and in humans (cli.py:135-146; humans run sequentially, sim.py:493-499)."""
        return humans * (upd_s + pred_s * self.scene.steps / self.t)

    def extrapolation(self, humans):
        return {"sampled_humans": 1, "sampled_steps": self.t, "humans": humans, "steps": self.scene.steps,
                "factor_humans": humans, "factor_steps": self.scene.steps / self.t,
                "basis": "predict is linear in T and in humans (cli.py:135-146, sim.py:493-499); "
                         "one human's update + t-step predict timed, x humans x T/t"}


def worker_choices():
    n = os.cpu_count() or 1
    return sorted({None, 2, 4, n} - {0, 1}, key=lambda w: (w is not None, w or 0))


def cpu_sample(scene, humans, t_steps=10, runs=5):
    """OPENBLAS_NUM_THREADS=1, best of workers in {None, 2, 4, nproc}, each
    1 warm-up + ``runs`` timed runs (mean); the cycle extrapolated from one human x t_steps."""
    cc = CpuCycle(scene, t_steps)
    per = {}
    for w in worker_choices():
        cc.run(w)  # warm-up
        ts = [cc.run(w) for _ in range(runs)]
        per[str(w)] = cc.cycle_s(float(np.mean([a for a, _ in ts])), float(np.mean([b for _, b in ts])), humans)
    best = min(per, key=per.get)
    cycle_s = per[best]
    psteps = humans * scene.n * scene.steps
    w = None if best == "None" else int(best)
    return {
        "value": psteps / cycle_s, "unit": UNIT, "cores": w or 1, "kind": "port",
        "hz": 1.0 / cycle_s, "cycle_s": cycle_s, "workers": w, "cycle_s_by_workers": per,
        "sample": (f"1 human (round robin) x {scene.n} particles x {cc.t} steps + 1 belief update; best of "
                   f"workers {list(per)} (1 warm-up + {runs} runs each, mean); extrapolated x{humans} humans "
                   f"x{scene.steps / cc.t:g} in T (reference CPU path restated in oracle/port.py, "
                   f"OPENBLAS_NUM_THREADS=1)"),
        "extrapolation": cc.extrapolation(humans),
        "host": host_info(),
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return 0
    scene = scene_for(args, 0, cycles=2)
    humans = len(scene.spaces) * world
    cc = CpuCycle(scene, args.ref_t)
    # warm-up steps pick the worker count (best of BASELINE.md 5's set), timed steps use it
    choices = worker_choices()
    per = {}
    for i in range(max(args.warmup, len(choices))):
        w = choices[i % len(choices)]
        u, p = cc.run(w)
        per.setdefault(str(w), []).append(cc.cycle_s(u, p, humans))
    best = min(per, key=lambda k: float(np.mean(per[k])))
    w = None if best == "None" else int(best)
    cycles = []
    for _ in range(args.steps):
        u, p = cc.run(w)
        cycles.append(cc.cycle_s(u, p, humans))
    cycle_s = float(np.mean(cycles))
    v = humans * scene.n * scene.steps / cycle_s
    sample = (f"each step: 1 human (round robin) x {scene.n} particles x {cc.t} steps + 1 belief update, "
              f"extrapolated x{humans} humans x{scene.steps / cc.t:g} in T; workers={w} (best of "
              f"{list(per)} over the warm-up steps); reference CPU path restated in oracle/port.py")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": cycle_s * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "hz": 1.0 / cycle_s,
        "p99_ms": float(np.percentile(cycles, 99)) * 1e3,
        "config": workload_config(args, scene, world),
        "extrapolated": True, "extrapolation": cc.extrapolation(humans),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": w or 1, "kind": "port", "sample": sample,
                         "host": host_info()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------
# N GPUs: one process per GPU
# ---------------------------------------------------------------------------------------
def relaunch(args):
    """``--gpus N`` without torchrun: re-launch this script under torch.distributed.run
    with N ranks (127.0.0.1 rendezvous), failing loudly when the box has fewer GPUs."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but this box has {have} CUDA device(s)", file=sys.stderr, flush=True)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr, flush=True)
        return 2
    torch.cuda.set_device(local)
    # --force-dist: run the multi-GPU code path (NCCL process group, fused reduce) even
    # at world size 1 -- a one-rank smoke test of the N > 1 branch on a single GPU
    distributed = world > 1 or args.force_dist
    if distributed:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator INIT lines (N ranks) on stdout
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        assert dist.get_world_size() == world
    from paper_2603_01122_b200 import _lib
    from paper_2603_01122_b200.engine import CycleEngine, EngineConfig, fused_reduce

    K, W = args.steps, args.warmup
    scene = scene_for(args, rank, cycles=W + K + 4)
    hpg = len(scene.spaces)
    ids = list(range(hpg * rank, hpg * rank + hpg))
    fused = distributed and not args.no_fused
    fused_path = args.fused_path if fused else None
    if rank == 0 and distributed:
        print(f"bench.py: {world} rank(s), fused grid: "
              f"{'none' if not fused else ('NVLink peer-memory atomicMax (peer.PeerUnion)' if fused_path == 'peer' else ('NCCL max-reduce of the whole grid to rank 0' if fused_path == 'nccl-dense' else 'NCCL max-reduce of the nonzero tiles to rank 0'))}",
              file=sys.stderr, flush=True)

    def make_engine(union_dtype, peer=None):
        cfg = EngineConfig(n=scene.n, steps=scene.steps, dt=scene.dt, smoothing_sigma=0.1, seed=0,
                           mode=args.mode, time_union=False, chunk_taper=args.chunk_taper, union_dtype=union_dtype)
        eng = CycleEngine(scene.control_set, scene.q, scene.spaces, scene.spec, cfg, human_ids=ids, peer=peer)
        # posterior after 10 observations (also warms every kernel)
        eng.prime(scene.warmup_track[0])
        for k in range(1, 11):
            eng.stage(scene.warmup_track[k], buf=k % 2)
            eng.run_cycle(buf=k % 2)
        torch.cuda.synchronize()
        eng.check_errors()
        return eng

    udt = torch.float64 if args.union_dtype == "float64" else torch.float32
    peer = None
    if fused_path == "peer":
        from paper_2603_01122_b200.peer import PeerUnion
        peer = PeerUnion((scene.steps, scene.spec.height, scene.spec.width), udt)
    eng = make_engine(args.union_dtype, peer)

    def sparse_tiles(e, b):
        """The union-tile flags the sparse NCCL reduce moves by, or None (dense reduce)."""
        if fused_path != "nccl" or e.utile is None or e.cfg.time_union:
            return None
        return e.utile[b]

    def device_cycle(g, e, b=0):
        """One graph-replayed cycle plus the fused-grid merge (on the current stream)."""
        if peer is not None:
            peer.zero(b)
            peer.barrier()
            g.replay()
            peer.barrier()
        else:
            g.replay()
            if fused:
                fused_reduce(e.unions[b], dst=0, tiles=sparse_tiles(e, b))

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
    # working sets below L2 (cfg1, cfg2): evict it between timed cycles (on `stream`, before
    # each cycle's start event), and time the cycles one by one
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if l2_flushed(scene) else None

    flush_ev = []  # (start, end) event pairs around the flushes, subtracted from the timed spans

    def l2_flush():
        if flush_buf is not None:
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record()
            flush_buf.zero_()
            b_.record()
            flush_ev.append((a_, b_))

    def flush_ms(i0, i1=None):
        """Total time of the flushes flush_ev[i0:i1]."""
        return sum(a_.elapsed_time(b_) for a_, b_ in flush_ev[i0:i1])

    # ---- kernel timing inside the replayed graph: event-record nodes before K2, after K2,
    # after K3 (the same graph and clock as ms_per_step) ----
    kev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(3)]
    gk = eng.capture(buf=0, with_h2d=False, events=kev)
    n_k = max(3, min(K, 10))
    k2, k3 = [], []
    with torch.cuda.stream(stream):
        for i in range(n_k + 2):
            l2_flush()
            gk.replay()
            stream.synchronize()
            if i >= 2:
                k2.append(kev[0].elapsed_time(kev[1]))
                k3.append(kev[1].elapsed_time(kev[2]))
    barrier()
    k2_ms, k3_ms = max_over_ranks(float(np.mean(k2))), max_over_ranks(float(np.mean(k3)))

    # ---- value: device-resident cycle (CUDA graph replay) ----
    g = eng.capture(buf=0, with_h2d=False)
    cyc_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    with torch.cuda.stream(stream):
        for _ in range(W):
            device_cycle(g, eng)
    launches0 = _lib.lib().gc_launch_count()
    barrier()
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local).__enter__()
    f0 = len(flush_ev)
    with torch.cuda.stream(stream):
        t_start.record(stream)
        for i in range(K):
            l2_flush()
            cyc_ev[i][0].record(stream)
            device_cycle(g, eng)
            cyc_ev[i][1].record(stream)
        t_end.record(stream)
    barrier()
    ms = (t_start.elapsed_time(t_end) - flush_ms(f0)) / K  # (the flushes, if any, excluded)
    launches_timed = _lib.lib().gc_launch_count() - launches0  # eager launches in the timed cycles
    ms = max_over_ranks(ms)
    per_cycle = [a.elapsed_time(b) for a, b in cyc_ev]
    # latency percentiles over >= LAT_CYCLES cycles: extra untimed-for-value replays
    n_lat = max(args.lat_cycles, K)
    extra = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_lat - K)]
    with torch.cuda.stream(stream):
        for a_, b_ in extra:
            a_.record(stream)
            device_cycle(g, eng)
            b_.record(stream)
    barrier()
    per_cycle += [a.elapsed_time(b) for a, b in extra]
    p99 = max_over_ranks(float(np.percentile(per_cycle, 99)))
    p50 = max_over_ranks(float(np.percentile(per_cycle, 50)))
    # graph replays do not pass through the C ABI launch counter: 3 kernels per cycle
    # (K1 belief, K2 predict, K3 epilogue) are captured in the graph
    # plus, with N > 1 and the sparse fused reduce, the eager tile gather (every rank) and
    # scatter (rank 0) of gc_union_tiles around the NCCL reduce -- nothing else runs eagerly
    gpu_launches = 3 * K + launches_timed
    assert launches_timed <= (2 * K if fused and fused_path == "nccl" else 0), launches_timed

    psteps_rank = hpg * scene.n * scene.steps
    psteps = psteps_rank * world
    ushape = (scene.steps, scene.spec.height, scene.spec.width)

    # ---- e2e: pinned H2D of observations + D2H of the fused union every cycle ----
    def e2e(e, dtype):
        h2d = e._nb
        d2h = math.prod(ushape) * (8 if dtype == torch.float64 else 4)
        tr = scene.track
        h_out = [torch.empty(ushape, dtype=dtype).pin_memory() for _ in range(2)]
        if not fused:
            # one CUDA graph per cycle: H2D of the observations, update, predict in
            # args.chunks horizon chunks whose layers stream to pinned host memory on a
            # copy stream while the next chunk computes; cycles run strictly one after
            # another, so the per-cycle time is the host-in -> host-out latency
            ga = [e.capture(buf=b, with_h2d=True, chunks=args.chunks, d2h=h_out[b]) for b in (0, 1)]
            done = [torch.cuda.Event() for _ in range(2)]

            def e2e_loop(n_cycles, base):
                evs = []
                for i in range(n_cycles):
                    b = i % 2
                    done[b].synchronize()           # pinned input/output b free again
                    e.stage(tr[(base + i) % len(tr)], buf=b)
                    with torch.cuda.stream(stream):
                        l2_flush()
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
            f0 = len(flush_ev)
            evs = e2e_loop(K, W)
            f1 = len(flush_ev)
            e_end.record(stream)
            barrier()
            evs += e2e_loop(n_lat - K, W + K)  # latency samples only
            barrier()
            note = (f"per cycle: pinned obs H2D + update + predict in {args.chunks} horizon chunks "
                    f"(sizes {[b - a for a, b in e.chunk_bounds(args.chunks)]}), each chunk's "
                    f"{'f64' if dtype == torch.float64 else 'f32'} union layers D2H on a copy stream while the "
                    f"next computes; cycles strictly sequential (latency = cycle time), one CUDA graph")
        else:
            # N > 1: the fused grid is merged by the NCCL max-reduce (or written in place over
            # peer memory); rank 0 reads it back, D2H of cycle k overlapped with cycle k+1
            # (double-buffered unions; with peer memory rank 0 re-zeroes buffer b after its
            # D2H, and every rank's next write of b follows the barrier that waits for that)
            ga = [e.capture(buf=b, with_h2d=True) for b in (0, 1)]
            copy = torch.cuda.Stream()
            done = [torch.cuda.Event() for _ in range(2)]
            copied = [torch.cuda.Event() for _ in range(2)]
            staged_ok = [torch.cuda.Event() for _ in range(2)]

            def e2e_loop(n_cycles, base):
                evs = []
                for i in range(n_cycles):
                    b = i % 2
                    staged_ok[b].synchronize()
                    e.stage(tr[(base + i) % len(tr)], buf=b)
                    with torch.cuda.stream(stream):
                        stream.wait_event(copied[b])
                        l2_flush()
                        s_ev = torch.cuda.Event(enable_timing=True)
                        s_ev.record(stream)
                        if e.peer is not None:
                            e.peer.barrier()      # rank 0's zero of b precedes every rank's writes
                        ga[b].replay()
                        staged_ok[b].record(stream)
                        if e.peer is not None:
                            e.peer.barrier()      # every rank's K3 writes precede rank 0's read
                        else:  # (the sparse reduce also OR-s the ranks' tile flags)
                            fused_reduce(e.unions[b], dst=0, tiles=sparse_tiles(e, b))
                        if e.utile is not None and (e.peer is not None or sparse_tiles(e, b) is None):
                            # the fused grid's nonzero tiles: OR of the ranks'
                            dist.reduce(e.utile[b], dst=0, op=dist.ReduceOp.MAX)
                        done[b].record(stream)
                    with torch.cuda.stream(copy):
                        copy.wait_event(done[b])
                        if rank == 0:
                            src = e.peer.tensor(b) if e.peer is not None else e.unions[b]
                            if e.utile is not None:  # tile-sparse publication of the fused grid
                                e.publish(b, h_out[b], union=src, stream=copy)
                            else:
                                h_out[b].copy_(src, non_blocking=True)
                            if e.peer is not None:
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
            f0 = len(flush_ev)
            evs = e2e_loop(K, W)
            f1 = len(flush_ev)
            stream.wait_stream(copy)
            e_end.record(stream)
            barrier()
            evs += e2e_loop(n_lat - K, W + K)  # latency samples only
            stream.wait_stream(copy)
            barrier()
            note = ("pinned obs H2D + " + ("peer-memory fused union (K3 atomicMax into rank 0's grid over "
                    "NVLink)" if e.peer is not None else "NCCL fused union") +
                    f" + rank-0 {'f64' if dtype == torch.float64 else 'f32'} "
                    f"{'tile-sparse publication (tile flags OR-reduced over ranks)' if e.utile is not None else 'D2H'}"
                    f" each cycle, overlapped with the next cycle")
        lat = [a_.elapsed_time(b_) for a_, b_ in evs]
        e_ms = max_over_ranks((e_start.elapsed_time(e_end) - flush_ms(f0, f1)) / K)  # (flushes excluded)
        e.check_errors()
        return {"value": psteps / (e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h if (rank == 0 or not fused) else 0,
                "dtype": "f64" if dtype == torch.float64 else "f32",
                "hz": 1000.0 / e_ms, "ms_per_step": e_ms,
                "p50_latency_ms": max_over_ranks(float(np.percentile(lat, 50))),
                "p99_latency_ms": max_over_ranks(float(np.percentile(lat, 99))), "note": note}

    e2e_main = e2e(eng, udt)
    other = None
    if not args.no_e2e_alt:
        # the other union precision through a second engine (same scene, same cycle)
        odt = "float32" if args.union_dtype == "float64" else "float64"
        opeer = None
        if fused_path == "peer":
            from paper_2603_01122_b200.peer import PeerUnion
            opeer = PeerUnion((scene.steps, scene.spec.height, scene.spec.width),
                              torch.float32 if odt == "float32" else torch.float64)
        eng2 = make_engine(odt, opeer)
        other = e2e(eng2, torch.float32 if odt == "float32" else torch.float64)
        del eng2
        if opeer is not None:
            opeer.close()
    clocks.__exit__(None, None, None)

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
    if ncu and ncu.get("workload") not in (None, args.config):
        ncu = None  # the captured per-particle-step figures belong to another workload
    ipp = (ncu or {}).get("lane_instr_per_particle_step")
    mpp = (ncu or {}).get("mufu_per_particle_step")
    traffic = (ncu or {}).get("dram_bytes_per_launch")
    k2_s = k2_ms * 1e-3
    # K2 is bound by SM instruction issue (no dense contraction, ~1 GB/s of HBM): the
    # roofline is executed lane-instructions per particle-step (ncu, static for this code
    # and workload) x particle-steps of the launch / the launch time inside the replayed graph
    roof = {"bound": "issue", "kernel": "k_predict", "achieved": None, "peak": issue_peak,
            "unit": "T lane-instr/s", "frac": None, "traffic": traffic, "work": None,
            "timing": "CUDA event-record nodes around K2 inside the replayed cycle graph (same clock as ms_per_step)",
            "peak_source": f"148 SM x 4 schedulers x 32 lanes x {sm_mhz:.0f} MHz ({pk['source']} sm_max_mhz)"}
    if ipp:
        ach = psteps_rank * ipp / k2_s / 1e12
        roof.update(achieved=ach, frac=ach / issue_peak,
                    work=f"{ipp} lane-instructions per particle-step (ncu) x {psteps_rank} particle-steps per launch")
    if mpp:
        xa = psteps_rank * mpp / k2_s / 1e12
        roof["xu"] = {"achieved": xa, "peak": xu_peak, "unit": "T MUFU lane-ops/s", "frac": xa / xu_peak,
                      "mufu_per_particle_step": mpp,
                      "note": "second bound: heading ex2s + speed-weight ex2 + chosen-heading ex2 + rsqrt per particle-step"}
    if traffic:
        gbs = traffic / k2_s / 1e9
        roof["hbm"] = {"achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s", "frac": gbs / pk["hbm_gbs"],
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
        "mode": args.mode, "fused_grid": fused_path, "union_dtype": args.union_dtype,
        "config": workload_config(args, scene, world),
        "e2e": e2e_main,
        "gpu_launches": gpu_launches,
        "kernels_ms": {"k_predict": k2_ms, "k_epilogue": k3_ms, "cycle": ms,
                       "k_predict_share": k2_ms / ms},
        "roofline": roof,
        "clocks": clk,
    }
    if other is not None:
        line["e2e_" + other["dtype"]] = other
    line["e2e_contract"] = ("e2e: the fused union on the host in the reference's float64 (T, H, W) layout"
                            if e2e_main["dtype"] == "f64" else
                            "e2e: float32 union on the host; e2e_f64 is the reference's float64 layout")
    if args.mode == "production" and not args.no_ref_mode:
        # the same cycle in deterministic (reference-RNG, bit-exact arithmetic) mode
        import dataclasses
        eng_r = CycleEngine(scene.control_set, scene.q, scene.spaces, scene.spec,
                            dataclasses.replace(eng.cfg, mode="reference"), human_ids=ids)
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
        line["cpu_baseline"] = cpu_sample(scene, hpg * world, t_steps=args.cpu_t, runs=args.cpu_runs)
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
    ap.add_argument("--goal-radius", type=float, default=None,
                    help="goal distance from each start in m (default 0.35 x room, SURVEY 8(d))")
    ap.add_argument("--mode", default="production", choices=["production", "reference"])
    ap.add_argument("--union-dtype", default="float64", choices=["float64", "float32"],
                    help="union precision of the headline e2e (float64 = the reference's layout)")
    ap.add_argument("--no-e2e-alt", action="store_true", help="skip the e2e block in the other union precision")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fused", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="take the multi-GPU path (NCCL group, fused reduce) even with one rank")
    ap.add_argument("--fused-path", default="nccl", choices=["nccl", "nccl-dense", "peer"],
                    help="N > 1 fused grid: NCCL max-reduce of the nonzero tiles (or of the whole grid), "
                         "or K3 writes over NVLink peer memory")
    ap.add_argument("--no-ref-mode", action="store_true")
    ap.add_argument("--lat-cycles", type=int, default=LAT_CYCLES,
                    help="cycles the p50/p99 latencies are taken over (at least --steps)")
    ap.add_argument("--chunks", type=int, default=4, help="horizon chunks of the e2e cycle (D2H overlap)")
    ap.add_argument("--chunk-taper", type=float, default=0.5, help="chunk size ratio (1.0 = uniform chunks)")
    ap.add_argument("--cpu-t", type=int, default=10, help="steps of the CPU baseline sample (<= 10, BASELINE.md 5)")
    ap.add_argument("--cpu-runs", type=int, default=5)
    ap.add_argument("--ref-t", type=int, default=10)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
