"""CycleEngine: the batched, device-resident update + predict cycle of many humans.

This is the reference's closed-loop caller pattern (sim.py:455-514) -- per observation
every human's belief is updated (belief.py:159-198), then every human is predicted with
its own hypothesis space, the stationary-masked Q when it stands still (sim.py:480,
:495), prefix (HUMAN_PREFIX, i) and cycle seed derive_seed(seed, 7, k), and the layers
are merged by the max union (+ optional conservative time union, sim.py:500-504) --
restructured for the B200:

  * all state (posteriors, count windows, the fused (T, H, W) union) stays in HBM;
  * one packed pinned H2D copy of the cycle's observations, then K1 (gc_belief_update,
    warp per human) -> memsets -> K2 (gc_predict, all humans in one launch) -> K3
    (gc_grid_epilogue: smoothing + atomicMax union [+ time union]);
  * the whole cycle is captured once in a CUDA graph and replayed;
  * optionally the union is read back to pinned host memory on a copy stream,
    double-buffered so the D2H of cycle k overlaps the compute of cycle k+1.

Multi-GPU: one engine per rank over that rank's humans; when a single fused grid is
requested either ``fused_reduce`` merges the per-rank unions with NCCL (max), or every
rank's K3 writes the owner's grid directly over NVLink peer memory (``peer.PeerUnion``).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .belief import belief_tables, launch_belief_update, mask_stationary
from .device import device
from .prediction import MODES, action_tables, geometry
from .rng import HUMAN_PREFIX, SIM_PREDICT, derive_seed
from .tables import assume_qg, hypothesis_arrays


@dataclass
class EngineConfig:
    n: int = 262_144
    steps: int = 250
    dt: float = 0.02
    smoothing_sigma: float = 0.1
    seed: int = 0
    mode: str = "production"
    obs_dt: float = 0.1
    stationary_speed: float = 0.05     # sim.py:480 (observed speed below -> masked Q)
    stationary_mask_v: float = 0.5     # mask_stationary threshold (sim.py:111)
    union_dtype: str = "float32"       # fused union precision: float32 | float64
    # "max" (occupancy.union_max, the sim's union) or "independent" 1 - prod(1 - p)
    # (occupancy.py:180-184); independent keeps per-human float64 layers and merges them
    # in human order.  union_partial: keep prod(1 - p) of this rank's humans instead, for
    # fused_reduce(..., mode="independent") across GPUs.
    union_mode: str = "max"
    union_partial: bool = False
    time_union: bool = False
    per_human_layers: bool = False
    # planner input (anastar.py:107-119, mppi.py:87-94): collision field of the fused
    # union thresholded into a (T, H, W) uint8 blocked mask each cycle; None = off
    robot_radius: Optional[float] = None
    collision_threshold: float = 0.1
    # particle-block sharding of every human over GPUs: (shard index, shard count); this
    # engine runs particles [i*n/k, (i+1)*n/k) of each human and its u32 counts must be
    # summed over the shards (``counts_reduce``) before the epilogue divides by n
    particle_shard: Optional[tuple] = None
    # horizon chunking (chunks > 1): chunk c spans ~ chunk_taper^c of the horizon, so the
    # last chunks -- whose D2H cannot overlap later compute -- are short; 1.0 = uniform
    chunk_taper: float = 0.5
    # shared-memory budget (KB) of K2's count window: a one-chunk
    # horizon whose last windows exceed it is split so its first part still runs on
    # shared-memory windows.  Off by default: at the cfg4 shard (T = 500, 2^20 particles
    # per human) the split measured 42.8 ms per cycle against 40.4 ms on the global path
    window_budget_kb: float = 0.0
    # K2's per-step histogram (gc_predict_args.hist_path): "global" -- warp-aggregated
    # reductions straight into the count windows (default; 3-5 % faster at every belief
    # shape measured) -- or "smem" -- shared-memory windows where they fit
    # (window_budget_kb then splits long horizons)
    hist_path: str = "global"
    # reference RNG mode: K2 evaluates the action weights with the hardware ex2 and runs
    # numpy's exp only where the pick is within the proven error margin (bit-identical
    # either way, gc_predict_args.ref_exact_only); False = numpy's exp everywhere
    ref_filter: bool = True
    # host read-back of the union (run_cycle / capture with d2h=...): "tiles" publishes only
    # the 32 x 32 tiles that are nonzero now or were nonzero in the host stack's previous
    # cycle (gc_publish_tiles: kernel stores into the pinned, mapped host stack); "dense"
    # copies every layer.  The host stack is bit-identical either way.
    d2h_mode: str = "tiles"


class CycleEngine:
    def __init__(self, control_set, q_model, spaces: Sequence, grid_spec, cfg: EngineConfig,
                 initial_log_weights: Optional[Sequence[np.ndarray]] = None,
                 human_ids: Optional[Sequence[int]] = None, counts_reduce=None, peer=None):
        self.dev = device()
        self.cfg = cfg
        self.counts_reduce = counts_reduce
        # peer: a peer.PeerUnion -- K3 atomicMax-es this engine's humans into the fused grid
        # of the owning rank (NVLink peer memory) instead of a local union; the owner zeroes
        # and reads it between PeerUnion.barrier() calls
        self.peer = peer
        if peer is not None:
            if cfg.union_mode != "max" or cfg.per_human_layers or cfg.robot_radius is not None:
                raise ValueError("a peer union takes the max union only (no per-human layers / blocked mask)")
            if cfg.time_union:
                raise ValueError("with a peer union the owner applies the time union (PeerUnion.finish)")
            want = torch.float32 if cfg.union_dtype == "float32" else torch.float64
            if peer.dtype != want or peer.shape != (cfg.steps, grid_spec.height, grid_spec.width):
                raise ValueError("PeerUnion shape/dtype must match (steps, H, W) and union_dtype")
        if cfg.particle_shard is not None:
            i, k = cfg.particle_shard
            if not (0 <= i < k) or cfg.n % k or (cfg.n // k) % 4:
                raise ValueError("particle_shard (i, k) needs 0 <= i < k, k | n and n / k a multiple of 4")
            self.n_local, self.p_offset = cfg.n // k, i * (cfg.n // k)
        else:
            self.n_local, self.p_offset = cfg.n, 0
        self.spec = grid_spec
        self.n_humans = len(spaces)
        self.control_set = control_set
        self.q_model = q_model
        self.q_masked = mask_stationary(q_model, control_set, cfg.stationary_mask_v)
        dev = self.dev
        self.tables = [action_tables(control_set, q_model, cfg.dt, dev),
                       action_tables(control_set, self.q_masked, cfg.dt, dev)]
        self.btab = belief_tables(control_set, q_model, dev)
        max_step = max(t.max_step for t in self.tables)
        self.geo = geometry(grid_spec, cfg.steps, max_step, float(cfg.smoothing_sigma), dev)
        H = self.n_humans
        betas, goals, off = [], [], [0]
        for sp in spaces:
            b, g = hypothesis_arrays(sp)
            if len(b) > _lib.GC_MAX_HYPOTHESES:
                raise NotImplementedError(f"at most {_lib.GC_MAX_HYPOTHESES} hypotheses per human")
            betas.append(b)
            goals.append(g)
            off.append(off[-1] + len(b))
        self.hyp_off = np.array(off, dtype=np.int32)
        up = lambda a, t: torch.as_tensor(np.array(a, dtype=t, order="C"), device=dev)
        self.d_hyp_off = up(self.hyp_off, np.int32)
        self.d_beta64 = up(np.concatenate(betas), np.float64)
        self.d_goal64 = up(np.concatenate(goals), np.float64)
        self.d_beta32 = up(np.concatenate(betas).astype(np.float32), np.float32)
        self._betas_np = betas  # host copy for gc_predict_args.assume_qg
        self.d_goal32 = up(np.concatenate(goals).astype(np.float32), np.float32)
        if initial_log_weights is None:
            lw = np.concatenate([np.full(len(b), -np.log(len(b))) for b in betas])
        else:
            lw = np.concatenate([np.asarray(x, dtype=float) for x in initial_log_weights])
        self.d_logw = up(lw, np.float64)
        self.d_status = torch.zeros(H, dtype=torch.int32, device=dev)
        # global human ids: prefix (HUMAN_PREFIX, i) and production stream id are the
        # same for a human whatever GPU / batch slot it lands on
        self.human_ids = np.arange(H) if human_ids is None else np.asarray(human_ids, dtype=np.int64)
        pre = np.zeros((H, 4), dtype=np.uint32)
        pre[:, 0] = HUMAN_PREFIX
        pre[:, 1] = self.human_ids.astype(np.uint32)
        self.d_prefix = up(pre, np.uint32)
        self.d_sid = up(self.human_ids.astype(np.uint32), np.uint32)
        self.d_plen = up(np.full(H, 2), np.int32)
        # packed per-cycle inputs: f64 [obs (H,4) | fallback (H,)], u64 seeds (H,),
        # f32 start (H,2), i32 table ids (H,)
        self._nb = H * 5 * 8 + H * 8 + H * 2 * 4 + H * 4
        self._nb = (self._nb + 15) // 16 * 16
        # two pinned staging buffers so the host can pack cycle k+1 while cycle k runs
        # zero-filled: a buffer captured or run before its first stage() holds a benign cycle
        # (start (0, 0), table 0) instead of uninitialised pinned memory
        self.h_ins = [torch.zeros(self._nb, dtype=torch.uint8).pin_memory() for _ in range(2)]
        self.h_in = self.h_ins[0]
        self.d_in = torch.empty(self._nb, dtype=torch.uint8, device=dev)
        o = 0
        self.d_obs = self.d_in[o:o + H * 32].view(torch.float64); o += H * 32
        self.d_fallback = self.d_in[o:o + H * 8].view(torch.float64); o += H * 8
        self.d_seed = self.d_in[o:o + H * 8].view(torch.int64); o += H * 8
        self.d_start = self.d_in[o:o + H * 8].view(torch.float32); o += H * 8
        self.d_tid = self.d_in[o:o + H * 4].view(torch.int32); o += H * 4
        self._views = [self._host_views(b.numpy(), H) for b in self.h_ins]
        self._select(0)
        self.counts = torch.zeros(H * self.geo.human_stride, dtype=torch.int32, device=dev)
        udt = torch.float32 if cfg.union_dtype == "float32" else torch.float64
        T, Hh, W = cfg.steps, grid_spec.height, grid_spec.width
        if peer is None:
            self.unions = [torch.zeros((T, Hh, W), dtype=udt, device=dev) for _ in range(2)]
        else:  # the owner's fused grids (None on the other ranks)
            self.unions = [peer.tensor(b) if peer.is_owner else None for b in range(2)]
        if cfg.union_mode not in ("max", "independent"):
            raise ValueError(f"unknown union mode {cfg.union_mode!r}")
        if cfg.union_partial and cfg.union_mode != "independent":
            raise ValueError("union_partial applies to the independent union")
        self.layers = (torch.zeros((H, T, Hh, W), dtype=torch.float64, device=dev)
                       if cfg.per_human_layers or cfg.union_mode == "independent" else None)
        self.d_err = torch.zeros(1, dtype=torch.int32, device=dev)
        if cfg.hist_path not in ("global", "smem"):
            raise ValueError(f"unknown hist_path {cfg.hist_path!r}")
        if cfg.d2h_mode not in ("tiles", "dense"):
            raise ValueError(f"unknown d2h_mode {cfg.d2h_mode!r}")
        # 32 x 32 union tiles K3 made nonzero this cycle, per union buffer (tile-sparse D2H)
        self.tile_grid = (T, -(-Hh // 32), -(-W // 32))
        self.utile = (torch.zeros((2,) + self.tile_grid, dtype=torch.uint8, device=dev)
                      if cfg.d2h_mode == "tiles" and cfg.union_mode == "max" else None)
        self._hflags = {}  # pinned host stack (data_ptr) -> its device-side tile-state flags
        self.blocked = None
        if cfg.robot_radius is not None:
            from .occupancy import disc_offsets
            self._disc = np.ascontiguousarray(disc_offsets(grid_spec, cfg.robot_radius))
            self.blocked = [torch.zeros((T, Hh, W), dtype=torch.uint8, device=dev) for _ in range(2)]
        self._tarr = (_lib.ActionTable * 2)(*[t.struct for t in self.tables])
        # production: the factorised sampler's fast speed-weight form holds for every
        # hypothesis (static: hypothesis spaces and tables are fixed) -- K2 checks it per CTA
        self._assume_qg = int(cfg.mode == "production" and assume_qg(self.tables, self._betas_np))
        self.last_xy = None
        # stage() of an unprimed engine: that cycle has no previous observation, so (like
        # sim.py:462-485, which updates only when last_xy is set) it predicts without an update
        self._skip_update = [False, False]
        self._stream = None  # the stream of the last cycle (belief reads/writes are ordered on it)
        # per pinned input buffer: the event after run_cycle's H2D copy out of it; stage()
        # waits for it before overwriting the buffer (cycles are issued asynchronously)
        self._h2d_done = [None, None]
        self.heading = np.zeros(H)
        self.cycle = 0
        self.graphs = {}
        self.h_out = None

    @staticmethod
    def _host_views(hnp, H):
        o = 0
        obs = hnp[o:o + H * 32].view(np.float64).reshape(H, 4); o += H * 32
        fb = hnp[o:o + H * 8].view(np.float64); o += H * 8
        seed = hnp[o:o + H * 8].view(np.uint64); o += H * 8
        start = hnp[o:o + H * 8].view(np.float32).reshape(H, 2); o += H * 8
        tid = hnp[o:o + H * 4].view(np.int32); o += H * 4
        return obs, fb, seed, start, tid

    def _select(self, buf):
        self.h_obs, self.h_fallback, self.h_seed, self.h_start, self.h_tid = self._views[buf]

    def prime(self, xy):
        """Record the observation preceding the first cycle (sim.py:462, :485)."""
        self.last_xy = np.asarray(xy, dtype=float).copy()

    # ---- host-side packing of one observation cycle ----------------------------------
    def stage(self, obs_xy: np.ndarray, buf: int = 0):
        """Pack the cycle's observations (H, 2) float64 into the pinned input buffer.

        Without a previous observation (no ``prime`` and no earlier cycle) the cycle only
        predicts from ``obs_xy``: no belief update, unmasked Q (sim.py:462-485 updates and
        sets ``stationary`` only once ``last_xy`` exists).  ``run_cycle`` honours this;
        a captured graph always contains the update, so replay it only on primed cycles."""
        obs_xy = np.asarray(obs_xy, dtype=float)
        if obs_xy.shape != (self.n_humans, 2) or not np.isfinite(obs_xy).all():
            raise ValueError(f"stage(): observations must be a finite ({self.n_humans}, 2) array")
        if self._h2d_done[buf] is not None:
            self._h2d_done[buf].synchronize()  # the previous cycle's copy out of this buffer is done
            self._h2d_done[buf] = None
        self._select(buf)
        primed = self.last_xy is not None
        prev = self.last_xy if primed else obs_xy
        self._skip_update[buf] = not primed
        self.h_obs[:, 0:2] = prev
        self.h_obs[:, 2:4] = obs_xy
        self.h_fallback[:] = self.heading
        d = obs_xy - prev
        moved = np.hypot(d[:, 0], d[:, 1])
        stationary = (moved / self.cfg.obs_dt < self.cfg.stationary_speed) & primed
        self.h_tid[:] = stationary.astype(np.int32)
        mv = moved > 1e-9
        self.heading = np.where(mv, np.arctan2(d[:, 1], d[:, 0]), self.heading)
        self.h_start[:] = obs_xy.astype(np.float32)
        self.h_seed[:] = np.uint64(derive_seed(self.cfg.seed, SIM_PREDICT, self.cycle))
        self.last_xy = obs_xy.copy()
        self.cycle += 1

    # ---- the device cycle ---------------------------------------------------------------
    def chunk_bounds(self, chunks: int):
        """1-based [t0, t1) step ranges of ``chunks`` horizon chunks; every chunk start is
        1 + a multiple of 4 (the turn phase of the production streams' small-launch path).  Chunk sizes shrink
        geometrically (``cfg.chunk_taper``) toward the end of the horizon."""
        T = self.cfg.steps
        chunks = max(1, min(chunks, (T + 3) // 4))
        w = [self.cfg.chunk_taper ** c for c in range(chunks)]
        starts, acc = [1], 0.0
        for c in range(chunks - 1):
            acc += w[c]
            s = 1 + 4 * int(round(T * acc / sum(w) / 4))
            if starts[-1] < s <= T:
                starts.append(s)
        return [(t0, t1) for t0, t1 in zip(starts, starts[1:] + [T + 1])]

    def window_bounds(self):
        """1-based [t0, t1) ranges of a one-chunk cycle: the whole horizon, or -- when its
        reachable-cell windows outgrow ``cfg.window_budget_kb`` of shared memory -- the
        longest prefix (ending on a 4-step boundary) whose windows fit, then the rest
        (K2 adds those steps straight to global memory).  Bit-identical either way."""
        T, cells = self.cfg.steps, self.geo.win_cells
        budget = self.cfg.window_budget_kb * 1024

        def fits(c):  # u16 counters two per word (rounded to 4 words)
            return ((int(c) + 1) // 2 + 3) // 4 * 16 <= budget

        if budget <= 0 or fits(cells[T - 1]) or self.counts_reduce is not None or self.cfg.hist_path != "smem":
            return [(1, T + 1)]
        t = 1
        while t + 4 <= T and fits(cells[t + 4 - 2]):
            t += 4
        return [(1, T + 1)] if t <= 1 else [(1, t), (t, T + 1)]

    def _ensure_state(self):
        if getattr(self, "state_xy", None) is None:
            N = self.n_humans * self.n_local
            self.state_xy = torch.empty(N * 2, dtype=torch.float32, device=self.dev)
            self.state_hyp = torch.empty(N, dtype=torch.uint8, device=self.dev)

    def _launch(self, buf: int, with_update: bool, stream, events=None, chunks: int = 1,
                d2h=None, copy_stream=None):
        """One cycle.  With chunks > 1 the horizon runs as several K2+K3 launches that hand
        particle state over; if ``d2h`` (pinned host tensor shaped like the union) is given,
        each chunk's layers are copied to it on ``copy_stream`` while later chunks compute."""
        cfg, geo, H = self.cfg, self.geo, self.n_humans
        sh = ctypes.c_void_p(stream.cuda_stream)
        self._stream = stream
        # the output fills run on a side stream concurrently with K1 (K1 occupies one warp
        # per human; the fills are HBM-bound): fork from, and join back into, `stream`
        u = self.unions[buf]
        if getattr(self, "_fill_stream", None) is None:
            self._fill_stream = torch.cuda.Stream(device=self.dev)
        fill = self._fill_stream
        fork = torch.cuda.Event()
        fork.record(stream)
        fill.wait_event(fork)
        # K2 waits only for the counts; the union / layer fills (160 MB at cfg3) keep
        # running under K2 and are joined before the first epilogue
        with torch.cuda.stream(fill):
            zero = lambda t: _lib.check(_lib.lib().gc_fill_zero(  # noqa: E731  (memset nodes)
                ctypes.c_void_p(t.data_ptr()), t.numel() * t.element_size(), ctypes.c_void_p(fill.cuda_stream)),
                "gc_fill_zero")
            zero(self.counts)
            join = torch.cuda.Event()
            join.record(fill)
            if self.peer is None:
                zero(u)
            if self.layers is not None:
                zero(self.layers)
            if self.utile is not None:
                zero(self.utile[buf])
            join_out = torch.cuda.Event()
            join_out.record(fill)
        if with_update:
            launch_belief_update(self.btab, self.d_hyp_off, self.d_beta64, self.d_goal64, self.d_obs,
                                 self.d_fallback, self.d_logw, self.d_logw, self.d_status, cfg.obs_dt,
                                 math.inf, 1, H, stream=stream)
        stream.wait_event(join)
        bounds = self.chunk_bounds(chunks) if chunks > 1 else self.window_bounds()
        if self.counts_reduce is not None and len(bounds) > 1:
            raise NotImplementedError("particle sharding runs the horizon in one chunk")
        if len(bounds) > 1:
            self._ensure_state()
        a = _lib.PredictArgs()
        a.n_humans, a.n, a.steps, a.rng_mode = H, self.n_local, cfg.steps, MODES[cfg.mode]
        a.p_offset = self.p_offset
        a.hist_path = _lib.GC_HIST_SMEM if cfg.hist_path == "smem" else _lib.GC_HIST_GLOBAL
        a.ref_exact_only = 0 if cfg.ref_filter else 1
        a.assume_qg = self._assume_qg
        a.grid_w, a.grid_h = self.spec.width, self.spec.height
        a.origin_x32 = float(np.float32(self.spec.origin[0]))
        a.origin_y32 = float(np.float32(self.spec.origin[1]))
        a.res32 = float(np.float32(self.spec.resolution))
        a.d_start_xy, a.d_hyp_off = self.d_start.data_ptr(), self.d_hyp_off.data_ptr()
        a.d_beta32, a.d_goal32 = self.d_beta32.data_ptr(), self.d_goal32.data_ptr()
        a.d_cdf, a.d_log_w = None, self.d_logw.data_ptr()
        a.d_seed, a.d_prefix, a.d_prefix_len = self.d_seed.data_ptr(), self.d_prefix.data_ptr(), self.d_plen.data_ptr()
        a.d_stream_id = self.d_sid.data_ptr()
        a.h_tables, a.n_tables, a.d_table_id = self._tarr, 2, self.d_tid.data_ptr()
        a.d_step_r, a.d_step_off = geo.d_step_r.data_ptr(), geo.d_step_off.data_ptr()
        a.human_stride, a.max_win_cells = geo.human_stride, geo.max_win_cells
        a.d_counts, a.d_error = self.counts.data_ptr(), self.d_err.data_ptr()
        if len(bounds) > 1:
            a.d_state_xy, a.d_state_hyp = self.state_xy.data_ptr(), self.state_hyp.data_ptr()
        e = _lib.EpilogueArgs()
        e.n_humans, e.n, e.steps = H, cfg.n, cfg.steps
        e.grid_w, e.grid_h, e.radius = self.spec.width, self.spec.height, geo.radius
        e.d_kernel, e.d_zx, e.d_zy = geo.d_kernel.data_ptr(), geo.d_zx.data_ptr(), geo.d_zy.data_ptr()
        e.origin_x32, e.origin_y32, e.res32 = a.origin_x32, a.origin_y32, a.res32
        e.n_tiles, e.d_start_xy = geo.n_tiles, self.d_start.data_ptr()
        e.d_step_r, e.d_step_off, e.human_stride = geo.d_step_r.data_ptr(), geo.d_step_off.data_ptr(), geo.human_stride
        e.d_tiles, e.d_counts = geo.d_tiles.data_ptr(), self.counts.data_ptr()
        if self.layers is not None:
            e.d_layers64 = self.layers.data_ptr()
        ordered = cfg.union_mode == "independent"
        if self.peer is not None:  # K3 writes the owner's fused grid over peer memory
            if d2h is not None:
                raise ValueError("with a peer union the owner copies the fused grid after PeerUnion.barrier()")
            if self.peer.dtype == torch.float32:
                e.d_union32 = self.peer.ptr(buf)
            else:
                e.d_union64 = self.peer.ptr(buf)
            if self.utile is not None:  # this rank's nonzero tiles (OR-reduced to the owner for publish)
                e.d_union_tile_flags = self.utile[buf].data_ptr()
        elif not ordered:  # max union by atomicMax inside K3
            if u.dtype == torch.float32:
                e.d_union32 = u.data_ptr()
            else:
                e.d_union64 = u.data_ptr()
            e.time_union = int(cfg.time_union)
            if self.utile is not None:
                e.d_union_tile_flags = self.utile[buf].data_ptr()
        tiles = d2h is not None and self.utile is not None
        if tiles:
            pa = self._publish_args(buf, u, d2h)
        for ci, (t0, t1) in enumerate(bounds):
            a.t_begin, a.t_end = (t0, t1) if len(bounds) > 1 else (0, 0)
            a.max_win_cells = int(geo.win_cells[t1 - 2])  # this launch's largest window
            if events is not None and ci == 0:
                events[0].record(stream)
            _lib.check(_lib.lib().gc_predict(ctypes.byref(a), sh), "gc_predict")
            if events is not None and ci == len(bounds) - 1:
                events[1].record(stream)
            if self.counts_reduce is not None:
                self.counts_reduce(self.counts)  # e.g. NCCL all-reduce(sum) over the shards
            if ci == 0:
                stream.wait_event(join_out)  # output grids zeroed before K3 writes them
            if len(bounds) > 1:
                e.tile_begin, e.tile_end = int(geo.tile_start[t0 - 1]), int(geo.tile_start[t1 - 1])
                e.t_begin, e.t_end = t0 - 1, t1 - 1
            _lib.check(_lib.lib().gc_grid_epilogue(ctypes.byref(e), sh), "gc_grid_epilogue")
            if ordered:
                # ordered merge of the per-human float64 layers of this chunk
                L0, L1 = t0 - 1, t1 - 1
                hw = self.spec.width * self.spec.height
                mode = _lib.GC_UNION_MISS if cfg.union_partial else _lib.GC_UNION_INDEPENDENT
                _lib.check(_lib.lib().gc_union_layers(
                    ctypes.c_void_p(self.layers[0, L0].data_ptr()), 8, H, cfg.steps * hw, (L1 - L0) * hw, mode,
                    ctypes.c_void_p(u[L0].data_ptr()), u.element_size(), sh), "gc_union_layers")
                if cfg.time_union and not cfg.union_partial:
                    _lib.check(_lib.lib().gc_time_union(ctypes.c_void_p(u.data_ptr()), u.element_size(), L0, L1,
                                                        hw, sh), "gc_time_union")
            if self.blocked is not None:
                L0, L1 = t0 - 1, t1 - 1
                _lib.check(_lib.lib().gc_collision_field(
                    ctypes.c_void_p(u[L0:L1].data_ptr()), u.element_size(), L1 - L0, self.spec.width,
                    self.spec.height, self._disc.ctypes.data_as(ctypes.c_void_p), len(self._disc),
                    float(cfg.collision_threshold), None,
                    ctypes.c_void_p(self.blocked[buf][L0:L1].data_ptr()), sh), "gc_collision_field")
            if d2h is not None:
                ev = torch.cuda.Event()
                ev.record(stream)
                copy_stream.wait_event(ev)
                with torch.cuda.stream(copy_stream):
                    if tiles:  # tile-sparse: kernel stores of the changed tiles into the host stack
                        pa.t_begin, pa.t_end = t0 - 1, t1 - 1
                        _lib.check(_lib.lib().gc_publish_tiles(ctypes.byref(pa), ctypes.c_void_p(
                            copy_stream.cuda_stream)), "gc_publish_tiles")
                    else:
                        d2h[t0 - 1:t1 - 1].copy_(u[t0 - 1:t1 - 1], non_blocking=True)
        if events is not None:
            events[2].record(stream)
        if d2h is not None:
            stream.wait_stream(copy_stream)  # the cycle ends when its layers are on the host

    def _publish_args(self, buf, union, d2h, time_or=None):
        if d2h.dtype != union.dtype or tuple(d2h.shape) != tuple(union.shape) or not d2h.is_pinned():
            raise ValueError("d2h must be a pinned host tensor shaped and typed like the union")
        hf = self._hflags.get(d2h.data_ptr())
        if hf is None:  # a new host stack: zero it once, then only changed tiles move
            d2h.zero_()
            hf = torch.zeros(self.tile_grid, dtype=torch.uint8, device=self.dev)
            self._hflags[d2h.data_ptr()] = hf
        pa = _lib.PublishArgs()
        pa.steps, pa.grid_w, pa.grid_h = self.cfg.steps, self.spec.width, self.spec.height
        pa.dtype_bytes = union.element_size()
        pa.time_or = int(self.cfg.time_union if time_or is None else time_or)
        pa.d_union, pa.d_tile_flags = union.data_ptr(), self.utile[buf].data_ptr()
        pa.d_host_flags, pa.h_dst = hf.data_ptr(), d2h.data_ptr()
        return pa

    def publish(self, buf: int, d2h, union=None, stream=None, time_or=None):
        """Tile-sparse copy of a union (default: this engine's union ``buf``; e.g. the fused
        grid after ``fused_reduce`` with the tile flags OR-reduced too) into the pinned host
        stack ``d2h`` on ``stream`` (gc_publish_tiles): afterwards ``d2h`` equals the union."""
        if self.utile is None:
            raise RuntimeError("publish() needs EngineConfig(d2h_mode='tiles', union_mode='max')")
        union = self.unions[buf] if union is None else union
        s = stream or torch.cuda.current_stream(self.dev)
        pa = self._publish_args(buf, union, d2h, time_or)
        _lib.check(_lib.lib().gc_publish_tiles(ctypes.byref(pa), ctypes.c_void_p(s.cuda_stream)), "gc_publish_tiles")

    def run_cycle(self, buf: int = 0, with_h2d: bool = True, with_update: bool = True, stream=None,
                  events=None, chunks: int = 1, d2h=None, copy_stream=None):
        """Eager (uncaptured) cycle on ``stream``; ``events`` = 3 CUDA events recorded
        before K2, after K2 and after K3 (kernel timing on the launching stream)."""
        s = stream or torch.cuda.current_stream()
        with_update = with_update and not self._skip_update[buf]
        with torch.cuda.stream(s):
            if with_h2d:
                self.d_in.copy_(self.h_ins[buf], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s)
                self._h2d_done[buf] = ev
            self._launch(buf, with_update, s, events, chunks=chunks, d2h=d2h, copy_stream=copy_stream)
        return self.unions[buf]

    def capture(self, buf: int = 0, with_h2d: bool = True, with_update: bool = True, chunks: int = 1,
                d2h=None, events=None):
        """Capture one cycle into a CUDA graph (replay with ``replay``).  With ``d2h`` (a
        pinned host tensor shaped like the union) the chunked D2H copies are part of the
        graph, on a forked copy stream.  ``events``: 3 CUDA events created with
        ``external=True`` (event-record nodes) recorded before K2, after K2 and after K3
        inside the graph, so every replay times its kernels on the graph's own clock."""
        if with_update and self._skip_update[buf]:
            raise RuntimeError("capture(): prime() the engine first (a graph always runs the belief update)")
        key = (buf, with_h2d, with_update, chunks, None if d2h is None else d2h.data_ptr(),
               None if events is None else id(events))
        if key in self.graphs:
            return self.graphs[key][0]
        # stream priorities are captured into the kernel nodes: the cycle's kernels run at high
        # priority and the chunk publications at low priority, so a publication CTA only takes
        # an SM slot no K2 CTA is waiting for (the last wave's idle slots) instead of delaying
        # K2 CTAs -- and with them the chunk's end -- by its whole PCIe-bound duration
        s = torch.cuda.Stream(priority=-1)
        cp = torch.cuda.Stream(priority=0) if d2h is not None else None
        s.wait_stream(torch.cuda.current_stream())
        # warm the library once outside capture (function attributes, lazy loading)
        self.run_cycle(buf, with_h2d, with_update, stream=s, chunks=chunks, d2h=d2h, copy_stream=cp)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            if with_h2d:
                self.d_in.copy_(self.h_ins[buf], non_blocking=True)
            self._launch(buf, with_update, s, events=events, chunks=chunks, d2h=d2h, copy_stream=cp)
        self.graphs[key] = (g, cp, events)  # keep the copy stream / events alive with the graph
        return g

    def _belief_stream(self):
        return self._stream if self._stream is not None else torch.cuda.current_stream(self.dev)

    def posterior(self, i: int) -> np.ndarray:
        """Human i's device posterior, read after the cycles already issued on the engine's stream."""
        a, b = self.hyp_off[i], self.hyp_off[i + 1]
        s = self._belief_stream()
        with torch.cuda.stream(s):
            out = self.d_logw[a:b].to("cpu", non_blocking=True)
        s.synchronize()
        return out.numpy()

    def reset_belief(self, i: int):
        """Uniform belief for human i (goal departure, sim.py:563-568; belief.py:120-123),
        ordered on the engine's launch stream after the cycles already issued there."""
        a, b = int(self.hyp_off[i]), int(self.hyp_off[i + 1])
        with torch.cuda.stream(self._belief_stream()):
            self.d_logw[a:b] = -math.log(b - a)

    def check_errors(self):
        """Raise for K2's sticky device status bits (and clear them)."""
        s = self._belief_stream()
        s.synchronize()
        word = int(self.d_err.item())
        if word:
            self.d_err.zero_()
            torch.cuda.synchronize(self.dev)
            _lib.check_error_word(word, "gc_predict")


def union_tiles(union: torch.Tensor, ids: torch.Tensor, packed: torch.Tensor, unpack: bool):
    """gc_union_tiles: gather (unpack=False) / scatter (unpack=True) the 32 x 32 tiles ``ids``
    (int32, the union-tile flag layout) of a (T, H, W) CUDA union to / from ``packed``
    (len(ids), 32, 32) on the current stream."""
    if union.device.type != "cuda":
        raise RuntimeError("union_tiles needs CUDA tensors (no CPU path)")
    T, H, W = union.shape
    sh = ctypes.c_void_p(torch.cuda.current_stream(union.device).cuda_stream)
    _lib.check(_lib.lib().gc_union_tiles(ctypes.c_void_p(union.data_ptr()), union.element_size(), T, W, H,
                                         ctypes.c_void_p(ids.data_ptr()), int(ids.numel()),
                                         ctypes.c_void_p(packed.data_ptr()), int(bool(unpack)), sh),
               "gc_union_tiles")


def sparse_max_reduce(union: torch.Tensor, tiles: torch.Tensor, group=None, dst: Optional[int] = None,
                      tile_op=union_tiles):
    """Max-merge per-rank (T, H, W) unions over the process group moving only nonzero tiles.

    ``tiles`` holds this rank's union-tile flags (K3's ``d_union_tile_flags``; a tile no
    rank flagged is zero on every rank).  The flags are OR-ed over the ranks (all-reduce max
    of bytes -- afterwards they describe the fused grid, as the publication needs), every
    rank packs the same tiles into a (count, 32, 32) buffer, the packed buffers are
    max-reduced (NCCL) and the receiving rank(s) scatter them back: the union equals the
    dense max-reduce bit for bit, from ~count/all of the bytes (bench scene: 8.5 % of the
    320 MB float64 grid).  One host sync per call (the tile count sizes the collective).
    ``tile_op`` is the gather/scatter (the CUDA kernel; the CPU multi-rank tests pass a
    torch restatement)."""
    import torch.distributed as dist
    dist.all_reduce(tiles, op=dist.ReduceOp.MAX, group=group)
    ids = torch.nonzero(tiles.reshape(-1)).reshape(-1).to(torch.int32)
    n = int(ids.numel())
    if n == 0:
        return union
    packed = torch.empty((n, 32, 32), dtype=union.dtype, device=union.device)
    tile_op(union, ids, packed, False)
    if dst is None:
        dist.all_reduce(packed, op=dist.ReduceOp.MAX, group=group)
    else:
        dist.reduce(packed, dst=dst, op=dist.ReduceOp.MAX, group=group)
    if dst is None or dist.get_rank(group) == dst:
        tile_op(union, ids, packed, True)
    return union


def fused_reduce(union: torch.Tensor, group=None, dst: Optional[int] = None, mode: str = "max",
                 time_union: bool = False, finish: bool = True, tiles: Optional[torch.Tensor] = None):
    """Merge per-rank unions into one fused grid over NCCL (torch.distributed); all_reduce
    when dst is None.  mode "max": max reduction of the per-rank max unions -- with
    ``tiles`` (the union-tile flags) only the nonzero tiles move (``sparse_max_reduce``).
    mode "independent": the ranks hold prod(1 - p) partials (EngineConfig(union_partial=True));
    they are multiplied (ReduceOp.PRODUCT) and, when ``finish``, complemented on the
    receiving rank(s) to 1 - prod (+ the conservative time union when ``time_union``).
    The cross-rank product is taken in NCCL's order, so the independent fused grid equals
    the single-GPU one up to float rounding (max is exact)."""
    import torch.distributed as dist
    if mode == "max" and tiles is not None:
        if time_union:
            raise ValueError("the sparse reduce needs flags that cover the union: the time union "
                             "spreads values past the flagged layers (reduce densely)")
        return sparse_max_reduce(union, tiles, group=group, dst=dst)
    if mode == "max":
        if dst is None:
            dist.all_reduce(union, op=dist.ReduceOp.MAX, group=group)
        else:
            dist.reduce(union, dst=dst, op=dist.ReduceOp.MAX, group=group)
        return union
    if mode != "independent":
        raise ValueError(f"unknown union mode {mode!r}")
    if dst is None:
        dist.all_reduce(union, op=dist.ReduceOp.PRODUCT, group=group)
    else:
        dist.reduce(union, dst=dst, op=dist.ReduceOp.PRODUCT, group=group)
    if finish and (dst is None or dist.get_rank() == dst):
        complement_layers(union, time_union=time_union)
    return union


def complement_layers(union: torch.Tensor, time_union: bool = False) -> torch.Tensor:
    """In place 1 - miss (+ time union) of a (T, H, W) miss-product stack on the GPU
    (gc_union_layers GC_UNION_COMPLEMENT, gc_time_union)."""
    if union.device.type != "cuda":
        raise RuntimeError("complement_layers needs a CUDA tensor (no CPU path)")
    sh = ctypes.c_void_p(torch.cuda.current_stream(union.device).cuda_stream)
    hw = union.shape[-1] * union.shape[-2]
    _lib.check(_lib.lib().gc_union_layers(ctypes.c_void_p(union.data_ptr()), union.element_size(), 1, 0,
                                          union.numel(), _lib.GC_UNION_COMPLEMENT, ctypes.c_void_p(union.data_ptr()),
                                          union.element_size(), sh), "gc_union_layers")
    if time_union:
        _lib.check(_lib.lib().gc_time_union(ctypes.c_void_p(union.data_ptr()), union.element_size(), 0,
                                            union.shape[0], hw, sh), "gc_time_union")
    return union
