"""Particle occupancy prediction on the GPU (reference prediction.py:1-414).

Public names and semantics follow the reference; the work runs in three kernels:
K2 ``gc_predict`` (hypothesis draw + whole-horizon propagation in registers fused with
the per-step histogram), K3 ``gc_grid_epilogue`` (counts/n, smoothing, union) and, for
the standalone helpers, ``gc_propagate_step`` / ``gc_sample_hypotheses``.

``PredictionConfig.mode``:
  "reference"  (default) regenerates the reference's own Philox streams in-register and
               runs its float32 arithmetic op for op: for the same inputs and seed the
               per-step counts -- hence every unsmoothed layer -- are bit-identical to
               gridcast.predict; smoothed layers agree to <= 1e-15.
  "production" Philox4x32 + the factorised exact-in-distribution sampler (fast path);
               layers agree with the reference in distribution (TV bound).
"""

from __future__ import annotations

import ctypes
from collections import OrderedDict
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .agents import ControlSet, HumanState, QFunction
from .belief import HypothesisSpace, JointBelief
from .device import device, stream_handle, upload_packed
from .occupancy import GridSpec, OccupancyGrid
from .tables import ActionTables, Geometry, assume_qg, hypothesis_arrays

CHUNK = 1024  # particles per reference random stream (prediction.py:33)
MODES = {"reference": _lib.GC_RNG_REFERENCE, "production": _lib.GC_RNG_PRODUCTION}
_MASK64 = (1 << 64) - 1


class EnumerationCapExceeded(ValueError):
    """Instance too large for exact enumeration."""


@dataclass(frozen=True)
class ParticleBatch:
    xy: np.ndarray
    hypothesis_idx: np.ndarray

    def __post_init__(self):
        xy = np.asarray(self.xy, dtype=np.float32)
        hyp = np.asarray(self.hypothesis_idx, dtype=np.int32)
        if xy.ndim != 2 or xy.shape[1] != 2 or xy.shape[0] == 0:
            raise ValueError("particle positions must form a nonempty (n, 2) array")
        if hyp.shape != (xy.shape[0],):
            raise ValueError("one hypothesis index per particle required")
        if (hyp < 0).any():
            raise ValueError("hypothesis indices must be nonnegative")
        object.__setattr__(self, "xy", xy)
        object.__setattr__(self, "hypothesis_idx", hyp)

    @property
    def n(self) -> int:
        return self.xy.shape[0]

    @classmethod
    def duplicated(cls, z: HumanState, hypothesis_idx) -> "ParticleBatch":
        n = len(hypothesis_idx)
        return cls(np.tile(np.array([z.x, z.y], dtype=np.float32), (n, 1)), hypothesis_idx)


@dataclass(frozen=True)
class PredictionConfig:
    n: int = 8192
    steps: int = 6
    dt: float = 0.5
    smoothing_sigma: float = 0.1
    seed: int = 0
    mode: str = "reference"

    def __post_init__(self):
        if self.n < 1 or self.steps < 1:
            raise ValueError("need n >= 1 and steps >= 1")
        if self.dt <= 0:
            raise ValueError("dt must be > 0")
        if self.smoothing_sigma < 0:
            raise ValueError("smoothing sigma must be >= 0")
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {sorted(MODES)}")


class PredictionStack:
    """T occupancy layers; layer k is p(z at base_time + (k+1) dt).

    Device-resident: ``layers_device`` is the (T, H, W) float64 CUDA tensor written by
    the epilogue; ``layers`` materialises a read-only host copy on first access (the
    reference returns host arrays, prediction.py:98-106)."""

    def __init__(self, spec: GridSpec, layers, base_time: float, dt: float):
        if dt <= 0:
            raise ValueError("dt must be > 0")
        self.spec, self.base_time, self.dt = spec, float(base_time), float(dt)
        if isinstance(layers, torch.Tensor):
            if layers.dim() != 3 or tuple(layers.shape[1:]) != spec.shape:
                raise ValueError("layers must be (T, height, width) matching the spec")
            self._dev, self._host = layers, None
        else:
            arr = np.asarray(layers, dtype=float)
            if arr.ndim != 3 or arr.shape[1:] != spec.shape:
                raise ValueError("layers must be (T, height, width) matching the spec")
            arr = arr.copy()
            arr.setflags(write=False)
            self._dev, self._host = None, arr

    @property
    def layers(self) -> np.ndarray:
        if self._host is None:
            arr = self._dev.cpu().numpy()
            arr.setflags(write=False)
            self._host = arr
        return self._host

    @property
    def layers_device(self) -> torch.Tensor:
        if self._dev is None:
            import warnings
            with warnings.catch_warnings():  # a host->device copy never writes the read-only array
                warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
                self._dev = torch.as_tensor(self._host, device=device())
        return self._dev

    @property
    def steps(self) -> int:
        return (self._dev if self._dev is not None else self._host).shape[0]

    def grid(self, layer: int) -> OccupancyGrid:
        return OccupancyGrid(self.spec, self.layers[layer])

    def grids(self) -> list:
        return [self.grid(k) for k in range(self.steps)]

    def layer_index_for(self, time: float) -> int:
        k = int(round((time - self.base_time) / self.dt)) - 1
        return min(max(k, 0), self.steps - 1)


# ---- caches of device tables ----------------------------------------------------------
_ACTION_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()
_GEOM_CACHE: "OrderedDict[tuple, Geometry]" = OrderedDict()


def action_tables(control_set, q, dt, dev) -> ActionTables:
    key = (id(control_set), id(q), float(dt), str(dev))
    hit = _ACTION_CACHE.get(key)
    if hit is not None and hit[0] is control_set and hit[1] is q:
        return hit[2]
    t = ActionTables(control_set, q, dt, dev)
    _ACTION_CACHE[key] = (control_set, q, t)
    while len(_ACTION_CACHE) > 64:
        _ACTION_CACHE.popitem(last=False)
    return t


def geometry(spec: GridSpec, steps: int, max_step: float, sigma: float, dev) -> Geometry:
    key = (spec.width, spec.height, spec.resolution, spec.origin, steps, max_step, sigma, str(dev))
    g = _GEOM_CACHE.get(key)
    if g is None:
        g = Geometry(spec, steps, max_step, sigma, dev)
        _GEOM_CACHE[key] = g
        while len(_GEOM_CACHE) > 32:
            _GEOM_CACHE.popitem(last=False)
    return g


def host_cdf(log_weights) -> np.ndarray:
    """cdf exactly as sample_hypotheses builds it (prediction.py:128-129)."""
    cdf = np.cumsum(np.exp(np.asarray(log_weights, dtype=float)))
    cdf[-1] = 1.0
    return cdf


def _prefix_words(prefix) -> list:
    words = [int(p) & 0xFFFFFFFF for p in prefix]
    if len(words) > 4:
        raise NotImplementedError("random-stream prefixes of at most 4 elements are supported")
    return words


@dataclass
class HumanJob:
    """One human of a batched predict: start state, belief, hypotheses, stream key."""

    z0: HumanState
    log_weights: np.ndarray
    beta_of: np.ndarray
    goal_xy_of: np.ndarray
    seed: int
    prefix: tuple = ()
    table: int = 0


def run_predict(jobs: Sequence[HumanJob], tables: Sequence[ActionTables], n: int, steps: int, dt: float,
                sigma: float, spec: GridSpec, mode: str, per_human_layers: bool = True,
                union64: bool = False, union32: bool = False, time_union: bool = False,
                uniforms: Optional[torch.Tensor] = None, hyp_in: Optional[torch.Tensor] = None,
                hyp_u: Optional[torch.Tensor] = None, want_hyp: bool = False, want_xy: bool = False,
                stream=None, union_mode: str = "max", hist_path: str = "global",
                ref_exact_only: bool = False, ref_fallbacks: Optional[torch.Tensor] = None):
    """Batched K2 + K3 launch; returns a dict of device tensors.  union_mode "max" merges
    the humans by atomicMax inside K3; "independent" (1 - prod(1 - p), occupancy.py:180-184)
    merges the per-human float64 layers afterwards in human order (gc_union_layers).

    ``uniforms`` (humans, steps, n) float32 and ``hyp_u`` (humans, n) float64 select
    GC_RNG_UNIFORMS: the reference arithmetic driven by caller-supplied draws (e.g. the
    reference's own rng.stream draws, prediction.py:128-131, :186-192).

    ``ref_exact_only`` runs numpy's exp for every reference-mode particle-step instead of
    the MUFU filter with exact fallback (bit-identical results; A/B); ``ref_fallbacks`` (a
    (1,) int64 device tensor) accumulates the particle-steps that took the exact path."""
    if hyp_u is not None and uniforms is None:
        raise ValueError("hyp_u needs uniforms (GC_RNG_UNIFORMS)")
    if uniforms is not None:
        if tuple(uniforms.shape) != (len(jobs), steps, n) or uniforms.dtype != torch.float32:
            raise ValueError("uniforms must be a (humans, steps, n) float32 device tensor")
        if hyp_u is not None and (tuple(hyp_u.shape) != (len(jobs), n) or hyp_u.dtype != torch.float64):
            raise ValueError("hyp_u must be a (humans, n) float64 device tensor")
    if union_mode not in ("max", "independent"):
        raise ValueError(f"unknown union mode {union_mode!r}")
    dev = device()
    H = len(jobs)
    max_step = max(t.max_step for t in tables)
    geo = geometry(spec, steps, max_step, float(sigma), dev)
    hyp_off = np.zeros(H + 1, dtype=np.int32)
    for i, j in enumerate(jobs):
        if len(j.beta_of) > _lib.GC_MAX_HYPOTHESES:
            raise NotImplementedError(f"at most {_lib.GC_MAX_HYPOTHESES} hypotheses per human")
        hyp_off[i + 1] = hyp_off[i] + len(j.beta_of)
    pre = np.zeros((H, 4), dtype=np.uint32)
    plen = np.zeros(H, dtype=np.int32)
    for i, j in enumerate(jobs):
        w = _prefix_words(j.prefix)
        pre[i, :len(w)] = w
        plen[i] = len(w)
    # every per-call input in ONE host-to-device copy (the small per-array uploads cost a
    # copy each -- most of a small predict's latency)
    (d_start, d_hyp_off, d_beta, d_goal, d_cdf, d_seed, d_pre, d_plen, d_tid, err) = upload_packed(dev, [
        np.array([[j.z0.x, j.z0.y] for j in jobs], dtype=np.float32),
        hyp_off,
        np.concatenate([j.beta_of for j in jobs]).astype(np.float32),
        np.concatenate([j.goal_xy_of for j in jobs]).astype(np.float32),
        np.concatenate([host_cdf(j.log_weights) for j in jobs]).astype(np.float64),
        np.array([int(j.seed) & _MASK64 for j in jobs], dtype=np.uint64),
        pre, plen,
        np.array([j.table for j in jobs], dtype=np.int32),
        np.zeros(1, dtype=np.int32),  # the device status word
    ])
    counts = torch.zeros(H * geo.human_stride, dtype=torch.int32, device=dev)
    out = {}
    if want_hyp:
        out["hyp"] = torch.empty((H, n), dtype=torch.int32, device=dev)
    if want_xy:
        out["xy"] = torch.empty((H, n, 2), dtype=torch.float32, device=dev)

    a = _lib.PredictArgs()
    a.n_humans, a.n, a.steps = H, n, steps
    a.rng_mode = _lib.GC_RNG_UNIFORMS if uniforms is not None else MODES[mode]
    a.grid_w, a.grid_h = spec.width, spec.height
    a.origin_x32 = float(np.float32(spec.origin[0]))
    a.origin_y32 = float(np.float32(spec.origin[1]))
    a.res32 = float(np.float32(spec.resolution))
    a.d_start_xy, a.d_hyp_off = d_start.data_ptr(), d_hyp_off.data_ptr()
    a.d_beta32, a.d_goal32, a.d_cdf, a.d_log_w = d_beta.data_ptr(), d_goal.data_ptr(), d_cdf.data_ptr(), None
    a.d_seed, a.d_prefix, a.d_prefix_len = d_seed.data_ptr(), d_pre.data_ptr(), d_plen.data_ptr()
    a.d_uniforms = uniforms.data_ptr() if uniforms is not None else None
    a.d_hyp_u = hyp_u.data_ptr() if hyp_u is not None else None
    a.d_hyp_in = hyp_in.data_ptr() if hyp_in is not None else None
    tarr = (_lib.ActionTable * len(tables))(*[t.struct for t in tables])
    a.h_tables, a.n_tables, a.d_table_id = tarr, len(tables), d_tid.data_ptr()
    a.d_step_r, a.d_step_off = geo.d_step_r.data_ptr(), geo.d_step_off.data_ptr()
    a.human_stride, a.max_win_cells = geo.human_stride, geo.max_win_cells
    a.d_counts = counts.data_ptr()
    a.d_hyp_out = out["hyp"].data_ptr() if want_hyp else None
    a.d_xy_out = out["xy"].data_ptr() if want_xy else None
    a.d_error = err.data_ptr()
    if hist_path not in ("global", "smem"):
        raise ValueError(f"unknown hist_path {hist_path!r}")
    a.hist_path = _lib.GC_HIST_SMEM if hist_path == "smem" else _lib.GC_HIST_GLOBAL
    a.ref_exact_only = int(bool(ref_exact_only))
    a.assume_qg = int(mode == "production" and uniforms is None and
                      assume_qg(tables, [j.beta_of for j in jobs]))
    if ref_fallbacks is not None:
        if ref_fallbacks.dtype != torch.int64 or ref_fallbacks.numel() < 1 or not ref_fallbacks.is_cuda:
            raise ValueError("ref_fallbacks must be a (1,) int64 device tensor")
        a.d_ref_fallbacks = ref_fallbacks.data_ptr()
    sh = stream_handle(stream)
    _lib.check(_lib.lib().gc_predict(ctypes.byref(a), sh), "gc_predict")

    e = _lib.EpilogueArgs()
    e.n_humans, e.n, e.steps = H, n, steps
    e.grid_w, e.grid_h, e.radius = spec.width, spec.height, geo.radius
    e.d_kernel, e.d_zx, e.d_zy = geo.d_kernel.data_ptr(), geo.d_zx.data_ptr(), geo.d_zy.data_ptr()
    e.origin_x32, e.origin_y32, e.res32 = a.origin_x32, a.origin_y32, a.res32
    e.n_tiles, e.d_start_xy = geo.n_tiles, d_start.data_ptr()
    e.d_step_r, e.d_step_off, e.human_stride = geo.d_step_r.data_ptr(), geo.d_step_off.data_ptr(), geo.human_stride
    e.d_tiles, e.d_counts = geo.d_tiles.data_ptr(), counts.data_ptr()
    ordered = union_mode == "independent" and (union64 or union32)
    if per_human_layers or ordered:
        out["layers"] = torch.zeros((H, steps, spec.height, spec.width), dtype=torch.float64, device=dev)
        e.d_layers64 = out["layers"].data_ptr()
    if union64:
        out["union64"] = torch.zeros((steps, spec.height, spec.width), dtype=torch.float64, device=dev)
        e.d_union64 = 0 if ordered else out["union64"].data_ptr()
    if union32:
        out["union32"] = torch.zeros((steps, spec.height, spec.width), dtype=torch.float32, device=dev)
        e.d_union32 = 0 if ordered else out["union32"].data_ptr()
    e.time_union = int(time_union and not ordered)
    _lib.check(_lib.lib().gc_grid_epilogue(ctypes.byref(e), sh), "gc_grid_epilogue")
    if ordered:
        cells = steps * spec.height * spec.width
        for key in ("union64", "union32"):
            if key in out:
                u = out[key]
                _lib.check(_lib.lib().gc_union_layers(
                    ctypes.c_void_p(out["layers"].data_ptr()), 8, H, cells, cells, _lib.GC_UNION_INDEPENDENT,
                    ctypes.c_void_p(u.data_ptr()), u.element_size(), sh), "gc_union_layers")
                if time_union:
                    _lib.check(_lib.lib().gc_time_union(ctypes.c_void_p(u.data_ptr()), u.element_size(), 0, steps,
                                                        spec.height * spec.width, sh), "gc_time_union")
        if not per_human_layers:
            del out["layers"]
    _lib.check_error_word(err.item(), "gc_predict")
    out["counts"] = counts
    out["geometry"] = geo
    return out


def _as_state(z_history) -> HumanState:
    if isinstance(z_history, HumanState) or (hasattr(z_history, "x") and hasattr(z_history, "y")):
        return z_history
    seq = list(z_history)
    if not seq:
        raise ValueError("empty state history")
    return seq[-1]


def sample_hypotheses(belief: JointBelief, n: int, seed: int, prefix: tuple = ()) -> np.ndarray:
    """n i.i.d. hypothesis indices drawn with the reference stream (prediction.py:124-131)."""
    if n < 1:
        raise ValueError("n must be >= 1")
    dev = device()
    cdf = torch.as_tensor(host_cdf(belief.log_weights), device=dev)
    out = torch.empty(n, dtype=torch.int32, device=dev)
    words = _prefix_words(prefix)
    arr = (ctypes.c_uint32 * max(1, len(words)))(*words)
    _lib.check(_lib.lib().gc_sample_hypotheses(ctypes.c_void_p(cdf.data_ptr()), len(cdf), n,
                                               int(seed) & _MASK64, arr, len(words),
                                               ctypes.c_void_p(out.data_ptr()), stream_handle()),
               "sample_hypotheses")
    return out.cpu().numpy()


def propagate_step(batch: ParticleBatch, control_set: ControlSet, q: QFunction, space: HypothesisSpace,
                   dt: float, seed: int, step: int = 0, workers: Optional[int] = None,
                   prefix: tuple = ()) -> ParticleBatch:
    """One reference-arithmetic step of an explicit batch (prediction.py:165-211)."""
    dev = device()
    tab = action_tables(control_set, q, dt, dev)
    beta_of, goal_of = hypothesis_arrays(space)
    if batch.hypothesis_idx.max() >= len(beta_of):
        raise ValueError("hypothesis index out of range for the space")
    xy = torch.as_tensor(batch.xy.copy(), device=dev)
    hyp = torch.as_tensor(batch.hypothesis_idx, device=dev)
    db = torch.as_tensor(beta_of.astype(np.float32), device=dev)
    dg = torch.as_tensor(np.array(goal_of, dtype=np.float32, order="C"), device=dev)
    words = _prefix_words(prefix)
    arr = (ctypes.c_uint32 * max(1, len(words)))(*words)
    _lib.check(_lib.lib().gc_propagate_step(
        ctypes.c_void_p(xy.data_ptr()), ctypes.c_void_p(hyp.data_ptr()), batch.n,
        ctypes.c_void_p(db.data_ptr()), ctypes.c_void_p(dg.data_ptr()), len(beta_of),
        ctypes.byref(tab.struct), None, int(seed) & _MASK64, arr, len(words), int(step),
        stream_handle()), "propagate_step")
    return ParticleBatch(xy.cpu().numpy(), batch.hypothesis_idx)


def predict(z_history, belief: JointBelief, cfg: PredictionConfig, control_set: ControlSet, q: QFunction,
            space: HypothesisSpace, grid_spec: GridSpec, workers: Optional[int] = None,
            base_time: float = 0.0, prefix: tuple = ()) -> PredictionStack:
    """Monte-Carlo occupancy prediction over cfg.steps steps (Alg. 1; prediction.py:223-255)."""
    z0 = _as_state(z_history)
    if len(belief) != space.size:
        raise ValueError("belief size does not match hypothesis space")
    dev = device()
    tab = action_tables(control_set, q, cfg.dt, dev)
    beta_of, goal_of = hypothesis_arrays(space)
    job = HumanJob(z0, belief.log_weights, beta_of, goal_of, cfg.seed, tuple(prefix), 0)
    out = run_predict([job], [tab], cfg.n, cfg.steps, cfg.dt, cfg.smoothing_sigma, grid_spec,
                      getattr(cfg, "mode", "reference"))
    return PredictionStack(grid_spec, out["layers"][0], base_time, cfg.dt)


def predict_naive(z_history, belief: JointBelief, cfg: PredictionConfig, control_set: ControlSet, q: QFunction,
                  space: HypothesisSpace, grid_spec: GridSpec, base_time: float = 0.0) -> PredictionStack:
    """The reference's plain per-particle loop (prediction.py:258-300) on the GPU
    (gc_predict_naive): float64 positions, the full q.table row of each particle's
    hypothesis, the same chunk-keyed streams drawn in float64, float64 cells.  Its layers
    equal the reference's (a decision could differ only if a uniform lands within an ulp
    of a cdf entry, the float64 exp being CUDA's rather than numpy's)."""
    from .agents import EmptyControlSetError
    from .tables import f64_tables, recognise_q
    z0 = _as_state(z_history)
    if len(belief) != space.size:
        raise ValueError("belief size does not match hypothesis space")
    lq = recognise_q(q)
    if lq is None:
        raise NotImplementedError("predict_naive on the B200 implements q_goal_progress and q_default "
                                  "(and their stationary-masked variants)")
    v, th = np.asarray(control_set.v, float), np.asarray(control_set.theta, float)
    mask = q.action_mask(control_set)
    keep = np.arange(len(v)) if mask is None else np.flatnonzero(~mask)
    if len(keep) == 0:
        raise EmptyControlSetError("all actions are masked")
    dev = device()
    up = lambda a_, t_: torch.as_tensor(np.array(a_, dtype=t_, order="C"), device=dev)  # noqa: E731
    sx, sy, at, pen = f64_tables(v, th, lq)
    disp = control_set.displacements(cfg.dt)
    beta_of, goal_of = hypothesis_arrays(space)
    hyp = up(sample_hypotheses(belief, cfg.n, cfg.seed), np.int32)
    bufs = dict(beta=up(beta_of, np.float64), goal=up(goal_of, np.float64), keep=up(keep, np.int32),
                sx=up(sx, np.float64), sy=up(sy, np.float64), at=up(at, np.float64), pen=up(pen, np.float64),
                dx=up(disp[:, 0], np.float64), dy=up(disp[:, 1], np.float64))
    T, H, W = cfg.steps, grid_spec.height, grid_spec.width
    counts = torch.zeros(T * H * W, dtype=torch.int32, device=dev)
    a = _lib.NaiveArgs()
    a.n, a.steps, a.n_hyp, a.m_keep = cfg.n, T, len(beta_of), len(keep)
    a.q_kind = _lib.GC_Q_DEFAULT if lq.family == "default" else _lib.GC_Q_GOAL_PROGRESS_FULL
    a.grid_w, a.grid_h, a.prefix_len, a.seed = W, H, 0, int(cfg.seed) & _MASK64
    a.start_x, a.start_y = float(z0.x), float(z0.y)
    a.origin_x, a.origin_y, a.res = grid_spec.origin[0], grid_spec.origin[1], grid_spec.resolution
    a.d_hyp, a.d_beta, a.d_goal, a.d_keep = (hyp.data_ptr(), bufs["beta"].data_ptr(), bufs["goal"].data_ptr(),
                                             bufs["keep"].data_ptr())
    a.d_sx, a.d_sy, a.d_at, a.d_pen = (bufs["sx"].data_ptr(), bufs["sy"].data_ptr(), bufs["at"].data_ptr(),
                                       bufs["pen"].data_ptr())
    a.d_dispx, a.d_dispy, a.d_counts = bufs["dx"].data_ptr(), bufs["dy"].data_ptr(), counts.data_ptr()
    _lib.check(_lib.lib().gc_predict_naive(ctypes.byref(a), stream_handle()), "predict_naive")
    # emplace_counts(...) / n as an elementwise IEEE division (a Python-scalar divisor would
    # let torch multiply by the reciprocal instead, which is not numpy's rounding)
    layers = counts.view(T, H, W).to(torch.float64)
    layers = layers / torch.full_like(layers, float(cfg.n))
    if cfg.smoothing_sigma > 0:
        from .occupancy import smooth_layers_device
        layers = smooth_layers_device(layers, grid_spec, cfg.smoothing_sigma)
    torch.cuda.current_stream().synchronize()
    return PredictionStack(grid_spec, layers, base_time, cfg.dt)


def predict_multi(humans: Sequence[tuple], cfg: PredictionConfig, control_set: ControlSet, q: QFunction,
                  space: HypothesisSpace, grid_spec: GridSpec, workers: Optional[int] = None,
                  base_time: float = 0.0, union_mode: str = "max") -> PredictionStack:
    """Per-human prediction merged layer-wise by pointwise max (prediction.py:380-409):
    one batched launch, union by the epilogue's atomicMax.  ``union_mode="independent"``
    (an extension; occupancy.union's 1 - prod(1 - p), occupancy.py:180-184) merges the
    per-human layers in order instead."""
    if not humans:
        raise ValueError("need at least one human")
    dev = device()
    tab = action_tables(control_set, q, cfg.dt, dev)
    beta_of, goal_of = hypothesis_arrays(space)
    jobs = []
    for hist, b in humans:
        if len(b) != space.size:
            raise ValueError("belief size does not match hypothesis space")
        jobs.append(HumanJob(_as_state(hist), b.log_weights, beta_of, goal_of, cfg.seed, (), 0))
    out = run_predict(jobs, [tab], cfg.n, cfg.steps, cfg.dt, cfg.smoothing_sigma, grid_spec,
                      getattr(cfg, "mode", "reference"), per_human_layers=False, union64=True,
                      union_mode=union_mode)
    return PredictionStack(grid_spec, out["union64"], base_time, cfg.dt)


def exact_predict(z_t: HumanState, belief: JointBelief, steps: int, dt: float, control_set: ControlSet,
                  q: QFunction, space: HypothesisSpace, grid_spec: GridSpec, max_table: Optional[int] = 2_000_000,
                  base_time: float = 0.0) -> PredictionStack:
    """Exact layers by enumerating the bootstrapped process (prediction.py:303-377), on the
    GPU (gc_exact_predict).  Same cap semantics as the reference (EnumerationCapExceeded
    above ``max_table`` entries, default 2e6); pass a larger ``max_table`` (or None) to
    enumerate instances the host-RAM reference cannot -- the tables live in HBM."""
    from .tables import f64_tables, recognise_q
    cells = grid_spec.width * grid_spec.height
    n_hyp = space.size
    m = len(control_set)
    if max_table is not None and cells * m * n_hyp > max_table:
        raise EnumerationCapExceeded(f"{cells} cells x {m} actions x {n_hyp} hypotheses exceeds cap "
                                     f"{max_table}; use the Monte-Carlo predictor")
    if len(belief) != n_hyp:
        raise ValueError("belief size does not match hypothesis space")
    dev = device()
    up = lambda a_, t_: torch.as_tensor(np.array(a_, dtype=t_, order="C"), device=dev)
    beta_of, goal_of = hypothesis_arrays(space)
    v, th = np.asarray(control_set.v, float), np.asarray(control_set.theta, float)
    lq = recognise_q(q)
    a = _lib.ExactArgs()
    keep = []
    if lq is not None:
        sx, sy, at, pen = f64_tables(v, th, lq)
        a.q_kind = _lib.GC_Q_DEFAULT if lq.family == "default" else _lib.GC_Q_GOAL_PROGRESS_FULL
    else:
        sx = sy = at = pen = np.zeros(m)
        a.q_kind = _lib.GC_Q_TABLE
        centers = grid_spec.all_centers()
        qt = np.stack([q.table(centers, np.tile(goal_of[h], (cells, 1)), control_set) for h in range(n_hyp)])
        qt0 = q.table(np.tile([[z_t.x, z_t.y]], (n_hyp, 1)), goal_of, control_set)
        keep += [up(qt, np.float64), up(qt0, np.float64)]
        a.d_qtable, a.d_qtable0 = keep[-2].data_ptr(), keep[-1].data_ptr()
    mask = q.action_mask(control_set)
    disp = control_set.displacements(dt)
    t_beta, t_goal, t_b = up(beta_of, np.float64), up(goal_of, np.float64), up(belief.probs(), np.float64)
    t_sx, t_sy, t_at, t_pen = up(sx, np.float64), up(sy, np.float64), up(at, np.float64), up(pen, np.float64)
    t_dx, t_dy = up(disp[:, 0], np.float64), up(disp[:, 1], np.float64)
    t_mask = up(mask.astype(np.uint8), np.uint8) if mask is not None else None
    pi = torch.empty(n_hyp * cells * m, dtype=torch.float64, device=dev)
    land = torch.empty(cells * m, dtype=torch.int32, device=dev)
    p = torch.empty(n_hyp * cells, dtype=torch.float64, device=dev)
    nxt = torch.empty_like(p)
    pi0 = torch.empty(n_hyp * m, dtype=torch.float64, device=dev)
    layers = torch.empty((steps, grid_spec.height, grid_spec.width), dtype=torch.float64, device=dev)
    a.n_hyp, a.m, a.grid_w, a.grid_h, a.steps = n_hyp, m, grid_spec.width, grid_spec.height, int(steps)
    a.origin_x, a.origin_y, a.res = grid_spec.origin[0], grid_spec.origin[1], grid_spec.resolution
    a.z0x, a.z0y = float(z_t.x), float(z_t.y)
    a.d_beta, a.d_goal, a.d_belief = t_beta.data_ptr(), t_goal.data_ptr(), t_b.data_ptr()
    a.d_sx, a.d_sy, a.d_at, a.d_pen = t_sx.data_ptr(), t_sy.data_ptr(), t_at.data_ptr(), t_pen.data_ptr()
    a.d_dispx, a.d_dispy = t_dx.data_ptr(), t_dy.data_ptr()
    a.d_masked = t_mask.data_ptr() if t_mask is not None else None
    a.d_pi, a.d_p, a.d_nxt, a.d_pi0 = pi.data_ptr(), p.data_ptr(), nxt.data_ptr(), pi0.data_ptr()
    a.d_landing, a.d_layers = land.data_ptr(), layers.data_ptr()
    _lib.check(_lib.lib().gc_exact_predict(ctypes.byref(a), stream_handle()), "exact_predict")
    torch.cuda.current_stream().synchronize()
    return PredictionStack(grid_spec, layers, base_time, dt)


def total_variation(a, b) -> float:
    return 0.5 * float(np.abs(np.asarray(a, dtype=float) - np.asarray(b, dtype=float)).sum())
