"""ORACLE (test infrastructure only): the reference prediction cycle restated.

  sample_hypotheses   prediction.py:124-131  (f64 cumsum cdf, searchsorted right)
  step_uniforms       prediction.py:186-192  (chunk-keyed f32 streams, CHUNK=1024)
  predict             prediction.py:223-255  (propagate -> emplace/n -> smooth per layer)
  smooth_dense        occupancy.py:122-154   (column-normalised truncated Gaussian)
  smooth_banded       SURVEY.md App. A.5     (same operator as a 7-tap-style banded stencil)
  predict_naive       prediction.py:258-300  (float64 per-particle loop, f64 chunk streams)
  union_max/union_independent/time_union occupancy.py:162-192, sim.py:500-504
  belief_update       belief.py:159-198 with agents.py:299-323, :355-371, :114-134
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import logsumexp

from . import cstep, philox
from .model import QSpec, Tables

CHUNK = 1024
LOG_WEIGHT_FLOOR = -745.0
EPS_STATIONARY = 1e-6


class Grid:
    def __init__(self, width, height, resolution, origin=(0.0, 0.0)):
        self.width = int(width)
        self.height = int(height)
        self.resolution = float(resolution)
        self.origin = (float(origin[0]), float(origin[1]))

    @property
    def shape(self):
        return (self.height, self.width)


def hypothesis_cdf(log_w) -> np.ndarray:
    cdf = np.cumsum(np.exp(np.asarray(log_w, dtype=float)))
    cdf[-1] = 1.0
    return cdf


def sample_hypotheses(log_w, n, seed, prefix=()) -> np.ndarray:
    u = philox.stream_random_f64(seed, tuple(prefix) + (0,), n)
    return np.searchsorted(hypothesis_cdf(log_w), u, side="right").astype(np.int32)


def step_uniforms(seed, prefix, t, n) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    for c, start in enumerate(range(0, n, CHUNK)):
        stop = min(start + CHUNK, n)
        out[start:stop] = philox.stream_random_f32(seed, tuple(prefix) + (1, t, c), stop - start)
    return out


def _smoothing_matrix(size, sigma_cells):
    radius = int(np.ceil(3.0 * sigma_cells))
    offs = np.arange(-radius, radius + 1)
    k = np.exp(-0.5 * (offs / sigma_cells) ** 2)
    m = np.zeros((size, size))
    for o, kv in zip(offs, k):
        src = np.arange(max(0, -o), min(size, size - o))
        m[src + o, src] += kv
    return m / m.sum(axis=0, keepdims=True)


def smooth_dense(values, grid, sigma_m):
    sc = sigma_m / grid.resolution
    if sc < 1e-12:
        return values.copy()
    my = _smoothing_matrix(grid.height, sc)
    mx = _smoothing_matrix(grid.width, sc)
    out = my @ values @ mx.T
    before, after = values.sum(), out.sum()
    if after > 0.0:
        out *= before / after
    return np.maximum(out, 0.0)


def smooth_banded(values, grid, sigma_m):
    """Same operator as smooth_dense as a banded separable stencil (App. A.5)."""
    sc = sigma_m / grid.resolution
    if sc < 1e-12:
        return values.copy()
    R = int(np.ceil(3.0 * sc))
    offs = np.arange(-R, R + 1)
    k = np.exp(-0.5 * (offs / sc) ** 2)

    def axis_pass(a, size, axis):
        # Z(j) = in-grid kernel mass of a unit source at j
        z = np.zeros(size)
        for o, kv in zip(offs, k):
            j = np.arange(max(0, -o), min(size, size - o))
            z[j] += kv
        a = np.moveaxis(a, axis, 0) / z[:, None]
        out = np.zeros_like(a)
        for o, kv in zip(offs, k):
            src = np.arange(max(0, -o), min(size, size - o))
            out[src + o] += kv * a[src]
        return np.moveaxis(out, 0, axis)

    out = axis_pass(values, grid.height, 0)
    out = axis_pass(out, grid.width, 1)
    before, after = values.sum(), out.sum()
    if after > 0.0:
        out *= before / after
    return np.maximum(out, 0.0)


def predict(z0, log_w, n, steps, dt, sigma, seed, tables: Tables, beta_of, goal_xy_of, grid,
            prefix=(), keep_xy=False, uniforms=None, hyp=None):
    """Oracle Alg. 1.  Returns dict(hyp, counts (T,H,W) int64, layers (T,H,W) f64[, xy])."""
    if hyp is None:
        hyp = sample_hypotheses(log_w, n, seed, prefix)
    xy = np.tile(np.array([z0[0], z0[1]], dtype=np.float32), (n, 1))
    beta32 = np.asarray(beta_of).astype(np.float32)
    goal32 = np.asarray(goal_xy_of).astype(np.float32)
    counts = np.zeros((steps, grid.height, grid.width), dtype=np.int64)
    layers = np.zeros((steps, grid.height, grid.width))
    xs = []
    for t in range(1, steps + 1):
        u = uniforms[t - 1] if uniforms is not None else step_uniforms(seed, prefix, t, n)
        xy = cstep.propagate(xy, hyp, beta32, goal32, tables, u)
        flat = cstep.cells(xy, grid)
        c = np.bincount(flat, minlength=grid.width * grid.height).reshape(grid.shape)
        counts[t - 1] = c
        vals = c.astype(float) / n
        if sigma > 0:
            vals = smooth_dense(vals, grid, sigma)
        layers[t - 1] = vals
        if keep_xy:
            xs.append(xy.copy())
    out = dict(hyp=hyp, counts=counts, layers=layers)
    if keep_xy:
        out["xy"] = np.stack(xs)
    return out


def predict_naive(z0, log_w, n, steps, dt, sigma, seed, v, theta, q: QSpec, beta_of, goal_xy_of, grid):
    """predict_naive (prediction.py:258-300): one particle at a time in float64 -- q.table
    of the particle's hypothesis (agents.py:222-224), beta x, max shift, exp, cumsum,
    #(cdf < u cdf[-1]); u from the f64 chunk streams (seed, 1, t, chunk) (no prefix);
    displacements v cos(theta) dt in f64 (agents.py:108-112); f64 cells_of."""
    v = np.asarray(v, float)
    theta = np.asarray(theta, float)
    beta_of = np.asarray(beta_of, float)
    goal_xy_of = np.asarray(goal_xy_of, float)
    hyp = sample_hypotheses(log_w, n, seed)
    xy = np.tile(np.array([z0[0], z0[1]], dtype=float), (n, 1))
    disp = np.stack([v * np.cos(theta) * dt, v * np.sin(theta) * dt], axis=1)
    keep = np.arange(len(v)) if not q.masked else np.flatnonzero(~(v > q.v_threshold))
    layers = np.empty((steps, grid.height, grid.width))
    for t in range(1, steps + 1):
        for c, start in enumerate(range(0, n, CHUNK)):
            stop = min(start + CHUNK, n)
            u = philox.stream_random_f64(seed, (1, t, c), stop - start)
            for i in range(start, stop):
                h = hyp[i]
                qt = q_table_f64(xy[i:i + 1], goal_xy_of[h:h + 1], v, theta, q)[0, keep]
                logits = beta_of[h] * qt
                logits -= logits.max()
                cdf = np.cumsum(np.exp(logits))
                j = min(int(np.sum(cdf < u[i - start] * cdf[-1])), len(keep) - 1)
                xy[i] += disp[keep[j]]
        ix = np.clip(np.floor((xy[:, 0] - grid.origin[0]) / grid.resolution).astype(np.int64), 0, grid.width - 1)
        iy = np.clip(np.floor((xy[:, 1] - grid.origin[1]) / grid.resolution).astype(np.int64), 0, grid.height - 1)
        vals = np.bincount(iy * grid.width + ix, minlength=grid.width * grid.height).reshape(grid.shape) / n
        if sigma > 0:
            vals = smooth_dense(vals, grid, sigma)
        layers[t - 1] = vals
    return dict(hyp=hyp, layers=layers, xy=xy)


def union_max(stacks):
    out = np.array(stacks[0], dtype=float, copy=True)
    for s in stacks[1:]:
        np.maximum(out, s, out=out)
    return out


def union_independent(stacks):
    """1 - prod(1 - clip(p, 0, 1)) in the reference's order (occupancy.py:180-184)."""
    miss = 1.0 - np.clip(np.asarray(stacks[0], dtype=float), 0.0, 1.0)
    for s in stacks[1:]:
        miss = miss * (1.0 - np.clip(np.asarray(s, dtype=float), 0.0, 1.0))
    return 1.0 - miss


def time_union(layers):
    return np.maximum.accumulate(np.asarray(layers, dtype=float), axis=0)


# --- belief update (float64) -----------------------------------------------------

def wrap(theta):
    return float((theta + math.pi) % (2.0 * math.pi) - math.pi)


def recover_control(zt, zn, dt, fallback_theta):
    dx, dy = zn[0] - zt[0], zn[1] - zt[1]
    d = math.hypot(dx, dy)
    if d < EPS_STATIONARY:
        return 0.0, wrap(fallback_theta)
    return d / dt, wrap(math.atan2(dy, dx))


def default_snap_tol(v, theta):
    def max_gap(vals, circular):
        u = np.unique(vals)
        if len(u) < 2:
            return 0.0
        g = np.diff(u)
        if circular:
            g = np.append(g, 2.0 * np.pi - (u[-1] - u[0]))
        return float(np.max(g))
    return 0.5 * (max_gap(v, False) + max_gap(theta, True)) + 1e-9


def snap(v, theta, uv, uth, tol=None):
    """Returns (idx, dist) or raises ValueError('snap') beyond tol."""
    tol = default_snap_tol(v, theta) if tol is None else float(tol)
    dist = np.abs(v - uv) + np.abs((theta - uth + np.pi) % (2.0 * np.pi) - np.pi)
    idx = int(np.argmin(dist))
    if dist[idx] > tol:
        raise ValueError("snap")
    return idx


def q_table_f64(xy, goal, v, theta, q: QSpec):
    """(n, m) float64 q.table (full base, masked -> -inf), agents.py:222-224."""
    xy = np.atleast_2d(xy)
    goal = np.atleast_2d(goal)
    if q.family == "goal_progress":
        sx = v * np.cos(theta) * q.tau
        sy = v * np.sin(theta) * q.tau
        rel = xy - goal
        out = rel @ np.stack([sx, sy])
        out *= -2.0
        at = sx * sx + sy * sy
        if q.w_v != 0.0 or q.w_th != 0.0:
            at = at + (q.w_v * v * v + q.w_th * theta * theta)
        out -= at[None, :]
        out -= np.einsum("ij,ij->i", rel, rel)[:, None]
    else:
        d2 = np.sum((xy - goal) ** 2, axis=1)
        pen = q.w_v * v * v + q.w_th * theta * theta
        out = -d2[:, None] - pen[None, :]
    if q.masked:
        out[:, v > q.v_threshold] = -np.inf
    return out


def policy_log_table(xy, goal, betas, v, theta, q: QSpec):
    qt = q_table_f64(xy, goal, v, theta, q)
    logits = np.asarray(betas, float)[:, None] * qt
    shift = np.max(logits, axis=1, keepdims=True)
    shifted = logits - shift
    shifted[~np.isfinite(logits)] = -np.inf
    lse = np.log(np.sum(np.exp(shifted), axis=1, keepdims=True))
    return shifted - lse


def belief_update(log_w, zt, zn, dt, v, theta, q: QSpec, beta_of, goal_xy_of,
                  fallback_theta=0.0, snap_tol=None):
    uv, uth = recover_control(zt, zn, dt, fallback_theta)
    idx = snap(v, theta, uv, uth, snap_tol)
    H = len(beta_of)
    xy = np.tile(np.array([[zt[0], zt[1]]], dtype=float), (H, 1))
    loglik = policy_log_table(xy, goal_xy_of, beta_of, v, theta, q)[:, idx]
    prior = np.asarray(log_w, dtype=float)
    zeroed = np.isneginf(prior)
    post = prior + loglik
    post[~zeroed] = np.maximum(post[~zeroed], LOG_WEIGHT_FLOOR)
    post[zeroed] = -np.inf
    return post - logsumexp(post), idx
