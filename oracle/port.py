"""ORACLE / CPU BASELINE (test + bench infrastructure only): the reference's CPU cycle,
restated with the same numpy structure so it can be timed on the GPU box's host cores
(the reference package itself cannot travel there).

Follows, op for op and with the same library calls:
  update_belief        belief.py:159-198 (float64, scipy logsumexp)
  predict              prediction.py:223-255 with sample_hypotheses :124-131,
                       propagate_step :165-211 (1024-particle chunks, ThreadPoolExecutor
                       over chunks, per-chunk numpy Philox streams), _propagate_chunk
                       :147-162 (q_goal_progress.shift_free agents.py:275-288 via BLAS),
                       emplace_counts occupancy.py:105-109, smooth_values :139-154 (dense
                       float64 matmuls)
  union_max / time union  occupancy.py:162-192, sim.py:500-504
Bit-identical to the reference on x86 hosts (tests/test_oracle_golden.py pins it).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy.special import logsumexp

from .model import Tables
from .predict import Grid, _smoothing_matrix, belief_update

CHUNK = 1024


def _stream(seed, *path):
    key = tuple(int(p) & 0xFFFFFFFF for p in path)
    ss = np.random.SeedSequence(entropy=int(seed) & ((1 << 64) - 1), spawn_key=key)
    return np.random.Generator(np.random.Philox(ss))


def _chunk(xy, hyp, betas_of, goals_of, tb: Tables, u01, full, default):
    goal = goals_of[hyp]
    rel = xy - goal
    if default:
        d2 = np.sum(rel ** 2, axis=1)
        logits = -d2[:, None] - tb.pen[None, :]
    else:
        logits = rel @ np.stack([tb.sx, tb.sy])
        logits *= -2.0
        logits -= tb.at[None, :]
        if full:
            logits -= np.einsum("ij,ij->i", rel, rel)[:, None]
    if len(tb.keep) != logits.shape[1]:
        logits = logits[:, tb.keep]
    logits *= betas_of[hyp][:, None]
    logits -= logits.max(axis=1, keepdims=True)
    w = np.exp(logits, out=logits)
    cdf = np.cumsum(w, axis=1, out=w)
    r = u01 * cdf[:, -1]
    picked = np.sum(cdf < r[:, None], axis=1)
    np.minimum(picked, len(tb.keep) - 1, out=picked)
    a = tb.keep[picked]
    return xy + np.stack([tb.dispx[a], tb.dispy[a]], axis=1)


def predict(z0, log_w, n, steps, dt, sigma, seed, tb: Tables, beta_of, goal_xy_of, grid: Grid,
            prefix=(), workers=None):
    cdf = np.cumsum(np.exp(np.asarray(log_w, float)))
    cdf[-1] = 1.0
    hyp = np.searchsorted(cdf, _stream(seed, *prefix, 0).random(n), side="right").astype(np.int32)
    xy = np.tile(np.array([z0[0], z0[1]], dtype=np.float32), (n, 1))
    b32 = np.asarray(beta_of).astype(np.float32)
    g32 = np.asarray(goal_xy_of).astype(np.float32)
    full = tb.q_kind == 1
    default = tb.q_kind == 2
    layers = np.empty((steps, grid.height, grid.width))
    chunks = [(s, min(s + CHUNK, n), i) for i, s in enumerate(range(0, n, CHUNK))]
    pool = ThreadPoolExecutor(max_workers=workers) if workers and workers > 1 and len(chunks) > 1 else None
    my = mx = None
    if sigma > 0 and sigma / grid.resolution >= 1e-12:
        my = _smoothing_matrix(grid.height, sigma / grid.resolution)
        mx = _smoothing_matrix(grid.width, sigma / grid.resolution)
    try:
        for t in range(1, steps + 1):
            out = np.empty_like(xy)

            def run(c):
                s, e, i = c
                u = _stream(seed, *prefix, 1, t, i).random(e - s, dtype=np.float32)
                out[s:e] = _chunk(xy[s:e], hyp[s:e], b32, g32, tb, u, full, default)

            if pool is not None:
                list(pool.map(run, chunks))
            else:
                for c in chunks:
                    run(c)
            xy = out
            ix = np.clip(np.floor((xy[:, 0] - grid.origin[0]) / grid.resolution).astype(np.int64), 0, grid.width - 1)
            iy = np.clip(np.floor((xy[:, 1] - grid.origin[1]) / grid.resolution).astype(np.int64), 0, grid.height - 1)
            vals = np.bincount(iy * grid.width + ix, minlength=grid.width * grid.height).reshape(
                grid.height, grid.width).astype(float) / n
            if my is not None:
                o = my @ vals @ mx.T
                before, after = vals.sum(), o.sum()
                if after > 0.0:
                    o *= before / after
                vals = np.maximum(o, 0.0)
            layers[t - 1] = vals
    finally:
        if pool is not None:
            pool.shutdown()
    return layers


def cycle(humans, tb_model, tb_masked, v, theta, qspec, grid, n, steps, dt, sigma, seed, obs_dt,
          workers=None, time_union=False):
    """One sim-style cycle (sim.py:455-504): update every human, predict every human with
    prefix (2, i), union_max, optional time union.  ``humans``: list of dicts with
    log_w, beta_of, goal_xy_of, prev, obs, heading, stationary."""
    stacks = []
    for i, hm in enumerate(humans):
        post, _ = belief_update(hm["log_w"], hm["prev"], hm["obs"], obs_dt, v, theta, qspec,
                                hm["beta_of"], hm["goal_xy_of"], hm["heading"], snap_tol=math.inf)
        hm["log_w"] = post
        tb = tb_masked if hm.get("stationary") else tb_model
        stacks.append(predict(hm["obs"], post, n, steps, dt, sigma, seed, tb, hm["beta_of"],
                              hm["goal_xy_of"], grid, prefix=(2, i), workers=workers))
    u = stacks[0].copy()
    for s in stacks[1:]:
        np.maximum(u, s, out=u)
    if time_union:
        np.maximum.accumulate(u, axis=0, out=u)
    return u


def default_workers() -> int:
    return os.cpu_count() or 1


__all__ = ["predict", "cycle", "logsumexp", "default_workers"]
