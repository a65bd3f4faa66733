"""Host-side lowering of the predictor's plug-ins to the flat tables the kernels read.

* ``recognise_q``   -- QFunction -> (family, tau, w_v, w_th, full) for the kernels
  (the plug-in surface that cannot cross a C ABI).  Our own
  q_goal_progress / q_default carry ``spec``; reference-built QFunctions are recognised
  from their closure cells; anything else raises NotImplementedError for prediction
  (no CPU fallback) and is lowered to a host-evaluated (|H|, m) table for updates.
* ``ActionTables``  -- per-action float32 tables exactly as the reference computes them
  under NEP 50 (agents.py:275-296, prediction.py:134-144), plus the factorised-sampler
  description (speed x heading grid) for production mode; uploaded once, cached.
* ``Geometry``      -- reachable-cell windows per step, count-buffer layout, epilogue
  tiles and smoothing tables for one (grid, dt, horizon, sigma) configuration.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from .agents import QSpec


@dataclass(frozen=True)
class LoweredQ:
    family: str   # "goal_progress" | "default"
    tau: float
    w_v: float
    w_th: float
    full: bool    # use the full base (-|rel|^2 included): base_policy absent


def _closure_vars(fn):
    if fn is None or getattr(fn, "__closure__", None) is None:
        return {}
    return dict(zip(fn.__code__.co_freevars, (c.cell_contents for c in fn.__closure__)))


def recognise_q(q) -> Optional[LoweredQ]:
    """Family of a QFunction (ours or the reference's), or None if unrecognised."""
    spec = getattr(q, "spec", None)
    full = getattr(q, "base_policy", None) is None
    if isinstance(spec, QSpec):
        return LoweredQ(spec.family, spec.tau, spec.w_v, spec.w_th, full)
    base = getattr(q, "base", None)
    bp = getattr(q, "base_policy", None)
    for fn in (bp, base):
        qn = getattr(fn, "__qualname__", "")
        cv = _closure_vars(fn)
        if qn.endswith("q_goal_progress.<locals>.shift_free"):
            return LoweredQ("goal_progress", float(cv["tau"]), float(cv["w_v"]), float(cv["w_th"]), full)
        if qn.endswith("q_goal_progress.<locals>.base"):
            inner = _closure_vars(cv.get("shift_free"))
            if "tau" in inner:
                return LoweredQ("goal_progress", float(inner["tau"]), float(inner["w_v"]),
                                float(inner["w_th"]), full)
        if qn.endswith("q_default.<locals>.base"):
            return LoweredQ("default", 0.5, float(cv["w_v"]), float(cv["w_th"]), True)
    return None


def _kind(lq: LoweredQ) -> int:
    if lq.family == "default":
        return _lib.GC_Q_DEFAULT
    return _lib.GC_Q_GOAL_PROGRESS_FULL if lq.full else _lib.GC_Q_GOAL_PROGRESS


def f32_tables(v, theta, lq: LoweredQ):
    """float32 sx, sy, at, pen with the reference's NEP-50 expression order."""
    v32 = np.asarray(v, dtype=float).astype(np.float32)
    th32 = np.asarray(theta, dtype=float).astype(np.float32)
    m = len(v32)
    zeros = np.zeros(m, np.float32)
    if lq.family == "goal_progress":
        sx = v32 * np.cos(th32) * lq.tau
        sy = v32 * np.sin(th32) * lq.tau
        at = sx * sx + sy * sy
        if lq.w_v != 0.0 or lq.w_th != 0.0:
            at = at + (lq.w_v * v32 * v32 + lq.w_th * th32 * th32)
        return sx.astype(np.float32), sy.astype(np.float32), at.astype(np.float32), zeros
    pen = lq.w_v * v32 * v32 + lq.w_th * th32 * th32
    return zeros, zeros, zeros, pen.astype(np.float32)


def f64_tables(v, theta, lq: LoweredQ):
    """float64 tables of q.table for the belief update (agents.py:222-224)."""
    v = np.asarray(v, dtype=float)
    th = np.asarray(theta, dtype=float)
    z = np.zeros_like(v)
    if lq.family == "goal_progress":
        sx = v * np.cos(th) * lq.tau
        sy = v * np.sin(th) * lq.tau
        at = sx * sx + sy * sy
        if lq.w_v != 0.0 or lq.w_th != 0.0:
            at = at + (lq.w_v * v * v + lq.w_th * th * th)
        return sx, sy, at, z
    return z, z, z, lq.w_v * v * v + lq.w_th * th * th


def _factorisation(v, theta, keep):
    """(n_speeds_kept, dv, headings, a_index) if actions form speeds{a*dv} x headings."""
    v = np.asarray(v, float)
    th = np.asarray(theta, float)
    speeds = np.unique(v)
    heads = np.unique(th)
    if len(speeds) < 2 or len(speeds) * len(heads) != len(v) or speeds[0] != 0.0:
        return None
    dv = speeds[1]
    if np.max(np.abs(speeds - dv * np.arange(len(speeds)))) > 1e-9:
        return None
    a_index = -np.ones((len(speeds), len(heads)), dtype=np.int32)
    ia = np.searchsorted(speeds, v)
    ib = np.searchsorted(heads, th)
    a_index[ia, ib] = np.arange(len(v))
    if (a_index < 0).any():
        return None
    keep_set = set(int(k) for k in keep)
    na = 0
    for a in range(len(speeds)):
        row = set(int(j) for j in a_index[a])
        if row <= keep_set:
            na = a + 1
        elif row & keep_set:
            return None
        else:
            break
    if na * len(heads) != len(keep_set) or na < 2:
        return None
    return na, float(dv), heads, a_index[:na]


class ActionTables:
    """Device-resident per-action tables for one (control set, Q, dt)."""

    def __init__(self, control_set, q, dt: float, device, require: bool = True):
        lq = recognise_q(q)
        if lq is None:
            if require:
                raise NotImplementedError(
                    "the B200 predictor implements q_goal_progress and q_default (and their "
                    "stationary-masked forms); this QFunction is not recognised and there is "
                    "no CPU fallback")
        self.lq = lq
        v = np.asarray(control_set.v, float)
        th = np.asarray(control_set.theta, float)
        self.m = len(v)
        mask = q.action_mask(control_set)
        keep = np.arange(self.m) if mask is None else np.flatnonzero(~mask)
        if len(keep) == 0:
            from .agents import EmptyControlSetError
            raise EmptyControlSetError("all actions are masked")
        self.keep_np = keep.astype(np.int32)
        disp = control_set.displacements(dt).astype(np.float32)
        self.disp_np = disp
        self.max_step = float(np.max(np.abs(disp[keep]))) if len(keep) else 0.0
        sx, sy, at, pen = f32_tables(v, th, lq) if lq else (np.zeros(self.m, np.float32),) * 4
        dev = lambda a, dt_=None: torch.as_tensor(np.array(a, order="C"), device=device)
        self._keep_alive = []
        self.d_sx, self.d_sy, self.d_at, self.d_pen = dev(sx), dev(sy), dev(at), dev(pen)
        self.d_dispx = dev(disp[:, 0].copy())
        self.d_dispy = dev(disp[:, 1].copy())
        self.d_keep = dev(self.keep_np)
        fact = _factorisation(v, th, keep) if lq and lq.family == "goal_progress" else None
        t = _lib.ActionTable()
        t.m, t.m_keep = self.m, len(keep)
        t.q_kind = _kind(lq) if lq else _lib.GC_Q_TABLE
        for name in ("sx", "sy", "at", "pen", "dispx", "dispy", "keep"):
            setattr(t, "d_" + name, getattr(self, "d_" + name).data_ptr())
        self.factorised = fact is not None
        if fact is not None:
            na, dv, heads, a_index = fact
            self.d_cos = dev(np.cos(heads).astype(np.float32))
            self.d_sin = dev(np.sin(heads).astype(np.float32))
            self.d_theta = dev(heads.astype(np.float32))
            self.d_aidx = dev(np.ascontiguousarray(a_index.reshape(-1)).astype(np.int32))
            t.n_speeds, t.n_headings = na, len(heads)
            t.dv, t.tau, t.w_v, t.w_th = dv, lq.tau, lq.w_v, lq.w_th
            t.d_cos_h, t.d_sin_h = self.d_cos.data_ptr(), self.d_sin.data_ptr()
            t.d_theta_h, t.d_a_index = self.d_theta.data_ptr(), self.d_aidx.data_ptr()
            self.h_cos = np.ascontiguousarray(np.cos(heads).astype(np.float32))
            self.h_sin = np.ascontiguousarray(np.sin(heads).astype(np.float32))
            self.h_theta = np.ascontiguousarray(heads.astype(np.float32))
            t.h_cos_h = self.h_cos.ctypes.data
            t.h_sin_h = self.h_sin.ctypes.data
            t.h_theta_h = self.h_theta.ctypes.data
            self.headings = heads
            # reference-mode max-logit guess (gc_action_table.ref_grid_rows): the standard
            # 24 headings, action a*24 + b, no heading weight
            std = -np.pi + np.arange(24) * (np.pi / 12)
            if (len(heads) == 24 and np.allclose(heads, std, rtol=0, atol=1e-9) and lq.w_th == 0.0
                    and np.array_equal(a_index, np.arange(na * 24, dtype=np.int32).reshape(na, 24))
                    and np.array_equal(keep, np.arange(na * 24))):
                t.ref_grid_rows = na
        self.struct = t


def assume_qg(tables, betas) -> bool:
    """gc_predict_args.assume_qg for a production launch: True when every factorised table
    and every hypothesis beta keep the factorised sampler's top-speed normalisation
    representable -- K2 needs 9 c + log2(24) < 100 with c = beta (tau^2 + w_v) dv^2 log2(e)
    (4 speeds; less with fewer); this host test keeps 10 units of margin in the exponent,
    so float rounding on the device can never disagree with it."""
    bmax = float(np.max(np.concatenate([np.asarray(b, dtype=float).ravel() for b in betas]))) if len(betas) else 0.0
    for t in tables:
        if not getattr(t, "factorised", False):
            continue
        st = t.struct
        c = bmax * (st.tau * st.tau + st.w_v) * st.dv * st.dv * 1.4426950408889634
        if not np.isfinite(c) or 9.0 * c + np.log2(24.0) >= 90.0:
            return False
    return True


def hypothesis_arrays(space):
    """beta_of (|H|,), goal_xy_of (|H|,2) with h = i_beta*|G| + i_goal (belief.py:54-62)."""
    betas = np.asarray(space.rationalities.array if hasattr(space.rationalities, "array")
                       else space.rationalities.betas, dtype=float)
    goals = np.atleast_2d(np.asarray(space.goals.positions, dtype=float))
    return np.repeat(betas, len(goals)), np.tile(goals, (len(betas), 1))


class Geometry:
    """Reachable-cell windows, count layout, epilogue tiles, smoothing tables."""

    TILE = 32

    def __init__(self, grid_spec, steps: int, max_step: float, sigma_m: float, device):
        self.W, self.H = int(grid_spec.width), int(grid_spec.height)
        self.res = float(grid_spec.resolution)
        self.ox, self.oy = float(grid_spec.origin[0]), float(grid_spec.origin[1])
        self.steps = int(steps)
        t = np.arange(1, steps + 1, dtype=float)
        r = np.ceil(t * max_step / self.res).astype(np.int64) + 2
        # the window never needs to exceed the grid itself
        r = np.minimum(r, max(self.W, self.H))
        self.step_r = r.astype(np.int32)
        side = np.minimum(2 * r + 1, np.maximum(self.W, self.H) * 2 + 1)
        cells = (2 * r + 1) ** 2
        self.step_off = np.concatenate([[0], np.cumsum(cells)[:-1]]).astype(np.int64)
        self.human_stride = int(cells.sum())
        self.max_win_cells = int(cells.max())
        self.win_cells = cells.astype(np.int64)  # (2 r_t + 1)^2 per step (non-decreasing)
        sc = sigma_m / self.res if sigma_m > 0 else 0.0
        if sc < 1e-12:
            self.radius = 0
            k = np.ones(1)
        else:
            self.radius = int(np.ceil(3.0 * sc))
            offs = np.arange(-self.radius, self.radius + 1)
            k = np.exp(-0.5 * (offs / sc) ** 2)
        if self.radius > _lib.GC_MAX_SMOOTH_RADIUS:
            raise NotImplementedError(f"smoothing radius above {_lib.GC_MAX_SMOOTH_RADIUS} cells is not implemented")
        self.kernel = k

        def zmass(size):
            z = np.zeros(size)
            for o, kv in zip(range(-self.radius, self.radius + 1), k):
                lo, hi = max(0, -o), min(size, size - o)
                if hi > lo:
                    z[lo:hi] += kv
            return z

        tiles = []
        self.tile_start = np.zeros(steps + 1, dtype=np.int64)  # first tile of step t (0-based)
        for ti in range(steps):
            self.tile_start[ti] = len(tiles)
            nt = -(-(2 * int(r[ti]) + 1 + 2 * self.radius) // self.TILE)
            for ty in range(nt):
                for tx in range(nt):
                    tiles.append((ti, tx, ty, 0))
        self.tile_start[steps] = len(tiles)
        self.n_tiles = len(tiles)
        dev = lambda a: torch.as_tensor(np.array(a, order="C"), device=device)
        self.d_step_r = dev(self.step_r)
        self.d_step_off = dev(self.step_off)
        self.d_tiles = dev(np.asarray(tiles, dtype=np.int32))
        self.d_kernel = dev(k.astype(np.float64))
        self.d_zx = dev(1.0 / zmass(self.W))  # reciprocal column masses (kernels multiply)
        self.d_zy = dev(1.0 / zmass(self.H))
        del side

    def window(self, start_xy32, t):
        """(x0, y0, w, h) of step t (0-based) for a float32 start -- mirrors the kernels."""
        fx = math.floor(np.float32(np.float32(start_xy32[0]) - np.float32(self.ox)) / np.float32(self.res))
        fy = math.floor(np.float32(np.float32(start_xy32[1]) - np.float32(self.oy)) / np.float32(self.res))
        cx = min(max(int(fx), 0), self.W - 1)
        cy = min(max(int(fy), 0), self.H - 1)
        R = int(self.step_r[t])
        x0, x1 = max(0, cx - R), min(self.W - 1, cx + R)
        y0, y1 = max(0, cy - R), min(self.H - 1, cy + R)
        return x0, y0, x1 - x0 + 1, y1 - y0 + 1


def ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())
