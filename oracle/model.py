"""ORACLE (test infrastructure only): per-action and per-hypothesis tables.

Restates, with the same numpy expressions (so the same float32/float64 roundings
under NEP 50), the table-shaped parts of the reference model:

  ControlSet.grid / displacements    agents.py:79-87, :108-112
  q_goal_progress (shift_free/base)  agents.py:262-296  -> sx, sy, at (float32)
  q_default                          agents.py:245-259  -> pen (float32)
  _action_tables (keep map)          prediction.py:134-144
  HypothesisSpace beta_of/goal_xy_of belief.py:54-62 (h = i_beta*|G| + i_goal)
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .cstep import Q_DEFAULT, Q_GOAL_PROGRESS, Q_GOAL_PROGRESS_FULL


@dataclass
class QSpec:
    """Recognised utility family: 'goal_progress' (tau, weights) or 'default' (weights).

    ``full`` selects the reference's ``base`` (with -|rel|^2) instead of
    ``base_policy``; ``mask_stationary`` drops base_policy (belief.py:222) so a masked
    goal-progress Q propagates with the full base.  ``v_threshold`` (None = no mask)
    is the mask_stationary threshold.
    """

    family: str = "goal_progress"
    tau: float = 0.5
    w_v: float = 0.0
    w_th: float = 0.0
    v_threshold: float | None = None

    @property
    def masked(self) -> bool:
        return self.v_threshold is not None


@dataclass
class Tables:
    v: np.ndarray
    theta: np.ndarray
    sx: np.ndarray
    sy: np.ndarray
    at: np.ndarray
    pen: np.ndarray
    dispx: np.ndarray
    dispy: np.ndarray
    keep: np.ndarray
    q_kind: int


def control_grid(n_speeds=4, n_headings=24, v_max=1.4):
    """(v, theta) float64 rows of ControlSet.grid (index = iv*n_headings + ith)."""
    speeds = np.linspace(0.0, v_max, n_speeds)
    headings = -np.pi + 2.0 * np.pi * np.arange(n_headings) / n_headings
    v = np.repeat(speeds, n_headings)
    th = np.tile(headings, n_speeds)
    # ControlAction wraps theta to [-pi, pi) (agents.py:24-26, :55)
    th = np.array([float((t + math.pi) % (2.0 * math.pi) - math.pi) for t in th])
    return v, th


def make_tables(v, theta, dt, q: QSpec) -> Tables:
    v = np.asarray(v, dtype=float)
    theta = np.asarray(theta, dtype=float)
    m = len(v)
    disp = np.stack([v * np.cos(theta) * dt, v * np.sin(theta) * dt], axis=1).astype(np.float32)
    v32 = v.astype(np.float32)
    th32 = theta.astype(np.float32)
    sx = np.zeros(m, np.float32)
    sy = np.zeros(m, np.float32)
    at = np.zeros(m, np.float32)
    pen = np.zeros(m, np.float32)
    if q.family == "goal_progress":
        tau = float(q.tau)
        sx = v32 * np.cos(th32) * tau
        sy = v32 * np.sin(th32) * tau
        at = sx * sx + sy * sy
        if q.w_v != 0.0 or q.w_th != 0.0:
            at = at + (float(q.w_v) * v32 * v32 + float(q.w_th) * th32 * th32)
        kind = Q_GOAL_PROGRESS_FULL if q.masked else Q_GOAL_PROGRESS
    elif q.family == "default":
        pen = float(q.w_v) * v32 * v32 + float(q.w_th) * th32 * th32
        kind = Q_DEFAULT
    else:
        raise ValueError(q.family)
    if q.masked:
        keep = np.flatnonzero(~(v > q.v_threshold))
    else:
        keep = np.arange(m)
    return Tables(v, theta, sx.astype(np.float32), sy.astype(np.float32),
                  at.astype(np.float32), pen.astype(np.float32),
                  np.ascontiguousarray(disp[:, 0]), np.ascontiguousarray(disp[:, 1]),
                  keep.astype(np.int32), kind)


def hypothesis_tables(betas, goals):
    """beta_of (|H|,), goal_xy_of (|H|,2) float64 with h = i_beta*|G| + i_goal."""
    betas = np.asarray(betas, dtype=float)
    goals = np.atleast_2d(np.asarray(goals, dtype=float))
    return np.repeat(betas, len(goals)), np.tile(goals, (len(betas), 1))
