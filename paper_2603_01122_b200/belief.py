"""Joint (beta, goal) belief and its Bayesian update (reference belief.py:1-222).

``update_belief`` runs on the GPU (K1, one warp per human: gc_belief_update); the
batched many-human form is ``engine.CycleEngine.observe``.  The small host records
(HypothesisSpace, JointBelief) keep the reference's layout h = i_beta*|G| + i_goal and
its validation (|logsumexp| <= 1e-9, no NaN).
"""

from __future__ import annotations

import ctypes
import math
from collections import OrderedDict
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from . import _lib
from .agents import ControlAction, ControlSet, GoalSet, HumanState, QFunction, RationalitySet
from .device import device, stream_handle, upload_packed
from .tables import f64_tables, hypothesis_arrays, recognise_q

LOG_WEIGHT_FLOOR = -745.0


class ControlSnapMismatch(ValueError):
    """Observed control farther from the control set than the snap tolerance."""


class EmptyMaskResultError(ValueError):
    """Stationary masking would leave no usable action."""


def _logsumexp(a: np.ndarray) -> float:
    a = np.asarray(a, dtype=float)
    m = np.max(a)
    if not np.isfinite(m):
        m = 0.0
    with np.errstate(divide="ignore"):
        return float(np.log(np.sum(np.exp(a - m))) + m)


@dataclass(frozen=True)
class HypothesisSpace:
    rationalities: RationalitySet
    goals: GoalSet

    @property
    def size(self) -> int:
        return len(self.rationalities) * len(self.goals)

    @property
    def beta_of(self) -> np.ndarray:
        return np.repeat(self.rationalities.array, len(self.goals))

    @property
    def goal_xy_of(self) -> np.ndarray:
        return np.tile(self.goals.positions, (len(self.rationalities), 1))

    def index_of(self, beta_index: int, goal_index: int) -> int:
        return beta_index * len(self.goals) + goal_index

    def goal_marginal(self, belief: "JointBelief") -> np.ndarray:
        return belief.probs().reshape(len(self.rationalities), len(self.goals)).sum(axis=0)

    def beta_marginal(self, belief: "JointBelief") -> np.ndarray:
        return belief.probs().reshape(len(self.rationalities), len(self.goals)).sum(axis=1)


@dataclass(frozen=True)
class JointBelief:
    log_weights: np.ndarray

    def __post_init__(self):
        lw = np.asarray(self.log_weights, dtype=float).reshape(-1)
        if lw.size == 0:
            raise ValueError("belief must cover at least one hypothesis")
        if np.isnan(lw).any():
            raise ValueError("belief log weights contain NaN")
        total = _logsumexp(lw)
        if abs(total) > 1e-9:
            raise ValueError(f"belief is not normalized (logsumexp={total:.3e})")
        lw = lw.copy()
        lw.setflags(write=False)
        object.__setattr__(self, "log_weights", lw)

    @classmethod
    def from_probs(cls, probs) -> "JointBelief":
        p = np.asarray(probs, dtype=float).reshape(-1)
        if (p < 0).any():
            raise ValueError("probabilities must be nonnegative")
        s = p.sum()
        if s <= 0:
            raise ValueError("probabilities must sum to a positive value")
        with np.errstate(divide="ignore"):
            return cls(np.log(p / s))

    def __len__(self) -> int:
        return self.log_weights.shape[0]

    def probs(self) -> np.ndarray:
        return np.exp(self.log_weights)


def init_belief(space: HypothesisSpace) -> JointBelief:
    n = space.size
    return JointBelief(np.full(n, -np.log(n)))


def reset_belief(belief: JointBelief) -> JointBelief:
    n = len(belief)
    return JointBelief(np.full(n, -np.log(n)))


def snap_control(u: ControlAction, control_set: ControlSet, tol: Optional[float] = None) -> int:
    tol = control_set.default_snap_tol() if tol is None else float(tol)
    idx, dist = control_set.nearest(u)
    if dist > tol:
        raise ControlSnapMismatch(
            f"observed control (v={u.v:.3f}, theta={u.theta:.3f}) is {dist:.3f} from the "
            f"nearest set action, beyond tolerance {tol:.3f}")
    return idx


def mask_stationary(q: QFunction, control_set: ControlSet, v_threshold: float) -> QFunction:
    """Mask every action faster than v_threshold (belief.py:201-222); like the reference
    the masked Q has no base_policy, so prediction uses the full base."""
    if not np.any(np.asarray(control_set.v) <= v_threshold):
        raise EmptyMaskResultError(f"no action with v <= {v_threshold}; masking would empty the control set")
    prev = q.mask

    def mask(v, theta):
        m = np.asarray(v) > v_threshold
        if prev is not None:
            m = m | np.asarray(prev(v, theta), dtype=bool)
        return m

    return QFunction(base=q.base, mask=mask, spec=getattr(q, "spec", None))


class BeliefTables:
    """float64 per-action tables of one (control set, Q) on the device."""

    def __init__(self, control_set, q, dev):
        self.lq = recognise_q(q)
        v = np.asarray(control_set.v, float)
        th = np.asarray(control_set.theta, float)
        self.m = len(v)
        self.q = q
        self.control_set = control_set
        mask = q.action_mask(control_set)
        up = lambda a: torch.as_tensor(np.array(a, order="C"), device=dev)
        self.d_v, self.d_theta = up(v), up(th)
        self.d_masked = up(mask.astype(np.uint8)) if mask is not None else None
        if self.lq is not None:
            sx, sy, at, pen = f64_tables(v, th, self.lq)
            self.kind = _lib.GC_Q_DEFAULT if self.lq.family == "default" else _lib.GC_Q_GOAL_PROGRESS_FULL
        else:
            sx = sy = at = pen = np.zeros(self.m)
            self.kind = _lib.GC_Q_TABLE
        self.d_sx, self.d_sy, self.d_at, self.d_pen = up(sx), up(sy), up(at), up(pen)
        self.snap_tol = control_set.default_snap_tol()


_TABLE_CACHE: "OrderedDict[tuple, BeliefTables]" = OrderedDict()


def belief_tables(control_set, q, dev) -> BeliefTables:
    key = (id(control_set), id(q), str(dev))
    t = _TABLE_CACHE.get(key)
    if t is None or t.q is not q or t.control_set is not control_set:
        t = BeliefTables(control_set, q, dev)
        _TABLE_CACHE[key] = t
        while len(_TABLE_CACHE) > 64:
            _TABLE_CACHE.popitem(last=False)
    return t


def observation_log_likelihood(z_t, action_index, control_set, q, space) -> np.ndarray:
    """(size,) log pi(u | z_t; beta, g) -- host helper (belief.py:145-156)."""
    from .agents import policy_log_table
    n = space.size
    xy = np.tile(np.array([[z_t.x, z_t.y]], dtype=float), (n, 1))
    return policy_log_table(xy, space.goal_xy_of, space.beta_of, control_set, q)[:, action_index]


def launch_belief_update(bt: BeliefTables, d_hyp_off, d_beta, d_goal, d_obs, d_fallback, d_prior,
                         d_post, d_status, dt, snap_tol, clamp, n_humans, d_qtable=None,
                         d_action=None, stream=None):
    a = _lib.BeliefArgs()
    a.n_humans, a.m = n_humans, bt.m
    a.d_v, a.d_theta = bt.d_v.data_ptr(), bt.d_theta.data_ptr()
    a.d_sx, a.d_sy, a.d_at, a.d_pen = (bt.d_sx.data_ptr(), bt.d_sy.data_ptr(),
                                       bt.d_at.data_ptr(), bt.d_pen.data_ptr())
    a.d_masked = bt.d_masked.data_ptr() if bt.d_masked is not None else None
    a.q_kind = bt.kind
    a.d_qtable = d_qtable.data_ptr() if d_qtable is not None else None
    a.d_hyp_off, a.d_beta, a.d_goal = d_hyp_off.data_ptr(), d_beta.data_ptr(), d_goal.data_ptr()
    a.d_obs, a.d_fallback_theta = d_obs.data_ptr(), d_fallback.data_ptr()
    a.dt, a.snap_tol, a.clamp_on_mismatch = float(dt), float(snap_tol), int(clamp)
    a.d_prior, a.d_post, a.d_status = d_prior.data_ptr(), d_post.data_ptr(), d_status.data_ptr()
    a.d_action = d_action.data_ptr() if d_action is not None else None
    _lib.check(_lib.lib().gc_belief_update(ctypes.byref(a), stream_handle(stream)), "gc_belief_update")


def update_belief(belief: JointBelief, z_t: HumanState, z_next: HumanState, dt: float,
                  control_set: ControlSet, q: QFunction, space: HypothesisSpace,
                  fallback_theta: float = 0.0, snap_tol: Optional[float] = None,
                  transition: Optional[Callable[[np.ndarray], np.ndarray]] = None) -> JointBelief:
    """One Bayesian update from an observed state pair (belief.py:159-198), on the GPU."""
    if len(belief) != space.size:
        raise ValueError("belief size does not match hypothesis space")
    if dt <= 0:
        raise ValueError("dt must be > 0")
    dev = device()
    bt = belief_tables(control_set, q, dev)
    beta_of, goal_of = hypothesis_arrays(space)
    prior = belief.log_weights
    if transition is not None:
        prior = np.asarray(transition(prior), dtype=float)
    H = len(beta_of)
    if H > _lib.GC_MAX_HYPOTHESES:
        raise NotImplementedError(f"at most {_lib.GC_MAX_HYPOTHESES} hypotheses per human")
    # np.array copies: the belief's log weights are read-only (immutable snapshots)
    up = lambda a, dt_: torch.as_tensor(np.array(a, dtype=dt_, order="C"), device=dev)  # noqa: E731
    d_qtable = None
    if bt.kind == _lib.GC_Q_TABLE:
        xy = np.tile(np.array([[z_t.x, z_t.y]], dtype=float), (H, 1))
        d_qtable = up(np.asarray(q.table(xy, goal_of, control_set), dtype=float), np.float64)
    # every per-call input in one host-to-device copy (a copy each costs most of a small
    # update's latency)
    (d_prior, d_off, d_beta, d_goal, d_obs, d_fb, d_status) = upload_packed(dev, [
        np.asarray(prior, dtype=np.float64), np.array([0, H], dtype=np.int32),
        np.asarray(beta_of, dtype=np.float64), np.asarray(goal_of, dtype=np.float64),
        np.array([z_t.x, z_t.y, z_next.x, z_next.y], dtype=np.float64),
        np.array([fallback_theta], dtype=np.float64), np.zeros(1, dtype=np.int32)])
    d_post = torch.empty_like(d_prior)
    tol = bt.snap_tol if snap_tol is None else float(snap_tol)
    launch_belief_update(bt, d_off, d_beta, d_goal, d_obs, d_fb, d_prior, d_post, d_status, dt,
                         tol if not math.isinf(tol) else math.inf, 0, 1, d_qtable=d_qtable)
    status = int(d_status.item())
    _lib.check(status, "update_belief")
    return JointBelief(d_post.cpu().numpy())
