"""MPPI local controller on the GPU (reference planners/mppi.py:1-250, agents.py:374-453).

``mppi_step`` keeps the reference signature and semantics: N perturbed Dubins rollouts
in fixed 256-rollout noise chunks keyed by (seed, MPPI_NOISE, chunk), quadratic goal
cost, control term, planning-interval term, collision penalty from the prediction
stack's blocked mask (collision field >= threshold, mppi.py:87-94), exponential weights
and the clamped weighted perturbation average.  The rollouts and reduction run in
``gc_mppi_step``; the blocked mask is computed on the device from a device-resident
stack (``gc_collision_field``), so a CycleEngine prediction feeds the controller with no
host round trip.

``noise="reference"`` draws the perturbations from the reference's own numpy streams
(bit-identical noise, so costs/controls match the reference to float64 rounding);
``noise="production"`` generates them in-register (Philox4x32-10 + Box-Muller).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _lib
from .agents import DEFAULT_ROBOT_LIMITS, RobotControl, RobotLimits, RobotState, wrap_angle  # noqa: F401
from .device import device, stream_handle
from .rng import MPPI_NOISE

ROLLOUT_CHUNK = 256


class DegenerateRolloutError(RuntimeError):
    """Every rollout cost came out non-finite."""


@dataclass(frozen=True)
class MppiConfig:
    horizon: int = 40
    rollouts: int = 512
    dt: float = 0.1
    temperature: float = 1.0
    perturbation_std: tuple = (0.5, 0.3)
    q_weights: tuple = (3.0, 3.0, 10.0, 0.0)
    q_final_weights: Optional[tuple] = None
    r_weights: tuple = (2.0, 1.0)
    collision_threshold: float = 0.1
    collision_penalty: float = 1000.0
    robot_radius: float = 0.25
    quadratic_control_cost: bool = False
    seed: int = 0
    limits: RobotLimits = field(default_factory=lambda: DEFAULT_ROBOT_LIMITS)

    def __post_init__(self):
        if self.horizon < 1 or self.rollouts < 1:
            raise ValueError("horizon and rollout count must be >= 1")
        if self.temperature <= 0:
            raise ValueError("temperature must be > 0")
        if any(s <= 0 for s in self.perturbation_std):
            raise ValueError("perturbation stds must be > 0")
        if self.dt <= 0:
            raise ValueError("dt must be > 0")

    @property
    def q_final(self) -> np.ndarray:
        if self.q_final_weights is not None:
            return np.asarray(self.q_final_weights, dtype=float)
        return np.asarray(self.q_weights, dtype=float) / 5.0


@dataclass
class MppiDiagnostics:
    best_cost: float
    mean_cost: float
    costs: np.ndarray
    weight_entropy: float


def mppi_weights(costs, temperature: float) -> np.ndarray:
    """Normalised exponential weights with the min-cost shift (host helper)."""
    costs = np.asarray(costs, dtype=float)
    finite = np.isfinite(costs)
    if not finite.any():
        raise DegenerateRolloutError("all rollout costs are non-finite")
    w = np.where(finite, np.exp(-(costs - costs[finite].min()) / temperature), 0.0)
    return w / w.sum()


def shift_nominal(controls: np.ndarray) -> np.ndarray:
    out = np.roll(controls, -1, axis=0)
    out[-1] = controls[-1]
    return out


def reference_noise(seed: int, rollouts: int, horizon: int, std) -> np.ndarray:
    """(N, K, 2) perturbations of the reference streams (mppi.py:208-211)."""
    std = np.asarray(std, dtype=float)
    out = np.empty((rollouts, horizon, 2))
    for index, start in enumerate(range(0, rollouts, ROLLOUT_CHUNK)):
        stop = min(start + ROLLOUT_CHUNK, rollouts)
        ss = np.random.SeedSequence(entropy=int(seed) & ((1 << 64) - 1),
                                    spawn_key=(MPPI_NOISE & 0xFFFFFFFF, index & 0xFFFFFFFF))
        gen = np.random.Generator(np.random.Philox(ss))
        out[start:stop] = gen.normal(0.0, 1.0, size=(stop - start, horizon, 2)) * std[None, None, :]
    return out


def blocked_mask_device(stack, cfg: MppiConfig) -> Optional[torch.Tensor]:
    """(L, H, W) uint8 blocked mask of a stack on the device (mppi.py:87-94)."""
    if stack is None or stack.steps == 0:
        return None
    from .occupancy import collision_layers_device
    _, blocked = collision_layers_device(stack.layers_device, stack.spec, cfg.robot_radius,
                                         threshold=cfg.collision_threshold, want_field=False)
    return blocked


def mppi_step(z: RobotState, nominal, goal: RobotState, stack, cfg: MppiConfig, seed: Optional[int] = None,
              workers: Optional[int] = None, base_time: float = 0.0, static_blocked=None, static_spec=None,
              noise: str = "reference", blocked: Optional[torch.Tensor] = None):
    """One control-sequence update from N perturbed rollouts (mppi.py:149-243), on the GPU.

    ``blocked`` may pass a precomputed device mask (e.g. CycleEngine.blocked[b]) for
    ``stack``; otherwise it is computed on the device from the stack."""
    seed = cfg.seed if seed is None else seed
    nominal = np.asarray(nominal, dtype=float)
    K, N = cfg.horizon, cfg.rollouts
    if nominal.shape != (K, 2):
        raise ValueError(f"nominal sequence must be ({K}, 2)")
    dev = device()
    up = lambda a_, t_: torch.as_tensor(np.array(a_, dtype=t_, order="C"), device=dev)  # noqa: E731
    if blocked is None:
        blocked = blocked_mask_device(stack, cfg)
    spec = stack.spec if stack is not None else static_spec
    layer_of = None
    if static_blocked is not None:
        sb = up(np.asarray(static_blocked, dtype=bool).astype(np.uint8), np.uint8)
        if blocked is None:
            if spec is None:
                raise ValueError("static_blocked without a stack needs static_spec")
            blocked = sb[None]
        else:
            blocked = blocked | sb[None]
    if blocked is not None:
        if stack is not None:
            layer_of = [stack.layer_index_for(base_time + (t + 1) * cfg.dt) for t in range(K)]
        else:
            layer_of = [0] * K
    a = _lib.MppiArgs()
    a.n_rollouts, a.horizon = N, K
    a.dt, a.temperature = cfg.dt, cfg.temperature
    a.std_a, a.std_w = float(cfg.perturbation_std[0]), float(cfg.perturbation_std[1])
    a.q[:] = [float(x) for x in cfg.q_weights]
    a.qf[:] = [float(x) for x in cfg.q_final]
    a.r[:] = [float(x) for x in cfg.r_weights]
    a.collision_penalty = cfg.collision_penalty
    a.quadratic_control_cost = int(cfg.quadratic_control_cost)
    a.a_max, a.omega_max, a.v_max = cfg.limits.a_max, cfg.limits.omega_max, cfg.limits.v_max
    a.z[:] = list(z.array)
    a.goal[:] = list(goal.array)
    d_nom = up(nominal, np.float64)
    a.d_nominal = d_nom.data_ptr()
    keep = [d_nom]
    if noise == "reference":
        d_noise = up(reference_noise(seed, N, K, cfg.perturbation_std), np.float64)
        a.d_noise, a.d_noise_out = d_noise.data_ptr(), None
    elif noise == "production":
        d_noise = torch.empty((N, K, 2), dtype=torch.float64, device=dev)
        a.d_noise, a.d_noise_out = None, d_noise.data_ptr()
        a.seed = int(seed) & ((1 << 64) - 1)
    else:
        raise ValueError("noise must be 'reference' or 'production'")
    keep.append(d_noise)
    if blocked is not None:
        blocked = blocked.contiguous()
        d_layer = up(layer_of, np.int32)
        keep.append(d_layer)
        a.d_blocked, a.d_layer_of = blocked.data_ptr(), d_layer.data_ptr()
        a.n_layers, a.grid_h, a.grid_w = blocked.shape[0], blocked.shape[1], blocked.shape[2]
        a.origin_x, a.origin_y, a.res = spec.origin[0], spec.origin[1], spec.resolution
    costs = torch.empty(N, dtype=torch.float64, device=dev)
    controls = torch.empty((K, 2), dtype=torch.float64, device=dev)
    weights = torch.empty(N, dtype=torch.float64, device=dev)
    diag = torch.zeros(3, dtype=torch.float64, device=dev)
    a.d_costs, a.d_controls, a.d_weights, a.d_diag = (costs.data_ptr(), controls.data_ptr(),
                                                      weights.data_ptr(), diag.data_ptr())
    _lib.check(_lib.lib().gc_mppi_step(ctypes.byref(a), stream_handle()), "mppi_step")
    dg = diag.cpu().numpy()
    c = costs.cpu().numpy()
    if not np.isfinite(c).any():
        raise DegenerateRolloutError("all rollout costs are non-finite")
    return controls.cpu().numpy(), MppiDiagnostics(float(dg[0]), float(dg[1]), c, float(dg[2]))
