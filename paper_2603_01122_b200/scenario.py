"""Synthetic pedestrian scenes of the benchmark shapes (BASELINE.json configs).

Common inputs: res 0.1 m, origin (0, 0); ControlSet.grid(4, 24, 1.4) (m = 96);
q_goal_progress(0.5); RationalitySet.log_spaced(5); goals on a circle of radius 0.35 x room
around each human's start (the cli.py:176-179 bench puts them 3.5 m from the
centre of its 10 m room) -- cfg1 3.5 m, cfg2 7 m, cfg3/cfg4 14 m; ``goal_radius`` overrides
it (e.g. 3.5 m at every config, the round-1 scene); belief = posterior after
10 observations (dt 0.1 s) of a Boltzmann walker with beta = 10 heading to goal 0.
Tracks are generated on the host before any timing starts.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .agents import ControlSet, GoalSet, HumanState, RationalitySet, boltzmann_policy, human_step, q_goal_progress
from .belief import HypothesisSpace
from .occupancy import GridSpec

CONFIGS = {
    # name: (humans, goals, n, steps, dt, grid cells, room m)
    "cfg1": dict(humans=1, goals=2, n=1024, steps=20, dt=0.1, cells=100),
    "cfg2": dict(humans=1, goals=4, n=65536, steps=100, dt=0.02, cells=200),
    "cfg3": dict(humans=8, goals=4, n=262144, steps=250, dt=0.02, cells=400),
    "cfg4_rank": dict(humans=8, goals=4, n=1 << 20, steps=500, dt=0.02, cells=400),
}


@dataclass
class Scene:
    name: str
    control_set: ControlSet
    q: object
    spaces: list
    spec: GridSpec
    starts: np.ndarray                 # (H, 2)
    n: int
    steps: int
    dt: float
    sigma: float = 0.1
    log_weights: list = field(default_factory=list)
    prev_xy: np.ndarray = None         # observation preceding the first cycle
    track: np.ndarray = None           # (cycles, H, 2) future observations


def _starts(h: int, room: float) -> np.ndarray:
    if h == 1:
        return np.array([[room / 2, room / 2]])
    cols = min(h, 4)
    rows = int(math.ceil(h / cols))
    xs = (np.arange(cols) + 0.5) * room / cols
    ys = (np.arange(rows) + 0.5) * room / rows
    pts = np.array([[x, y] for y in ys for x in xs])[:h]
    return pts


def make_scene(name: str = "cfg3", cycles: int = 64, seed: int = 0, humans: int | None = None,
               human_offset: int = 0, goal_radius: float | None = None) -> Scene:
    """Build the scene; ``humans``/``human_offset`` select a shard (multi-GPU weak scaling)."""
    c = dict(CONFIGS[name])
    H = humans if humans is not None else c["humans"]
    room = c["cells"] * 0.1
    gr = 0.35 * room if goal_radius is None else float(goal_radius)
    spec = GridSpec(c["cells"], c["cells"], 0.1)
    cs = ControlSet.grid(4, 24, 1.4)
    q = q_goal_progress(0.5)
    rs = RationalitySet.log_spaced(5)
    base = _starts(max(H, c["humans"]), room)
    rng = np.random.default_rng(seed + 7919 * human_offset)
    starts, spaces, goals0 = [], [], []
    for i in range(H):
        s = base[(i + human_offset) % len(base)] + rng.uniform(-0.5, 0.5, 2)
        ang = 2.0 * np.pi * np.arange(c["goals"]) / c["goals"] + rng.uniform(0, np.pi / 2)
        goals = np.stack([s[0] + gr * np.cos(ang), s[1] + gr * np.sin(ang)], axis=1)
        spaces.append(HypothesisSpace(rs, GoalSet(goals)))
        starts.append(s)
        goals0.append(goals[0])
    starts = np.array(starts)
    # Boltzmann walker (beta = 10 toward goal 0), 10 warm-up observations + the track
    n_obs = 11 + cycles
    track = np.zeros((n_obs, H, 2))
    track[0] = starts
    for i in range(H):
        z = HumanState(*starts[i])
        for k in range(1, n_obs):
            p = boltzmann_policy(z, 10.0, goals0[i], cs, q)
            j = min(int(np.searchsorted(np.cumsum(p), rng.random(), side="right")), len(cs) - 1)
            z = human_step(z, cs[j], 0.1)
            track[k, i] = (z.x, z.y)
    sc = Scene(name, cs, q, spaces, spec, track[10], c["n"], c["steps"], c["dt"])
    sc.goal_radius = gr
    sc.warmup_track = track[:11]
    sc.prev_xy = track[10]
    sc.track = track[11:]
    return sc
