"""CPU: host-side utilities of the drop-in API (no device work)."""

import json
import math

import numpy as np

import golden_io
from paper_2603_01122_b200 import agents, gridio, rng
from paper_2603_01122_b200.occupancy import GridSpec, OccupancyGrid


def test_rng_stream_is_the_reference_stream():
    """rng.stream(seed, *path) (rng.py:27-31) draws the golden Philox values."""
    z = golden_io.load("philox.npz")
    meta = json.loads(str(z["meta"]))
    for i, (seed, path) in enumerate(zip(meta["seeds"], meta["paths"])):
        np.testing.assert_array_equal(rng.stream(seed, *path).random(12), z["f64"][i])
        np.testing.assert_array_equal(rng.stream(seed, *path).random(24, dtype=np.float32), z["f32"][i])
        assert rng.derive_seed(seed, *path) == int(meta["derived"][i])


def test_robot_step_clamps_and_matches_batch():
    lim = agents.RobotLimits(v_max=1.1, a_max=1.0, omega_max=1.0)
    z = agents.RobotState(1.0, 2.0, 1.05, math.pi - 0.01)
    s = agents.robot_step(z, agents.RobotControl(5.0, 3.0), 0.1, lim)
    assert s.v == 1.1  # a clamped to 1.0, then v clamped to v_max
    assert abs(s.theta - (-math.pi + 0.09)) < 1e-12  # omega clamped to 1.0, heading wrapped
    assert s.x == 1.0 + 1.05 * math.cos(math.pi - 0.01) * 0.1  # pre-step speed and heading
    r = np.random.default_rng(1)
    states = np.column_stack([r.uniform(-5, 5, 50), r.uniform(-5, 5, 50), r.uniform(0, 1.1, 50),
                              r.uniform(-math.pi, math.pi, 50)])
    ctrl = r.uniform(-3, 3, (50, 2))
    out = agents.robot_step_batch(states, ctrl, 0.1, lim)
    for i in range(50):
        e = agents.robot_step(agents.RobotState(*states[i]), agents.RobotControl(*ctrl[i]), 0.1, lim)
        np.testing.assert_allclose(out[i], [e.x, e.y, e.v, e.theta], rtol=0, atol=1e-15)


def test_grid_csv_round_trip_is_exact(tmp_path):
    spec = GridSpec(7, 5, 0.1)
    vals = np.random.default_rng(2).dirichlet(np.ones(35)).reshape(5, 7)
    g = OccupancyGrid(spec, vals)
    p = tmp_path / "g.csv"
    gridio.grid_to_csv(g, p)
    back = gridio.grid_from_csv(p, spec)
    np.testing.assert_array_equal(back.values, vals)
    assert p.read_text().splitlines()[0].count(",") == 6  # row 0 = lowest y, W columns
