"""CPU: pin the oracle restatement against the golden vectors of the live reference.

The fixtures (tests/golden/*.npz) were produced by oracle/gen_golden.py from
/root/reference/pkg/src; these tests need neither the reference nor a GPU.
"""

import json
import math

import numpy as np
import pytest

import golden_io
from oracle import cstep, model, philox
from oracle import predict as OP


def test_philox_streams_match_reference():
    z = golden_io.load("philox.npz")
    meta = json.loads(str(z["meta"]))
    for i, (seed, path) in enumerate(zip(meta["seeds"], meta["paths"])):
        np.testing.assert_array_equal(philox.stream_random_f32(seed, path, 24), z["f32"][i])
        np.testing.assert_array_equal(philox.stream_random_f64(seed, path, 12), z["f64"][i])
        assert philox.derive_seed(seed, *path) == int(meta["derived"][i])


def test_numpy_exp_restatement_bit_exact():
    z = golden_io.load("exp.npz")
    y = cstep.exp_np_f32(z["x"])
    assert np.array_equal(y.view(np.uint32), z["y"].view(np.uint32))


@pytest.mark.parametrize("name", golden_io.predict_case_names())
def test_tables_match_reference_displacements(name):
    c = golden_io.PredictCase(name)
    np.testing.assert_array_equal(np.stack([c.dispx, c.dispy], 1), c.ref_disp)
    m = c.meta
    q = m["q"]
    tb = model.make_tables(m["v"], m["theta"], c.dt,
                           model.QSpec(q["family"], q["tau"], q["w_v"], q["w_th"], q["v_threshold"]))
    for k in ("sx", "sy", "at", "pen", "dispx", "dispy", "keep"):
        np.testing.assert_array_equal(getattr(tb, k), getattr(c, k))


@pytest.mark.parametrize("name", golden_io.predict_case_names())
def test_oracle_predict_bit_exact(name):
    c = golden_io.PredictCase(name)
    if c.n * c.steps > 400_000:
        pytest.skip("large case covered by test_oracle_predict_positions")
    W, H, res, org = c.grid
    out = OP.predict(c.z0, c.log_w, c.n, c.steps, c.dt, c.sigma, c.seed, c.tables(),
                     c.beta_of, c.goal_xy_of, OP.Grid(W, H, res, org), prefix=c.prefix, keep_xy=True)
    np.testing.assert_array_equal(out["hyp"], c.hyp)
    np.testing.assert_array_equal(out["counts"], c.counts())
    np.testing.assert_array_equal(out["xy"][0], c.xy_first)
    np.testing.assert_array_equal(out["xy"][-1], c.xy_last)
    np.testing.assert_array_equal(out["layers"][c.layer_steps], c.layers)


def test_oracle_predict_positions_cfg2():
    c = golden_io.PredictCase("cfg2_t30")
    W, H, res, org = c.grid
    out = OP.predict(c.z0, c.log_w, c.n, c.steps, c.dt, c.sigma, c.seed, c.tables(),
                     c.beta_of, c.goal_xy_of, OP.Grid(W, H, res, org), prefix=c.prefix, keep_xy=True)
    np.testing.assert_array_equal(out["counts"], c.counts())
    np.testing.assert_array_equal(out["xy"][-1], c.xy_last)


def test_unsmoothed_layers_are_counts_over_n():
    c = golden_io.PredictCase("cfg1_s0")
    cnt = c.counts()
    np.testing.assert_array_equal(cnt[c.layer_steps].astype(float) / c.n, c.layers)


def test_smoothing_restatements():
    z = golden_io.load("smooth.npz")
    items = json.loads(str(z["meta"]))
    off = 0
    for w, h, res, sig in items:
        x = z["x"][off:off + w * h].reshape(h, w)
        y = z["y"][off:off + w * h].reshape(h, w)
        off += w * h
        g = OP.Grid(w, h, res)
        np.testing.assert_array_equal(OP.smooth_dense(x, g, sig), y)
        np.testing.assert_allclose(OP.smooth_banded(x, g, sig), y, rtol=0, atol=1e-15)


def test_belief_chains():
    z = golden_io.load("belief.npz")
    meta = json.loads(str(z["meta"]))
    v, th = model.control_grid(4, 24, 1.4)
    beta_of, goal_xy_of = model.hypothesis_tables(meta["betas"], meta["goals"])
    for chain in meta["chains"]:
        qd = chain["q"]
        qs = model.QSpec(qd["family"], qd["tau"], qd["w_v"], qd["w_th"], qd["v_threshold"])
        for row in chain["rows"]:
            prior = np.array(row["prior"])
            tol = None
            if row["status"] == 1:
                with pytest.raises(ValueError):
                    OP.belief_update(prior, row["z"], row["zn"], meta["dt"], v, th, qs,
                                     beta_of, goal_xy_of, row["heading"])
                tol = math.inf
            post, _ = OP.belief_update(prior, row["z"], row["zn"], meta["dt"], v, th, qs,
                                       beta_of, goal_xy_of, row["heading"], snap_tol=tol)
            ref = np.array(row["post"])
            fin = np.isfinite(ref)
            np.testing.assert_array_equal(np.isfinite(post), fin)
            np.testing.assert_allclose(post[fin], ref[fin], rtol=1e-12, atol=1e-12)


def test_multi_union_and_time_union():
    z = golden_io.load("multi.npz")
    meta = json.loads(str(z["meta"]))
    v, th = model.control_grid(4, 24, 1.4)
    tb = model.make_tables(v, th, meta["dt"], model.QSpec())
    stacks = []
    for i, hm in enumerate(meta["humans"]):
        beta_of, goal_xy_of = model.hypothesis_tables(np.geomspace(0.1, 10, 5), hm["goals"])
        out = OP.predict(hm["start"], np.array(hm["log_w"]), meta["n"], meta["steps"], meta["dt"],
                         meta["sigma"], int(meta["seed"]), tb, beta_of, goal_xy_of,
                         OP.Grid(100, 100, 0.1), prefix=(2, i))
        stacks.append(out["layers"])
    u = OP.union_max(stacks)
    np.testing.assert_array_equal(u, z["union"])
    np.testing.assert_array_equal(OP.time_union(u), z["time_union"])
    ind = OP.union_independent(stacks)
    np.testing.assert_array_equal(ind, z["independent"])
    np.testing.assert_array_equal(OP.time_union(ind), z["independent_tu"])


@pytest.mark.parametrize("name", ["cfg1_s0", "cfg1_s01", "ragged_w", "masked", "qdefault"])
def test_cpu_baseline_port_matches_reference(name):
    """The timed CPU baseline (oracle/port.py) is the reference computation."""
    from oracle import port
    c = golden_io.PredictCase(name)
    W, H, res, org = c.grid
    layers = port.predict(c.z0, c.log_w, c.n, c.steps, c.dt, c.sigma, c.seed, c.tables(),
                          c.beta_of, c.goal_xy_of, OP.Grid(W, H, res, org), prefix=c.prefix, workers=4)
    np.testing.assert_array_equal(layers[c.layer_steps], c.layers)


@pytest.mark.parametrize("name", golden_io.naive_case_names())
def test_oracle_predict_naive_matches_reference(name):
    """float64 per-particle loop (prediction.py:258-300): layers identical to the reference's."""
    c = golden_io.NaiveCase(name)
    W, H, res, org = c.grid
    out = OP.predict_naive(c.z0, c.log_w, c.n, c.steps, c.dt, c.sigma, c.seed, c.meta["v"], c.meta["theta"],
                           c.qspec(), c.beta_of, c.goal_xy_of, OP.Grid(W, H, res, org))
    if c.sigma == 0:
        np.testing.assert_array_equal(out["layers"], c.layers)
    else:
        np.testing.assert_allclose(out["layers"], c.layers, rtol=0, atol=1e-15)


def _oracle_sparse_counts(z0, log_w, n, steps, seed, prefix, tables, beta_of, goal_xy_of, grid):
    """The oracle cycle (C step + pinned streams) with sparse per-step counts (t, iy, ix)."""
    hyp = OP.sample_hypotheses(log_w, n, seed, prefix)
    xy = np.tile(np.array(z0, dtype=np.float32), (n, 1))
    b32, g32 = np.asarray(beta_of, np.float32), np.asarray(goal_xy_of, np.float32)
    idx, val = [], []
    for t in range(1, steps + 1):
        xy = cstep.propagate(xy, hyp, b32, g32, tables, OP.step_uniforms(seed, prefix, t, n))
        cells, cnt = np.unique(cstep.cells(xy, grid), return_counts=True)
        idx.append(np.stack([np.full(len(cells), t - 1), cells // grid.width, cells % grid.width], 1))
        val.append(cnt)
    return hyp, xy, np.concatenate(idx), np.concatenate(val)


def test_oracle_long_horizon_cfg4_case():
    """long_cfg4.npz (T = 500, the GPU's global-histogram path) reproduced by the oracle."""
    z = golden_io.load("long_cfg4.npz")
    m = json.loads(str(z["meta"]))
    tb = model.Tables(np.asarray(model.control_grid(4, 24, 1.4)[0]), np.asarray(model.control_grid(4, 24, 1.4)[1]),
                      z["sx"], z["sy"], z["at"], z["pen"], z["dispx"], z["dispy"], z["keep"], int(z["q_kind"]))
    beta_of, goal_xy_of = model.hypothesis_tables(m["betas"], m["goals"])
    hyp, xy, idx, val = _oracle_sparse_counts(m["z0"], z["log_w"], m["n"], m["steps"], m["seed"], tuple(m["prefix"]),
                                              tb, beta_of, goal_xy_of, OP.Grid(400, 400, 0.1))
    np.testing.assert_array_equal(hyp, z["hyp"])
    np.testing.assert_array_equal(xy, z["xy_last"])
    np.testing.assert_array_equal(idx, z["count_idx"])
    np.testing.assert_array_equal(val, z["count_val"])


def test_oracle_cfg3_scene_human0():
    """cfg3_cycle.npz human 0 (262,144 particles of the bench scene; the first 6 of its 25
    steps, to keep the CPU suite short -- the GPU test checks all 25) by the oracle."""
    import hashlib
    z = golden_io.load("cfg3_cycle.npz")
    m = json.loads(str(z["meta"]))
    hm = m["humans"][0]
    v, th = model.control_grid(4, 24, 1.4)
    tb = model.make_tables(v, th, m["dt"], model.QSpec("goal_progress", 0.5, 0.0, 0.0,
                                                       0.5 if hm["stationary"] else None))
    beta_of, goal_xy_of = model.hypothesis_tables(m["betas"], hm["goals"])
    T = 6
    hyp, xy, idx, val = _oracle_sparse_counts(hm["start"], np.array(hm["log_w"]), m["n"], T, int(m["seed"]),
                                              (2, 0), tb, beta_of, goal_xy_of, OP.Grid(400, 400, 0.1))
    assert hashlib.sha256(hyp.astype(np.int32).tobytes()).hexdigest() == hm["hyp_sha256"]
    sel = z["count_idx_0"][:, 0] < T
    np.testing.assert_array_equal(idx, z["count_idx_0"][sel])
    np.testing.assert_array_equal(val, z["count_val_0"][sel])


def test_reference_drawn_uniforms_match_oracle_streams():
    """uniforms_cfg1.npz (drawn by gridcast.rng) == the oracle's stream restatement."""
    zu = golden_io.load("uniforms_cfg1.npz")
    c = golden_io.PredictCase("cfg1_s0")
    np.testing.assert_array_equal(philox.stream_random_f64(c.seed, tuple(c.prefix) + (0,), c.n), zu["hyp_u"])
    for t in range(1, c.steps + 1):
        np.testing.assert_array_equal(OP.step_uniforms(c.seed, c.prefix, t, c.n), zu["step_u"][t - 1])
    np.testing.assert_array_equal(OP.sample_hypotheses(c.log_w, c.n, c.seed, c.prefix), c.hyp)
