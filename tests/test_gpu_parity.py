"""GPU parity: the CUDA path (through the C ABI) vs the reference's golden vectors and
the oracle restatement.  Reference RNG mode must reproduce counts bit-for-bit."""

import json
import math

import numpy as np
import pytest
import torch

import golden_io

pytestmark = pytest.mark.gpu

import paper_2603_01122_b200 as G  # noqa: E402
from paper_2603_01122_b200 import prediction as PR  # noqa: E402


def _objects(case):
    m = case.meta
    cs = G.ControlSet([G.ControlAction(float(v), float(t)) for v, t in zip(m["v"], m["theta"])])
    space = G.HypothesisSpace(G.RationalitySet(tuple(m["betas"])), G.GoalSet(np.array(m["goals"])))
    qd = m["q"]
    if qd["family"] == "goal_progress":
        q = G.q_goal_progress(qd["tau"], (qd["w_v"], qd["w_th"]))
    else:
        q = G.q_default((qd["w_v"], qd["w_th"]))
    if qd["v_threshold"] is not None:
        q = G.mask_stationary(q, cs, qd["v_threshold"])
    W, H, res, org = case.grid
    spec = G.GridSpec(W, H, res, org)
    return cs, space, q, spec


def full_counts(out, jobs, spec, steps):
    """Expand the windowed count buffer into (humans, T, H, W)."""
    geo = out["geometry"]
    c = out["counts"].cpu().numpy().view(np.uint32)
    res = np.zeros((len(jobs), steps, spec.height, spec.width), dtype=np.int64)
    for h, j in enumerate(jobs):
        for t in range(steps):
            x0, y0, w, hh = geo.window((np.float32(j.z0.x), np.float32(j.z0.y)), t)
            base = h * geo.human_stride + geo.step_off[t]
            res[h, t, y0:y0 + hh, x0:x0 + w] = c[base:base + w * hh].reshape(hh, w)
    return res


@pytest.mark.parametrize("name", golden_io.predict_case_names())
def test_predict_reference_mode_bit_exact(name):
    case = golden_io.PredictCase(name)
    cs, space, q, spec = _objects(case)
    dev = torch.device("cuda")
    tab = PR.action_tables(cs, q, case.dt, dev)
    # tables computed on this host equal the reference's (else the box's numpy differs)
    np.testing.assert_array_equal(tab.disp_np, case.ref_disp)
    bo, go = space.beta_of, space.goal_xy_of
    job = PR.HumanJob(G.HumanState(*case.z0), case.log_w, bo, go, case.seed, case.prefix, 0)
    out = PR.run_predict([job], [tab], case.n, case.steps, case.dt, case.sigma, spec, "reference",
                         want_hyp=True, want_xy=True)
    np.testing.assert_array_equal(out["hyp"][0].cpu().numpy(), case.hyp)
    np.testing.assert_array_equal(out["xy"][0].cpu().numpy(), case.xy_last)
    counts = full_counts(out, [job], spec, case.steps)[0]
    np.testing.assert_array_equal(counts, case.counts())
    layers = out["layers"][0].cpu().numpy()
    got = layers[case.layer_steps]
    if case.sigma == 0:
        np.testing.assert_array_equal(got, case.layers)
    else:
        np.testing.assert_allclose(got, case.layers, rtol=0, atol=1e-15)
    np.testing.assert_allclose(layers.sum(axis=(1, 2)), case.layer_sums, rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", ["cfg1_s0", "ragged_w", "masked", "qdefault", "lattice"])
def test_public_predict_and_helpers(name):
    case = golden_io.PredictCase(name)
    cs, space, q, spec = _objects(case)
    b = G.JointBelief(case.log_w)
    cfg = G.PredictionConfig(n=case.n, steps=case.steps, dt=case.dt, smoothing_sigma=case.sigma,
                             seed=case.seed)
    st = G.predict(G.HumanState(*case.z0), b, cfg, cs, q, space, spec, prefix=case.prefix)
    if case.sigma == 0:
        np.testing.assert_array_equal(st.layers[case.layer_steps], case.layers)
    else:
        np.testing.assert_allclose(st.layers[case.layer_steps], case.layers, rtol=0, atol=1e-15)
    hyp = G.sample_hypotheses(b, case.n, case.seed, prefix=case.prefix)
    np.testing.assert_array_equal(hyp, case.hyp)
    batch = G.ParticleBatch.duplicated(G.HumanState(*case.z0), hyp)
    batch = G.propagate_step(batch, cs, q, space, case.dt, case.seed, step=1, prefix=case.prefix)
    np.testing.assert_array_equal(batch.xy, case.xy_first)


def test_belief_update_chains():
    z = golden_io.load("belief.npz")
    meta = json.loads(str(z["meta"]))
    cs = G.ControlSet.grid(4, 24, 1.4)
    space = G.HypothesisSpace(G.RationalitySet(tuple(meta["betas"])), G.GoalSet(np.array(meta["goals"])))
    worst = 0.0
    for chain in meta["chains"]:
        qd = chain["q"]
        if qd["family"] == "goal_progress":
            q = G.q_goal_progress(qd["tau"], (qd["w_v"], qd["w_th"]))
        else:
            q = G.q_default((qd["w_v"], qd["w_th"]))
        if qd["v_threshold"] is not None:
            q = G.mask_stationary(q, cs, qd["v_threshold"])
        for row in chain["rows"]:
            prior = G.JointBelief(np.array(row["prior"]))
            zt, zn = G.HumanState(*row["z"]), G.HumanState(*row["zn"])
            tol = None
            if row["status"] == 1:
                with pytest.raises(G.ControlSnapMismatch):
                    G.update_belief(prior, zt, zn, meta["dt"], cs, q, space, fallback_theta=row["heading"])
                tol = math.inf
            post = G.update_belief(prior, zt, zn, meta["dt"], cs, q, space, fallback_theta=row["heading"],
                                   snap_tol=tol)
            ref = np.array(row["post"])
            fin = np.isfinite(ref)
            np.testing.assert_array_equal(np.isfinite(post.log_weights), fin)
            pr, pg = np.exp(ref[fin]), np.exp(post.log_weights[fin])
            rel = np.max(np.abs(pg - pr) / np.maximum(pr, 1e-300))
            worst = max(worst, rel)
    assert worst < 1e-5, worst  # north-star bound; observed ~1e-13


def test_multi_union_time_union():
    z = golden_io.load("multi.npz")
    meta = json.loads(str(z["meta"]))
    cs = G.ControlSet.grid(4, 24, 1.4)
    q = G.q_goal_progress(0.5)
    spec = G.GridSpec(100, 100, 0.1)
    dev = torch.device("cuda")
    tab = PR.action_tables(cs, q, meta["dt"], dev)
    jobs = []
    for i, hm in enumerate(meta["humans"]):
        space = G.HypothesisSpace(G.RationalitySet.log_spaced(5), G.GoalSet(np.array(hm["goals"])))
        jobs.append(PR.HumanJob(G.HumanState(*hm["start"]), np.array(hm["log_w"]), space.beta_of,
                                space.goal_xy_of, int(meta["seed"]), (2, i), 0))
    out = PR.run_predict(jobs, [tab], meta["n"], meta["steps"], meta["dt"], meta["sigma"], spec,
                         "reference", per_human_layers=False, union64=True)
    np.testing.assert_allclose(out["union64"].cpu().numpy(), z["union"], rtol=0, atol=1e-15)
    out = PR.run_predict(jobs, [tab], meta["n"], meta["steps"], meta["dt"], meta["sigma"], spec,
                         "reference", per_human_layers=False, union64=True, union32=True, time_union=True)
    np.testing.assert_allclose(out["union64"].cpu().numpy(), z["time_union"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(out["union32"].cpu().numpy(), z["time_union"].astype(np.float32), rtol=0,
                               atol=1e-7)
    # the "independent" union 1 - prod(1 - p) (occupancy.py:180-184), ordered over humans
    out = PR.run_predict(jobs, [tab], meta["n"], meta["steps"], meta["dt"], meta["sigma"], spec,
                         "reference", per_human_layers=True, union64=True, union_mode="independent")
    np.testing.assert_allclose(out["union64"].cpu().numpy(), z["independent"], rtol=0, atol=1e-15)
    host = 1.0 - np.prod(1.0 - np.clip(out["layers"].cpu().numpy(), 0, 1), axis=0)
    np.testing.assert_array_equal(out["union64"].cpu().numpy(), host)
    out = PR.run_predict(jobs, [tab], meta["n"], meta["steps"], meta["dt"], meta["sigma"], spec,
                         "reference", per_human_layers=False, union64=True, union32=True, time_union=True,
                         union_mode="independent")
    np.testing.assert_allclose(out["union64"].cpu().numpy(), z["independent_tu"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(out["union32"].cpu().numpy(), z["independent_tu"].astype(np.float32), rtol=0,
                               atol=1e-7)
    assert "layers" not in out


def test_predict_multi_semantics():
    case = golden_io.PredictCase("lattice")
    cs, space, q, spec = _objects(case)
    b = G.init_belief(space)
    cfg = G.PredictionConfig(n=2048, steps=3, dt=1.0, smoothing_sigma=0.0, seed=21)
    z0 = G.HumanState(4.5, 4.5)
    merged = G.predict_multi([(z0, b)], cfg, cs, q, space, spec)
    single = G.predict(z0, b, cfg, cs, q, space, spec)
    np.testing.assert_array_equal(merged.layers, single.layers)
    merged2 = G.predict_multi([(z0, b), (z0, b)], cfg, cs, q, space, spec)
    np.testing.assert_array_equal(merged2.layers, single.layers)


def test_smoothing_and_emplace_helpers():
    z = golden_io.load("smooth.npz")
    items = json.loads(str(z["meta"]))
    off = 0
    for w, h, res, sig in items:
        x = z["x"][off:off + w * h].reshape(h, w)
        y = z["y"][off:off + w * h].reshape(h, w)
        off += w * h
        np.testing.assert_allclose(G.smooth_values(x, G.GridSpec(w, h, res), sig), y, rtol=0, atol=1e-15)
    spec = G.GridSpec(4, 4, 1.0)
    g = G.emplace(G.ParticleBatch(np.array([[-3.0, 9.0], [2.5, 2.5]], np.float32), np.zeros(2, np.int32)), spec)
    assert g.at(0, 3) == 0.5 and g.at(2, 2) == 0.5


def test_collision_field_bit_exact():
    """f2 row: collision_field (occupancy.py:222-239) on the GPU == the reference bit-for-bit,
    from float64 and from float32 layers; thresholded blocked mask."""
    from paper_2603_01122_b200.occupancy import collision_layers_device
    z = golden_io.load("collision.npz")
    items = json.loads(str(z["meta"]))
    off = 0
    for w, h, res, rad, _ in items:
        x = z["x"][off:off + w * h].reshape(h, w)
        y = z["y"][off:off + w * h].reshape(h, w)
        off += w * h
        spec = G.GridSpec(w, h, res)
        got = G.occupancy.collision_field(G.OccupancyGrid(spec, x), rad)
        np.testing.assert_array_equal(got, y)
        d32 = torch.as_tensor(x.astype(np.float32)[None], device="cuda")
        f, blk = collision_layers_device(d32, spec, rad, threshold=0.02)
        ref32 = G.occupancy.collision_field(G.OccupancyGrid(spec, x.astype(np.float32).astype(float)), rad)
        np.testing.assert_array_equal(f[0].cpu().numpy(), ref32)
        np.testing.assert_array_equal(blk[0].cpu().numpy(), (ref32 >= 0.02).astype(np.uint8))


def test_gcst_save_from_device_stack(tmp_path):
    from paper_2603_01122_b200 import gridio
    spec = G.GridSpec(33, 17, 0.1)
    r = np.random.default_rng(1)
    host = r.random((40, 17, 33))
    dev32 = torch.as_tensor(host.astype(np.float32), device="cuda")
    st = PR.PredictionStack(spec, dev32, 1.0, 0.02)
    gridio.save_stack(st, tmp_path / "a.grd", chunk_layers=7)
    back = gridio.load_stack(tmp_path / "a.grd")
    np.testing.assert_array_equal(back.layers, host.astype(np.float32).astype(np.float64))


def test_exact_predict_gpu_matches_reference():
    """f4 row: GPU exact enumeration vs the reference's exact_predict (lattice + a grid
    control set with goal-progress, stationary-masked and q_default utilities)."""
    z = golden_io.load("exact.npz")
    case = golden_io.PredictCase("lattice")
    cs, space, q, spec = _objects(case)
    st = G.exact_predict(G.HumanState(4.5, 4.5), G.JointBelief(z["log_w"]), 3, 1.0, cs, q, space, spec)
    np.testing.assert_allclose(st.layers, z["layers"], rtol=0, atol=1e-14)
    with pytest.raises(PR.EnumerationCapExceeded):
        G.exact_predict(G.HumanState(4.5, 4.5), G.JointBelief(z["log_w"]), 2, 1.0, cs, q, space, spec, max_table=10)
    zg = golden_io.load("exact_grid.npz")
    cs2 = G.ControlSet([G.ControlAction(float(a), float(t)) for a, t in zip(zg["v"], zg["theta"])])
    space2 = G.HypothesisSpace(G.RationalitySet((0.5, 3.0)), G.GoalSet(np.array([[2.5, 1.0], [0.4, 2.0]])))
    spec2 = G.GridSpec(30, 24, 0.1)
    b2 = G.JointBelief(zg["log_w"])
    for tag, q2 in (("gp", G.q_goal_progress(0.5)), ("mask", G.mask_stationary(G.q_goal_progress(0.5), cs2, 0.7)),
                    ("def", G.q_default((0.5, 0.2)))):
        st2 = G.exact_predict(G.HumanState(1.43, 1.17), b2, 6, 0.2, cs2, q2, space2, spec2)
        np.testing.assert_allclose(st2.layers, zg[tag], rtol=0, atol=1e-13)
        np.testing.assert_allclose(st2.layers.sum(axis=(1, 2)), 1.0, atol=1e-12)


def test_exact_predict_beyond_reference_cap():
    """The HBM-resident tables enumerate a cfg1-sized instance (100x100 cells x 96 actions
    x 10 hypotheses = 9.6e6 entries, 4.8x the reference's 2e6 cap)."""
    cs = G.ControlSet.grid(4, 24, 1.4)
    space = G.HypothesisSpace(G.RationalitySet.log_spaced(5), G.GoalSet(np.array([[8.5, 5.0], [1.5, 7.0]])))
    spec = G.GridSpec(100, 100, 0.1)
    st = G.exact_predict(G.HumanState(5.05, 5.05), G.init_belief(space), 10, 0.1, cs, G.q_goal_progress(0.5),
                         space, spec, max_table=None)
    np.testing.assert_allclose(st.layers.sum(axis=(1, 2)), 1.0, atol=1e-12)
    assert (st.layers >= 0).all()


def test_engine_cycle_matches_reference_mode_and_blocked_mask():
    """CycleEngine (sim.py:455-504 pattern) in reference mode: its fused union equals the
    per-human reference-mode union of the same humans/prefixes/seed, its posteriors equal
    update_belief, and its blocked mask equals collision_field(union) >= threshold."""
    from paper_2603_01122_b200.engine import CycleEngine, EngineConfig
    from paper_2603_01122_b200.scenario import make_scene
    sc = make_scene("cfg1", cycles=3, humans=3)
    cfg = EngineConfig(n=1500, steps=8, dt=0.1, smoothing_sigma=0.1, seed=5, mode="reference",
                       union_dtype="float64", robot_radius=0.25, collision_threshold=0.05)
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, cfg)
    eng.prime(sc.prev_xy)
    eng.stage(sc.track[0], buf=0)
    eng.run_cycle(buf=0)
    torch.cuda.synchronize()
    from paper_2603_01122_b200 import rng
    seed = rng.derive_seed(5, 7, 0)
    layers = []
    for i, sp in enumerate(sc.spaces):
        prior = G.init_belief(sp)
        post = G.update_belief(prior, G.HumanState(*sc.prev_xy[i]), G.HumanState(*sc.track[0][i]), 0.1,
                               sc.control_set, sc.q, sp, snap_tol=math.inf)
        np.testing.assert_allclose(np.exp(eng.posterior(i)), post.probs(), rtol=1e-12, atol=1e-300)
        moved = np.hypot(*(sc.track[0][i] - sc.prev_xy[i])) / 0.1
        q = G.mask_stationary(sc.q, sc.control_set, 0.5) if moved < 0.05 else sc.q
        pc = G.PredictionConfig(n=1500, steps=8, dt=0.1, smoothing_sigma=0.1, seed=seed)
        layers.append(G.predict(G.HumanState(*sc.track[0][i]), post, pc, sc.control_set, q, sp, sc.spec,
                                prefix=(2, i)).layers)
    union = np.maximum.reduce(layers)
    np.testing.assert_allclose(eng.unions[0].cpu().numpy(), union, rtol=0, atol=1e-15)
    from paper_2603_01122_b200.occupancy import collision_layers_device
    f, _ = collision_layers_device(torch.as_tensor(union, device="cuda"), sc.spec, 0.25)
    np.testing.assert_array_equal(eng.blocked[0].cpu().numpy(), (f.cpu().numpy() >= 0.05).astype(np.uint8))
    eng.reset_belief(1)
    np.testing.assert_allclose(np.exp(eng.posterior(1)), 1.0 / sc.spaces[1].size)


@pytest.mark.parametrize("chunks", [1, 3])
def test_engine_independent_union_and_partials(chunks):
    """EngineConfig(union_mode="independent"): the union is 1 - prod(1 - p) of the engine's
    own per-human layers in human order (+ time union), chunked or not; the union_partial
    miss product completed by complement_layers gives the same float64 grid."""
    from paper_2603_01122_b200.engine import CycleEngine, EngineConfig, complement_layers
    from paper_2603_01122_b200.scenario import make_scene
    sc = make_scene("cfg1", cycles=3, humans=3)
    res = {}
    for partial in (False, True):
        cfg = EngineConfig(n=2000, steps=10, dt=0.1, smoothing_sigma=0.1, seed=5, mode="production",
                           union_dtype="float64", union_mode="independent", union_partial=partial,
                           time_union=True)
        eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, cfg)
        eng.prime(sc.prev_xy)
        eng.stage(sc.track[0], buf=0)
        if chunks > 1:
            host = torch.empty(eng.unions[0].shape, dtype=eng.unions[0].dtype).pin_memory()
            eng.capture(buf=0, chunks=chunks, d2h=host).replay()
        else:
            eng.run_cycle(buf=0)
        torch.cuda.synchronize()
        eng.check_errors()
        u = eng.unions[0]
        if partial:
            complement_layers(u, time_union=True)
        res[partial] = (u.cpu().numpy(), eng.layers.cpu().numpy())
    u, L = res[False]
    ind = 1.0 - np.prod(1.0 - np.clip(L, 0, 1), axis=0)
    np.testing.assert_array_equal(u, np.maximum.accumulate(ind, axis=0))
    np.testing.assert_array_equal(res[True][1], L)  # same layers (same streams)
    np.testing.assert_array_equal(res[True][0], u)
    assert u.max() > 0 and np.all(u >= np.max(L, axis=0) - 1e-15)


@pytest.mark.parametrize("tag,with_stack,quad,n", [("nostack", False, False, 512), ("stack", True, False, 700),
                                                  ("quad", True, True, 300)])
def test_mppi_step_matches_reference(tag, with_stack, quad, n):
    """f3 row: GPU MPPI with the reference's noise streams vs the reference mppi_step."""
    from paper_2603_01122_b200 import planners as PL
    z = golden_io.load("mppi.npz")
    spec = G.GridSpec(60, 40, 0.1)
    stack = PR.PredictionStack(spec, z["layers"], 0.0, 0.1) if with_stack else None
    cfg = PL.MppiConfig(horizon=20, rollouts=n, dt=0.1, quadratic_control_cost=quad, seed=3)
    controls, diag = PL.mppi_step(PL.RobotState(1.0, 2.0, 0.4, 0.3), z[tag + "_nominal"],
                                  PL.RobotState(5.0, 2.2, 0.0, 0.0), stack, cfg, seed=11)
    np.testing.assert_allclose(diag.costs, z[tag + "_costs"], rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(controls, z[tag + "_controls"], rtol=1e-10, atol=1e-12)


def test_mppi_production_noise_statistics():
    """In-register Gaussian perturbations give the same control update (an MC estimate of
    the same path integral) as the reference streams, within sampling noise."""
    from paper_2603_01122_b200 import planners as PL
    cfg = PL.MppiConfig(horizon=10, rollouts=65536, dt=0.1, seed=5, temperature=20.0)
    args = (PL.RobotState(0.0, 0.0, 0.5, 0.0), np.zeros((10, 2)), PL.RobotState(3.0, 0.0, 0.0, 0.0), None, cfg)
    cp, dp = PL.mppi_step(*args, noise="production")
    cr, dr = PL.mppi_step(*args, noise="reference")
    assert np.isfinite(cp).all() and dp.weight_entropy > 0
    np.testing.assert_allclose(cp, cr, atol=0.02)
    assert abs(dp.mean_cost - dr.mean_cost) < 0.01 * abs(dr.mean_cost)


@pytest.mark.parametrize("mode", ["reference", "production"])
def test_chunked_horizon_is_bit_identical(mode):
    """Horizon chunking (K2 state hand-over + per-chunk K3/time union/blocked mask + chunked
    D2H inside a CUDA graph) reproduces the single-launch cycle bit-for-bit."""
    from paper_2603_01122_b200.engine import CycleEngine, EngineConfig
    from paper_2603_01122_b200.scenario import make_scene
    sc = make_scene("cfg1", cycles=2, humans=3)
    cfg = EngineConfig(n=3000, steps=22, dt=0.1, smoothing_sigma=0.1, seed=9, mode=mode, time_union=True,
                       robot_radius=0.25, collision_threshold=0.02)
    out = {}
    for chunks in (1, 3):
        eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, cfg)
        eng.prime(sc.prev_xy)
        eng.stage(sc.track[0], buf=0)
        host = torch.empty(eng.unions[0].shape, dtype=eng.unions[0].dtype).pin_memory()
        g = eng.capture(buf=0, chunks=chunks, d2h=host if chunks > 1 else None)
        g.replay()
        torch.cuda.synchronize()
        eng.check_errors()
        out[chunks] = (eng.unions[0].cpu().numpy(), eng.blocked[0].cpu().numpy(), host.numpy().copy())
    np.testing.assert_array_equal(out[1][0], out[3][0])
    np.testing.assert_array_equal(out[1][1], out[3][1])
    np.testing.assert_array_equal(out[3][2], out[1][0])
    assert out[1][0].max() > 0


@pytest.mark.parametrize("mode", ["reference", "production"])
def test_particle_block_sharding_is_partition_independent(mode):
    """One human's particles split over 'GPUs' (two engines here): the summed u32 counts
    reproduce the unsharded union bit-for-bit (streams keyed by the global particle index)."""
    from paper_2603_01122_b200.engine import CycleEngine, EngineConfig
    from paper_2603_01122_b200.scenario import make_scene
    import dataclasses
    sc = make_scene("cfg1", cycles=2, humans=2)
    cfg = EngineConfig(n=4096, steps=12, dt=0.1, smoothing_sigma=0.1, seed=3, mode=mode)

    def run(c, reduce=None):
        eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, c, counts_reduce=reduce)
        eng.prime(sc.prev_xy)
        eng.stage(sc.track[0], buf=0)
        eng.run_cycle(buf=0)
        torch.cuda.synchronize()
        return eng.unions[0].cpu().numpy()

    full = run(cfg)
    held = {}
    run(dataclasses.replace(cfg, particle_shard=(0, 2)), reduce=lambda c: held.setdefault("c", c.clone()))
    merged = run(dataclasses.replace(cfg, particle_shard=(1, 2)), reduce=lambda c: c.add_(held["c"]))
    np.testing.assert_array_equal(merged, full)


@pytest.mark.parametrize("name", golden_io.naive_case_names())
def test_predict_naive_matches_reference(name):
    """predict_naive (prediction.py:258-300) through gc_predict_naive: the float64
    per-particle loop reproduces the reference's layers (counts/n exactly at sigma 0)."""
    case = golden_io.NaiveCase(name)
    cs, space, q, spec = _objects(case)
    b = G.JointBelief(case.log_w)
    cfg = G.PredictionConfig(n=case.n, steps=case.steps, dt=case.dt, smoothing_sigma=case.sigma,
                             seed=case.seed)
    st = G.predict_naive(G.HumanState(*case.z0), b, cfg, cs, q, space, spec)
    if case.sigma == 0:
        np.testing.assert_array_equal(st.layers, case.layers)
    else:
        np.testing.assert_allclose(st.layers, case.layers, rtol=0, atol=1e-15)
    np.testing.assert_allclose(st.layers.sum(axis=(1, 2)), 1.0, atol=1e-9)


def test_predict_naive_abi_rejects_empty_control_set():
    """m_keep = 0 (every action masked) -> GC_EMPTY_CONTROL_SET -> EmptyControlSetError."""
    import ctypes
    from paper_2603_01122_b200 import _lib
    a = _lib.NaiveArgs()
    a.n, a.steps, a.m_keep = 4, 1, 0
    with pytest.raises(G.EmptyControlSetError):
        _lib.check(_lib.lib().gc_predict_naive(ctypes.byref(a), None), "predict_naive")
