"""GPU: drop-in conformance -- the behaviours the reference's own suite pins
(pkg/tests/test_prediction.py, test_belief.py, test_occupancy.py) checked
against the B200 implementation through its public, reference-named API.

Deviation by design: prediction with an arbitrary (unrecognised) lambda utility raises
NotImplementedError -- there is no CPU fallback (test_prediction.py:88-98 uses one).
"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2603_01122_b200 as G  # noqa: E402
from paper_2603_01122_b200.prediction import EnumerationCapExceeded  # noqa: E402


def lattice():
    """10x10 unit cells, unit moves in 4 directions + 4 stays (test_prediction.py:32-50)."""
    spec = G.GridSpec(10, 10, 1.0)
    heads = (0.0, math.pi / 2, -math.pi / 2, -math.pi)
    cs = G.ControlSet([G.ControlAction(0.0, h) for h in heads] + [G.ControlAction(1.0, h) for h in heads])
    space = G.HypothesisSpace(G.RationalitySet((0.5, 2.0)), G.GoalSet(np.array([[8.5, 4.5], [0.5, 4.5]])))
    return G.HumanState(4.5, 4.5), cs, G.q_goal_progress(1.0), space, spec


MODES = ["reference", "production"]


# ---- sampling ---------------------------------------------------------------------------

def test_sample_point_mass_and_frequencies():
    assert (G.sample_hypotheses(G.JointBelief.from_probs([0.0, 1.0, 0.0]), 500, seed=0) == 1).all()
    idx = G.sample_hypotheses(G.JointBelief.from_probs([0.25] * 4), 100_000, seed=1)
    np.testing.assert_allclose(np.bincount(idx, minlength=4) / len(idx), 0.25, atol=0.01)
    idx = G.sample_hypotheses(G.JointBelief.from_probs([0.7, 0.3]), 100_000, seed=2)
    np.testing.assert_allclose(np.bincount(idx, minlength=2) / len(idx), [0.7, 0.3], atol=0.01)
    b = G.JointBelief.from_probs([0.5, 0.5])
    np.testing.assert_array_equal(G.sample_hypotheses(b, 1000, seed=3), G.sample_hypotheses(b, 1000, seed=3))


# ---- propagation ------------------------------------------------------------------------

def test_single_forced_action_and_hypotheses_unchanged():
    cs = G.ControlSet([G.ControlAction(1.0, 0.0)])
    space = G.HypothesisSpace(G.RationalitySet((1.0,)), G.GoalSet(np.array([[5.0, 0.0]])))
    batch = G.ParticleBatch.duplicated(G.HumanState(0, 0), np.zeros(100, dtype=np.int32))
    out = G.propagate_step(batch, cs, G.q_goal_progress(0.5), space, dt=0.5, seed=0)
    np.testing.assert_allclose(out.xy, [[0.5, 0.0]] * 100, atol=1e-6)
    np.testing.assert_array_equal(out.hypothesis_idx, batch.hypothesis_idx)
    z0, cs, q, space, spec = lattice()
    hyp = G.sample_hypotheses(G.init_belief(space), 4096, seed=6)
    b = G.ParticleBatch.duplicated(z0, hyp)
    for step in range(3):
        b = G.propagate_step(b, cs, q, space, 1.0, seed=6, step=step)
        np.testing.assert_array_equal(b.hypothesis_idx, hyp)


def test_arbitrary_lambda_utility_has_no_cpu_fallback():
    cs = G.ControlSet([G.ControlAction(1.0, 0.0), G.ControlAction(0.0, 0.0)])
    space = G.HypothesisSpace(G.RationalitySet((50.0,)), G.GoalSet(np.array([[0.0, 0.0]])))
    q = G.QFunction(base=lambda xy, g, v, th: np.tile([0.0, -1.0], (len(xy), 1)))
    batch = G.ParticleBatch.duplicated(G.HumanState(0, 0), np.zeros(64, dtype=np.int32))
    with pytest.raises(NotImplementedError):
        G.propagate_step(batch, cs, q, space, dt=1.0, seed=4)


@pytest.mark.parametrize("mode", MODES)
def test_one_and_three_step_match_enumeration(mode):
    z0, cs, q, space, spec = lattice()
    b = G.init_belief(space)
    exact = G.exact_predict(z0, b, 1, 1.0, cs, q, space, spec)
    mc = G.predict(z0, b, G.PredictionConfig(n=65536, steps=1, dt=1.0, smoothing_sigma=0.0, seed=5, mode=mode),
                   cs, q, space, spec)
    assert G.total_variation(mc.layers[0], exact.layers[0]) < 0.05
    b = G.JointBelief.from_probs([0.35, 0.35, 0.15, 0.15])
    exact = G.exact_predict(z0, b, 3, 1.0, cs, q, space, spec)
    mc = G.predict(z0, b, G.PredictionConfig(n=65536, steps=3, dt=1.0, smoothing_sigma=0.0, seed=14, mode=mode),
                   cs, q, space, spec)
    for k in range(3):
        assert G.total_variation(mc.layers[k], exact.layers[k]) < 0.05


@pytest.mark.parametrize("mode", MODES)
def test_predict_delta_mass_and_smoothing(mode):
    cs = G.ControlSet([G.ControlAction(1.0, 0.0)])
    space = G.HypothesisSpace(G.RationalitySet((1.0,)), G.GoalSet(np.array([[5.0, 0.5]])))
    st = G.predict(G.HumanState(0.5, 0.5), G.init_belief(space),
                   G.PredictionConfig(n=256, steps=1, dt=1.0, smoothing_sigma=0.0, seed=0, mode=mode),
                   cs, G.q_goal_progress(0.5), space, G.GridSpec(6, 2, 1.0))
    assert st.layers[0][0, 1] == pytest.approx(1.0)
    assert st.layers[0].sum() == pytest.approx(1.0, abs=1e-9)
    z0, cs, q, space, spec = lattice()
    for sigma in (0.0, 0.7):
        st = G.predict(z0, G.init_belief(space),
                       G.PredictionConfig(n=4096, steps=4, dt=1.0, smoothing_sigma=sigma, seed=12, mode=mode),
                       cs, q, space, spec)
        for k in range(st.steps):
            assert st.layers[k].sum() == pytest.approx(1.0, abs=1e-6)
            assert (st.layers[k] >= 0).all()


@pytest.mark.parametrize("mode", MODES)
def test_deterministic_for_any_worker_count(mode):
    """test_prediction.py:128-136: bitwise identical for any worker count -- and, on the GPU,
    for repeated launches (integer count atomics, order-independent max)."""
    z0, cs, q, space, spec = lattice()
    cfg = G.PredictionConfig(n=8192, steps=3, dt=1.0, smoothing_sigma=0.1, seed=11, mode=mode)
    stacks = [G.predict(z0, G.init_belief(space), cfg, cs, q, space, spec, workers=w) for w in (None, 1, 2, 5)]
    for s in stacks[1:]:
        np.testing.assert_array_equal(s.layers, stacks[0].layers)


@pytest.mark.parametrize("mode", MODES)
def test_monte_carlo_error_shrinks_with_n(mode):
    z0, cs, q, space, spec = lattice()
    b = G.init_belief(space)
    exact = G.exact_predict(z0, b, 3, 1.0, cs, q, space, spec)
    worst = {}
    for n in (1024, 8192, 65536):
        mc = G.predict(z0, b, G.PredictionConfig(n=n, steps=3, dt=1.0, smoothing_sigma=0.0, seed=15, mode=mode),
                       cs, q, space, spec)
        worst[n] = max(G.total_variation(mc.layers[k], exact.layers[k]) for k in range(3))
    assert worst[1024] + 0.02 >= worst[8192] and worst[8192] + 0.02 >= worst[65536] and worst[65536] < 0.05


# ---- exact enumeration ------------------------------------------------------------------

def test_exact_predict_semantics():
    cs = G.ControlSet([G.ControlAction(1.0, 0.0)])
    space = G.HypothesisSpace(G.RationalitySet((1.0,)), G.GoalSet(np.array([[9.5, 0.5]])))
    st = G.exact_predict(G.HumanState(0.5, 0.5), G.init_belief(space), 4, 1.0, cs, G.q_goal_progress(0.5),
                         space, G.GridSpec(10, 1, 1.0))
    for t in range(4):
        expected = np.zeros((1, 10))
        expected[0, t + 1] = 1.0
        np.testing.assert_allclose(st.layers[t], expected, atol=1e-15)
    _, cs, q, _, _ = lattice()
    space = G.HypothesisSpace(G.RationalitySet((0.5, 2.0)), G.GoalSet(np.array([[7.5, 4.5], [1.5, 4.5]])))
    st = G.exact_predict(G.HumanState(4.5, 4.5), G.init_belief(space), 3, 1.0, cs, q, space, G.GridSpec(9, 9, 1.0))
    for k in range(3):
        np.testing.assert_allclose(st.layers[k], st.layers[k][:, ::-1], atol=1e-12)
        assert abs(st.layers[k].sum() - 1.0) < 1e-12
    z0, cs, q, space, spec = lattice()
    with pytest.raises(EnumerationCapExceeded):
        G.exact_predict(z0, G.init_belief(space), 2, 1.0, cs, q, space, spec, max_table=10)


# ---- multi-human union ------------------------------------------------------------------

def test_predict_multi_identity_disjoint_idempotent():
    z0, cs, q, space, spec = lattice()
    b = G.init_belief(space)
    cfg = G.PredictionConfig(n=2048, steps=3, dt=1.0, smoothing_sigma=0.0, seed=21)
    np.testing.assert_array_equal(G.predict_multi([(z0, b)], cfg, cs, q, space, spec).layers,
                                  G.predict(z0, b, cfg, cs, q, space, spec).layers)
    cs1 = G.ControlSet([G.ControlAction(0.0, 0.0)])
    sp1 = G.HypothesisSpace(G.RationalitySet((1.0,)), G.GoalSet(np.array([[0.0, 0.0]])))
    b1 = G.init_belief(sp1)
    merged = G.predict_multi([(G.HumanState(1.5, 1.5), b1), (G.HumanState(8.5, 8.5), b1)],
                             G.PredictionConfig(n=64, steps=2, dt=1.0, smoothing_sigma=0.0, seed=22),
                             cs1, G.q_goal_progress(0.5), sp1, G.GridSpec(10, 10, 1.0))
    assert merged.layers[0][1, 1] == pytest.approx(1.0) and merged.layers[0][8, 8] == pytest.approx(1.0)
    assert merged.layers[0].sum() == pytest.approx(2.0)
    cfg = G.PredictionConfig(n=1024, steps=2, dt=1.0, smoothing_sigma=0.0, seed=23)
    np.testing.assert_array_equal(G.predict_multi([(z0, b), (z0, b)], cfg, cs, q, space, spec).layers,
                                  G.predict(z0, b, cfg, cs, q, space, spec).layers)


# ---- belief -----------------------------------------------------------------------------

def make_space(n_betas=2, goals=((2.0, 0.0), (0.0, 2.0))):
    betas = tuple(np.geomspace(0.5, 2.0, n_betas)) if n_betas > 1 else (1.0,)
    return G.HypothesisSpace(G.RationalitySet(betas), G.GoalSet(np.array(goals)))


def small_cs():
    return G.ControlSet([G.ControlAction(v, th) for v in (0.0, 1.0) for th in (0.0, math.pi / 2, -math.pi / 2, -math.pi)])


def test_belief_generic_utilities_via_host_tables():
    space, cs = make_space(), small_cs()
    prior = G.JointBelief.from_probs([0.4, 0.3, 0.2, 0.1])
    flat = G.QFunction(base=lambda xy, g, v, th: np.zeros((len(xy), len(v))))
    post = G.update_belief(prior, G.HumanState(0, 0), G.HumanState(0.5, 0), 0.5, cs, flat, space)
    np.testing.assert_allclose(post.probs(), prior.probs(), atol=1e-12)

    def half_masked(xy, goal_xy, v, th):
        out = np.zeros((len(xy), 8))
        out[goal_xy[:, 0] == 2.0, 4:] = -np.inf
        return out

    post = G.update_belief(G.init_belief(space), G.HumanState(0, 0), G.HumanState(0, 0), 0.5, cs,
                           G.QFunction(base=half_masked), space, fallback_theta=math.pi / 2)
    assert space.goal_marginal(post)[0] == pytest.approx(2.0 / 3.0, abs=1e-9)
    rng = np.random.default_rng(8)
    table = rng.uniform(-3, 0, (1, len(cs)))
    prior = G.JointBelief.from_probs(rng.dirichlet(np.ones(space.size)))
    mk = lambda shift: G.QFunction(base=lambda xy, g, v, th: np.tile(table + shift, (len(xy), 1)))
    p0 = G.update_belief(prior, G.HumanState(0, 0), G.HumanState(0.5, 0), 0.5, cs, mk(0.0), space)
    p1 = G.update_belief(prior, G.HumanState(0, 0), G.HumanState(0.5, 0), 0.5, cs, mk(42.0), space)
    np.testing.assert_allclose(p0.probs(), p1.probs(), atol=1e-9)


def test_belief_log_linear_agreement_and_normalisation():
    space = make_space(3, ((2.0, 0.0), (0.0, 2.0), (-2.0, -1.0)))
    cs, q = small_cs(), G.q_goal_progress(0.5)
    b = G.init_belief(space)
    rng = np.random.default_rng(2)
    z = G.HumanState(0.1, -0.2)
    for _ in range(60):
        u = cs[int(rng.integers(len(cs)))]
        z2 = G.human_step(z, u, 0.5)
        d = math.hypot(z2.x - z.x, z2.y - z.y)
        uc = G.ControlAction(d / 0.5, math.atan2(z2.y - z.y, z2.x - z.x)) if d > 1e-6 else G.ControlAction(0.0, 0.0)
        from paper_2603_01122_b200.belief import observation_log_likelihood, snap_control
        idx = snap_control(uc, cs)
        lin = b.probs() * np.exp(observation_log_likelihood(z, idx, cs, q, space))
        lin /= lin.sum()
        b = G.update_belief(b, z, z2, 0.5, cs, q, space)
        assert np.max(np.abs(b.probs() - lin) / np.maximum(lin, 1e-300)) < 1e-6
        z = z2


def test_belief_convergence_zero_prior_and_mismatch():
    goals = tuple((3.0 * math.cos(a), 3.0 * math.sin(a)) for a in np.linspace(0, 2 * math.pi, 10, endpoint=False))
    space = G.HypothesisSpace(G.RationalitySet(tuple(np.geomspace(0.1, 10, 5))), G.GoalSet(np.array(goals)))
    cs, q = G.ControlSet.grid(4, 24, v_max=1.4), G.q_goal_progress(0.5)
    z, b, gen = G.HumanState(0.0, 0.0), G.init_belief(space), np.random.default_rng(11)
    hit = None
    for k in range(1, 11):
        p = G.boltzmann_policy(z, 10.0, goals[3], cs, q)
        j = int(np.searchsorted(np.cumsum(p), gen.random(), side="right"))
        z2 = G.human_step(z, cs[min(j, len(cs) - 1)], 0.1)
        b = G.update_belief(b, z, z2, 0.1, cs, q, space)
        z = z2
        if space.goal_marginal(b)[3] > 0.9:
            hit = k
            break
    assert hit is not None and hit <= 10
    space, cs = make_space(), small_cs()
    post = G.update_belief(G.JointBelief(np.array([-np.inf, 0.0, -np.inf, -np.inf])), G.HumanState(0, 0),
                           G.HumanState(0.5, 0), 0.5, cs, q, space)
    assert post.probs()[0] == 0.0 and post.probs()[2] == 0.0 and post.probs()[1] == pytest.approx(1.0)
    with pytest.raises(G.ControlSnapMismatch):
        G.update_belief(G.init_belief(space), G.HumanState(0, 0), G.HumanState(4.0, 0), 0.5, cs, q, space)


def test_mask_stationary_semantics():
    cs, q = small_cs(), G.q_goal_progress(0.5)
    p0 = G.boltzmann_policy(G.HumanState(0, 0), 1.0, (1, 1), cs, q)
    p1 = G.boltzmann_policy(G.HumanState(0, 0), 1.0, (1, 1), cs, G.mask_stationary(q, cs, 10.0))
    np.testing.assert_allclose(p0, p1, atol=1e-12)
    for beta in (0.1, 1.0, 50.0):
        p = G.boltzmann_policy(G.HumanState(0, 0), beta, (1, 1), cs, G.mask_stationary(q, cs, 0.0))
        assert p[cs.v > 0.0].sum() == 0.0 and p.sum() == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(G.EmptyMaskResultError):
        G.mask_stationary(q, G.ControlSet([G.ControlAction(1.0, 0.0), G.ControlAction(1.0, 1.0)]), 0.5)


# ---- occupancy --------------------------------------------------------------------------

def test_occupancy_emplace_smooth_union_collision():
    spec = G.GridSpec(8, 8, 0.5)
    g = G.emplace(G.ParticleBatch(np.array([[1.3, 2.1]] * 50, np.float32), np.zeros(50, np.int32)), spec)
    ix, iy = spec.cell_of(1.3, 2.1)
    assert g.mass() == pytest.approx(1.0, abs=1e-9) and g.at(ix, iy) == pytest.approx(1.0)
    rng = np.random.default_rng(0)
    pts = rng.uniform(-1, 4, (5000, 2))
    g = G.emplace(G.ParticleBatch(pts.astype(np.float32), np.zeros(5000, np.int32)), G.GridSpec(10, 7, 0.3))
    assert g.mass() == pytest.approx(1.0, abs=1e-9)
    spec = G.GridSpec(15, 15, 1.0)
    v = np.zeros((15, 15))
    v[7, 7] = 1.0
    s = G.gaussian_smooth(G.OccupancyGrid(spec, v), 1.0)
    k = np.exp(-0.5 * (np.arange(-3, 4) / 1.0) ** 2)
    k /= k.sum()
    expected = np.zeros((15, 15))
    expected[4:11, 4:11] = np.outer(k, k)
    np.testing.assert_allclose(s.values, expected, atol=1e-12)
    g20 = G.OccupancyGrid(G.GridSpec(20, 20, 1.0), np.full((20, 20), 0.01))
    np.testing.assert_allclose(G.gaussian_smooth(g20, 1.0).values[6:-6, 6:-6], 0.01, atol=1e-9)
    a, b = G.OccupancyGrid(G.GridSpec(2, 1, 1.0), np.array([[0.5, 0.0]])), \
        G.OccupancyGrid(G.GridSpec(2, 1, 1.0), np.array([[0.5, 0.2]]))
    u = G.union([a, b], mode="independent")
    assert u.values[0, 0] == pytest.approx(0.75) and u.values[0, 1] == pytest.approx(0.2)
    with pytest.raises(G.GridSpecMismatch):
        G.union_max([G.OccupancyGrid.zeros(G.GridSpec(5, 5, 1.0)), G.OccupancyGrid.zeros(G.GridSpec(5, 5, 0.5))])
    spec = G.GridSpec(8, 6, 0.1)
    grid = G.OccupancyGrid(spec, np.random.default_rng(9).random((6, 8)) * 0.05)
    field = G.collision_field(grid, 0.25)
    for ix in range(8):
        for iy in range(6):
            assert field[iy, ix] == pytest.approx(G.collision_probability(grid, spec.cell_center(ix, iy), 0.25),
                                                  abs=1e-12)
