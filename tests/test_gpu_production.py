"""GPU: production RNG mode is exact in distribution.

* one-step action distributions (every action on its own cell) vs the exact float64
  Boltzmann mixture -- factorised sampler (plain, stationary-masked, weighted) and the
  generic per-action sampler;
* multi-step layers vs the reference mode, TV bounded by the reference's own
  seed-to-seed spread (self-calibrated);
* the lattice instance vs exact enumeration (test_prediction.py:100-106 pattern);
* hypothesis frequencies vs the belief.
"""

import math

import numpy as np
import pytest
import torch

import golden_io

pytestmark = pytest.mark.gpu

import paper_2603_01122_b200 as G  # noqa: E402
from paper_2603_01122_b200 import prediction as PR  # noqa: E402


def exact_action_probs(z, belief, cs, q, space):
    """float64 mixture over hypotheses of the Boltzmann policy at state z."""
    p = np.zeros(len(cs))
    w = belief.probs()
    for h, (b, g) in enumerate(zip(space.beta_of, space.goal_xy_of)):
        if w[h] > 0:
            p += w[h] * G.boltzmann_policy(z, b, g, cs, q)
    return p


def one_step_tv(q_factory, n=1 << 22, weights=None, mask_v=None, goals=((0.5, 0.3), (0.1, 0.15)),
                speeds=4, betas=(0.3, 2.0, 9.0), origin=(0.0, 0.0), shape=(400, 400), cs=None):
    cs = G.ControlSet.grid(speeds, 24, 1.4) if cs is None else cs
    q = q_factory()
    if mask_v is not None:
        q = G.mask_stationary(q, cs, mask_v)
    space = G.HypothesisSpace(G.RationalitySet(betas), G.GoalSet(np.array(goals)))
    b = G.JointBelief.from_probs(weights if weights is not None else np.full(space.size, 1.0 / space.size))
    W, H = shape
    spec = G.GridSpec(W, H, 0.001, origin)
    z = G.HumanState(origin[0] + 0.2005, origin[1] + 0.2005)
    goals = tuple((gx + origin[0], gy + origin[1]) for gx, gy in goals)
    dev = torch.device("cuda")
    tab = PR.action_tables(cs, q, 0.1, dev)
    job = PR.HumanJob(z, b.log_weights, space.beta_of, space.goal_xy_of, 12345, (), 0)
    out = PR.run_predict([job], [tab], n, 1, 0.1, 0.0, spec, "production")
    layer = out["layers"][0, 0].cpu().numpy()
    # exact: action -> cell with the production kernel's float32 cell arithmetic
    p = exact_action_probs(z, b, cs, q, space)
    disp = cs.displacements(0.1).astype(np.float32)
    x = np.float32(z.x) + disp[:, 0]
    y = np.float32(z.y) + disp[:, 1]
    inv = np.float32(1.0) / np.float32(0.001)
    ix = np.clip(np.floor((x - np.float32(origin[0])) * inv).astype(int), 0, W - 1)
    iy = np.clip(np.floor((y - np.float32(origin[1])) * inv).astype(int), 0, H - 1)
    exact = np.zeros((H, W))
    np.add.at(exact, (iy, ix), p)
    return 0.5 * np.abs(layer - exact).sum(), tab.factorised


def test_factorised_one_step_exact_in_distribution():
    tv, fact = one_step_tv(lambda: G.q_goal_progress(0.5))
    assert fact
    assert tv < 0.006, tv


def test_factorised_masked_and_weighted():
    tv, fact = one_step_tv(lambda: G.q_goal_progress(0.5), mask_v=0.5)
    assert fact and tv < 0.006, tv
    tv, fact = one_step_tv(lambda: G.q_goal_progress(0.4, (0.3, 0.2)), weights=[0.1, 0.2, 0.05, 0.3, 0.05, 0.3])
    assert fact and tv < 0.006, tv


@pytest.mark.parametrize("speeds", [2, 3, 4])
def test_factorised_speed_counts(speeds):
    """Top-speed normalisation of the speed weights for 2, 3 and 4 speeds (n_speeds - 1
    moving speeds + stay), including a distant goal (small Q = 2^-kr)."""
    tv, fact = one_step_tv(lambda: G.q_goal_progress(0.5), speeds=speeds, goals=((0.5, 0.3), (40.0, 30.0)))
    assert fact and tv < 0.006, tv


def test_factorised_offset_origin_and_rectangular_grid():
    """Grid units u = (x - origin) / res with a negative origin and a 420 x 380 grid."""
    tv, fact = one_step_tv(lambda: G.q_goal_progress(0.5), origin=(-1.5, 2.25), shape=(420, 380))
    assert fact and tv < 0.006, tv


def test_factorised_large_beta_fallback():
    """beta = 300 overflows the top-speed constants 2^(c top^2): the CTA keeps the
    max-shift speed weights (and the other hypotheses of that human with it)."""
    tv, fact = one_step_tv(lambda: G.q_goal_progress(0.5), betas=(0.3, 2.0, 300.0))
    assert fact and tv < 0.006, tv


def test_generic_sampler_one_step():
    tv, fact = one_step_tv(lambda: G.q_default((0.3, 2.0)))
    assert not fact
    assert tv < 0.006, tv


def _random_actions(m, seed=0):
    r = np.random.default_rng(seed)
    return G.ControlSet([G.ControlAction(float(v), float(t))
                         for v, t in zip(r.uniform(0.05, 1.4, m), r.uniform(-np.pi, np.pi, m))])


@pytest.mark.parametrize("m,mask_v,betas", [
    (96, None, (0.3, 2.0, 9.0)),     # one-pass generic sampler, goal-progress utility
    (96, 0.5, (0.3, 2.0, 9.0)),      # masked (the FULL utility) over the kept actions
    (48, None, (0.3, 2.0, 9.0)),     # the 48-action instantiation
    (60, None, (0.3, 2.0, 9.0)),     # an action count without an instantiation: two-pass form
    (96, None, (0.3, 2.0, 900.0)),   # a bound so loose the weights underflow: two-pass fallback
])
def test_generic_sampler_non_grid_sets(m, mask_v, betas):
    """The production generic sampler (round 2: one pass with an analytic bound of the max
    logit, compiled for 96 / 48 actions; two passes otherwise or when the bound underflows)
    is exact in distribution on control sets that are not speed x heading grids."""
    cs = _random_actions(m)
    tv, fact = one_step_tv(lambda: G.q_goal_progress(0.5), cs=cs, mask_v=mask_v, betas=betas)
    assert not fact and tv < 0.006, tv


def test_far_goal_high_beta_no_overflow():
    # |rel| ~ 57 m, beta = 9: logits reach hundreds; weights must stay finite
    tv, _ = one_step_tv(lambda: G.q_goal_progress(0.5), goals=((40.2, 40.2), (-39.8, 0.2)))
    assert tv < 0.006, tv


def test_multistep_tv_within_reference_seed_spread():
    cs = G.ControlSet.grid(4, 24, 1.4)
    q = G.q_goal_progress(0.5)
    goals = np.array([[17.0, 10.0], [10.0, 17.0], [3.0, 10.0], [10.0, 3.0]])
    space = G.HypothesisSpace(G.RationalitySet.log_spaced(5), G.GoalSet(goals))
    case = golden_io.PredictCase("cfg2_t30")
    b = G.JointBelief(case.log_w)
    spec = G.GridSpec(200, 200, 0.1)
    z = G.HumanState(10.0, 10.0)
    worst = {}
    for sigma in (0.0, 0.1):
        layers = {}
        for tag, seed, mode in (("a", 1, "reference"), ("b", 2, "reference"), ("p", 3, "production")):
            cfg = G.PredictionConfig(n=65536, steps=100, dt=0.02, smoothing_sigma=sigma, seed=seed, mode=mode)
            layers[tag] = G.predict(z, b, cfg, cs, q, space, spec).layers
        tv = lambda u, v: max(0.5 * np.abs(u[k] - v[k]).sum() for k in range(100))
        spread = tv(layers["a"], layers["b"])
        got = max(tv(layers["p"], layers["a"]), tv(layers["p"], layers["b"]))
        worst[sigma] = (got, spread)
        assert got <= 1.5 * spread + 0.005, (sigma, got, spread)


def test_lattice_production_matches_enumeration():
    z = golden_io.load("exact.npz")
    case = golden_io.PredictCase("lattice")
    m = case.meta
    cs = G.ControlSet([G.ControlAction(float(v), float(t)) for v, t in zip(m["v"], m["theta"])])
    space = G.HypothesisSpace(G.RationalitySet(tuple(m["betas"])), G.GoalSet(np.array(m["goals"])))
    q = G.q_goal_progress(1.0)
    spec = G.GridSpec(10, 10, 1.0)
    b = G.JointBelief(z["log_w"])
    cfg = G.PredictionConfig(n=65536, steps=3, dt=1.0, smoothing_sigma=0.0, seed=14, mode="production")
    mc = G.predict(G.HumanState(4.5, 4.5), b, cfg, cs, q, space, spec)
    for k in range(3):
        assert G.total_variation(mc.layers[k], z["layers"][k]) < 0.05


def test_production_hypothesis_frequencies():
    cs = G.ControlSet.grid(4, 24, 1.4)
    q = G.q_goal_progress(0.5)
    space = G.HypothesisSpace(G.RationalitySet((1.0, 3.0)), G.GoalSet(np.array([[1.0, 1.0], [2.0, 2.0]])))
    probs = np.array([0.1, 0.2, 0.3, 0.4])
    b = G.JointBelief.from_probs(probs)
    tab = PR.action_tables(cs, q, 0.1, torch.device("cuda"))
    job = PR.HumanJob(G.HumanState(1.5, 1.5), b.log_weights, space.beta_of, space.goal_xy_of, 99, (), 0)
    out = PR.run_predict([job], [tab], 200_000, 1, 0.1, 0.0, G.GridSpec(40, 40, 0.1), "production",
                         want_hyp=True)
    freq = np.bincount(out["hyp"][0].cpu().numpy(), minlength=4) / 200_000
    np.testing.assert_allclose(freq, probs, atol=0.01)


def test_production_streams_independent_of_launch_shape():
    """A human's production draws depend only on (seed, stream, particle, step): alone
    (small launch: K = 1 particle per thread, lanes take turns drawing Philox blocks) and as
    the first of 160 humans (K = 4, one block per thread per step) its layers are identical."""
    cs = G.ControlSet.grid(4, 24, 1.4)
    q = G.q_goal_progress(0.5)
    space = G.HypothesisSpace(G.RationalitySet.log_spaced(5), G.GoalSet(np.array([[8.5, 5.0], [1.5, 7.0]])))
    spec = G.GridSpec(100, 100, 0.1)
    dev = torch.device("cuda")
    tab = PR.action_tables(cs, q, 0.1, dev)
    lw = np.log(np.random.default_rng(4).dirichlet(np.ones(space.size)))
    lw -= np.log(np.exp(lw).sum())
    job = PR.HumanJob(G.HumanState(5.0, 5.0), lw, space.beta_of, space.goal_xy_of, 99, (), 0)
    others = [PR.HumanJob(G.HumanState(2.0 + 0.03 * i, 3.0), lw, space.beta_of, space.goal_xy_of, 99, (), 0)
              for i in range(159)]
    n, T = 4096, 9  # 9 steps: K = 1 takes turns over 4 steps, a partial last turn included
    alone = PR.run_predict([job], [tab], n, T, 0.1, 0.0, spec, "production")["layers"][0].cpu().numpy()
    multi = PR.run_predict([job] + others, [tab], n, T, 0.1, 0.0, spec, "production")["layers"][0].cpu().numpy()
    assert alone.sum() > 0
    np.testing.assert_array_equal(alone, multi)


def test_mixed_tables_in_one_launch():
    """One launch with humans on the 4-speed grid table and on mask_stationary's 2-speed
    table (the engine's moving / stationary humans): K2 picks the step-loop instance per CTA
    (4-speed tables without the speed-count selects, the rest general), and each human's
    one-step occupancy matches its own exact distribution."""
    cs = G.ControlSet.grid(4, 24, 1.4)
    q = G.q_goal_progress(0.5)
    qm = G.mask_stationary(q, cs, 0.5)
    dev = torch.device("cuda")
    tabs = [PR.action_tables(cs, q, 0.1, dev), PR.action_tables(cs, qm, 0.1, dev)]
    assert tabs[0].struct.n_speeds == 4 and tabs[1].struct.n_speeds == 2
    space = G.HypothesisSpace(G.RationalitySet((0.3, 2.0, 9.0)), G.GoalSet(np.array([[0.5, 0.3], [0.1, 0.15]])))
    b = G.JointBelief.from_probs(np.full(space.size, 1.0 / space.size))
    spec = G.GridSpec(400, 400, 0.001)
    z = G.HumanState(0.2005, 0.2005)
    jobs = [PR.HumanJob(z, b.log_weights, space.beta_of, space.goal_xy_of, 12345, (), t) for t in (1, 0, 1)]
    n = 1 << 21
    out = PR.run_predict(jobs, tabs, n, 1, 0.1, 0.0, spec, "production")
    layers = out["layers"][:, 0].cpu().numpy()
    disp = cs.displacements(0.1).astype(np.float32)
    x = np.float32(z.x) + disp[:, 0]
    y = np.float32(z.y) + disp[:, 1]
    inv = np.float32(1.0) / np.float32(0.001)
    ix = np.clip(np.floor(x * inv).astype(int), 0, 399)
    iy = np.clip(np.floor(y * inv).astype(int), 0, 399)
    for hi, qq in zip(range(3), (qm, q, qm)):
        p = exact_action_probs(z, b, cs, qq, space)
        exact = np.zeros((400, 400))
        np.add.at(exact, (iy, ix), p)
        tv = 0.5 * np.abs(layers[hi] - exact).sum()
        assert tv < 0.006, (hi, tv)
