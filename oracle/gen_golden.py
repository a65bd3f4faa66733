"""Generate tests/golden/*.npz from the LIVE reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python -m oracle.gen_golden

Imports the reference package read-only from /root/reference/pkg/src and records its
outputs on seeded inputs.  The fixtures travel with the repo (the reference does
not exist on the GPU box).  Cases (reference file:line they exercise):

  philox.npz    rng.stream f32/f64 draws + derive_seed          rng.py:27-39
  exp.npz       numpy float32 exp on the hot-path input range    prediction.py:156
  predict_*.npz predict() hyp indices, per-step counts, float32 positions, layers
                                                                prediction.py:223-255
  belief.npz    update_belief() chains incl. masked/zero-prior/fallback
                                                                belief.py:159-198
  smooth.npz    smooth_values() on random layers                occupancy.py:139-154
  multi.npz     sim-style per-human predict + union_max + time union
                                                                sim.py:489-504
  exact.npz     exact_predict() on the lattice instance         prediction.py:303-377
  naive_*.npz   predict_naive() float64 per-particle loop        prediction.py:258-300
  cfg3_cycle.npz  the headline shape: 8 humans x 262,144 particles of the cfg3 scene after
                10 belief updates, 25 steps, sim-style seed/prefix/masked Q, sigma 0.1,
                per-human counts, max union and time union       sim.py:455-505
  long_cfg4.npz   a cfg4 human (T = 500: windows beyond shared memory -> K2's global-
                histogram path), 4096 particles                 prediction.py:223-255
  uniforms_cfg1.npz the reference's own pre-drawn uniforms of the cfg1_s0 case (hypothesis
                and step draws) for GC_RNG_UNIFORMS            prediction.py:128-131, :186-192

    PYTHONPATH=/root/reference/pkg/src python -m oracle.gen_golden [case ...]
regenerates only the named cases (philox exp predict belief smooth multi exact collision
gcst mppi naive cfg3_cycle long_cfg4 uniforms).
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _ref():
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import gridcast  # noqa: F401
    return gridcast


def gen_philox(G):
    from gridcast import rng
    r = np.random.default_rng(123)
    seeds, paths, f32, f64, derived = [], [], [], [], []
    for i in range(64):
        seed = int(r.integers(0, 2**63)) if i % 3 else int(r.integers(0, 2**20))
        plen = int(r.integers(0, 6))
        path = [int(r.integers(0, 2**32)) if j % 2 else int(r.integers(0, 300)) for j in range(plen)]
        seeds.append(seed)
        paths.append(path)
        f32.append(rng.stream(seed, *path).random(24, dtype=np.float32))
        f64.append(rng.stream(seed, *path).random(12))
        derived.append(rng.derive_seed(seed, *path))
    np.savez_compressed(
        os.path.join(OUT, "philox.npz"),
        meta=json.dumps(dict(seeds=seeds, paths=paths, derived=[str(d) for d in derived])),
        f32=np.stack(f32), f64=np.stack(f64),
    )


def gen_exp():
    r = np.random.default_rng(7)
    x = np.concatenate([
        r.uniform(-110, 0, 60000), r.uniform(-2, 0, 20000), np.linspace(-104.0, -86.0, 20000),
        np.array([0.0, -0.0, -1e-30, -87.33654, -103.972, -103.97208404541015625, -104.0]),
    ]).astype(np.float32)
    np.savez_compressed(os.path.join(OUT, "exp.npz"), x=x, y=np.exp(x))


def _spec(G, case):
    cs = G.ControlSet([G.ControlAction(float(v), float(t)) for v, t in zip(case["v"], case["theta"])])
    space = G.HypothesisSpace(G.RationalitySet(tuple(case["betas"])), G.GoalSet(np.array(case["goals"])))
    fam = case["q"]
    if fam["family"] == "goal_progress":
        q = G.q_goal_progress(fam["tau"], (fam["w_v"], fam["w_th"]))
    else:
        q = G.q_default((fam["w_v"], fam["w_th"]))
    if fam.get("v_threshold") is not None:
        from gridcast.belief import mask_stationary
        q = mask_stationary(q, cs, fam["v_threshold"])
    g = case["grid"]
    spec = G.GridSpec(g[0], g[1], g[2], tuple(g[3]))
    return cs, space, q, spec


def _grid_cs():
    from oracle.model import control_grid
    v, th = control_grid(4, 24, 1.4)
    return v.tolist(), th.tolist()


def predict_cases():
    v, th = _grid_cs()
    lat_th = [0.0, math.pi / 2, -math.pi / 2, -math.pi] * 2
    lat_v = [0.0] * 4 + [1.0] * 4
    gp = dict(family="goal_progress", tau=0.5, w_v=0.0, w_th=0.0, v_threshold=None)
    cases = {
        # cfg1 (BASELINE.json configs[0]): 1 human, 2 goals, 5 betas, 1024 particles, T=20,
        # dt 0.1, 100x100 @ 0.1 m; sigma 0 (count parity) and 0.1 (smoothed layers)
        "cfg1_s0": dict(v=v, theta=th, betas=list(np.geomspace(0.1, 10, 5)),
                        goals=[[8.5, 5.0], [1.5, 7.0]], q=gp, grid=[100, 100, 0.1, [0.0, 0.0]],
                        z0=[5.0, 5.0], n=1024, steps=20, dt=0.1, sigma=0.0, seed=0, prefix=[2, 0],
                        belief="posterior"),
        "cfg1_s01": dict(v=v, theta=th, betas=list(np.geomspace(0.1, 10, 5)),
                         goals=[[8.5, 5.0], [1.5, 7.0]], q=gp, grid=[100, 100, 0.1, [0.0, 0.0]],
                         z0=[5.0, 5.0], n=1024, steps=20, dt=0.1, sigma=0.1, seed=3, prefix=[],
                         belief="posterior"),
        # ragged particle count (partial last chunk), weights, edge clamping near origin
        "ragged_w": dict(v=v, theta=th, betas=[0.5, 2.0, 8.0], goals=[[-1.0, 0.3], [3.0, 2.9]],
                         q=dict(family="goal_progress", tau=0.3, w_v=0.2, w_th=0.1, v_threshold=None),
                         grid=[40, 30, 0.1, [0.0, 0.0]], z0=[0.35, 0.2], n=3333, steps=12, dt=0.1,
                         sigma=0.0, seed=99, prefix=[2, 5], belief="random"),
        # stationary-masked Q (mask_stationary drops base_policy -> full base)
        "masked": dict(v=v, theta=th, betas=list(np.geomspace(0.1, 10, 5)),
                       goals=[[4.0, 9.0], [9.0, 1.0], [0.5, 0.5], [6.0, 6.0]],
                       q=dict(family="goal_progress", tau=0.5, w_v=0.0, w_th=0.0, v_threshold=0.5),
                       grid=[100, 100, 0.1, [0.0, 0.0]], z0=[5.0, 5.0], n=2048, steps=10, dt=0.1,
                       sigma=0.0, seed=5, prefix=[2, 1], belief="random"),
        # q_default with weights (position-independent policy)
        "qdefault": dict(v=v, theta=th, betas=[0.3, 1.0, 3.0],
                         goals=[[1.0, 1.0], [2.0, 3.0]],
                         q=dict(family="default", tau=0.5, w_v=0.3, w_th=2.0, v_threshold=None),
                         grid=[64, 48, 0.05, [-0.5, 0.25]], z0=[1.1, 1.3], n=1500, steps=8, dt=0.05,
                         sigma=0.0, seed=11, prefix=[], belief="uniform"),
        # cfg2 shape (65,536 particles, 4 goals, dt 0.02, 200x200) truncated to 30 steps
        "cfg2_t30": dict(v=v, theta=th, betas=list(np.geomspace(0.1, 10, 5)),
                        goals=[[17.0, 10.0], [10.0, 17.0], [3.0, 10.0], [10.0, 3.0]], q=gp,
                        grid=[200, 200, 0.1, [0.0, 0.0]], z0=[10.0, 10.0], n=65536, steps=30, dt=0.02,
                        sigma=0.0, seed=2, prefix=[2, 0], belief="posterior"),
        # edge cases: one particle, one step, a 1x1 grid, a start outside the grid
        "one_particle": dict(v=v, theta=th, betas=[1.0, 5.0], goals=[[2.0, 2.0]], q=gp,
                             grid=[30, 30, 0.1, [0.0, 0.0]], z0=[1.5, 1.5], n=1, steps=7, dt=0.1,
                             sigma=0.0, seed=123, prefix=[2, 9], belief="random"),
        "one_step": dict(v=v, theta=th, betas=[0.5, 2.0], goals=[[3.0, 0.0], [0.0, 3.0]], q=gp,
                         grid=[40, 40, 0.1, [0.0, 0.0]], z0=[2.0, 2.0], n=777, steps=1, dt=0.1,
                         sigma=0.1, seed=5, prefix=[], belief="random"),
        "grid1x1": dict(v=v, theta=th, betas=[1.0], goals=[[0.5, 0.5]], q=gp,
                        grid=[1, 1, 0.1, [0.0, 0.0]], z0=[0.05, 0.05], n=300, steps=4, dt=0.1,
                        sigma=0.0, seed=8, prefix=[], belief="uniform"),
        "outside": dict(v=v, theta=th, betas=[0.3, 3.0], goals=[[1.0, 1.0], [-2.0, 0.5]], q=gp,
                        grid=[25, 20, 0.1, [0.0, 0.0]], z0=[-0.7, 2.6], n=2000, steps=9, dt=0.1,
                        sigma=0.1, seed=31, prefix=[2, 3], belief="random"),
        # zero-probability hypotheses (log weight -inf) and the maximum sizes: 128
        # hypotheses (8 betas x 16 goals) and 256 actions (8 speeds x 32 headings)
        "zero_hyps": dict(v=v, theta=th, betas=list(np.geomspace(0.1, 10, 5)),
                          goals=[[8.0, 5.0], [2.0, 5.0], [5.0, 8.0], [5.0, 2.0]], q=gp,
                          grid=[100, 100, 0.1, [0.0, 0.0]], z0=[5.0, 5.0], n=4096, steps=6, dt=0.1,
                          sigma=0.0, seed=77, prefix=[2, 1], belief="zeros"),
        "max_sizes": dict(v=np.repeat(np.linspace(0, 1.4, 8), 32).tolist(),
                          theta=[float((t + math.pi) % (2 * math.pi) - math.pi) for t in
                                 np.tile(-np.pi + 2 * np.pi * np.arange(32) / 32, 8)],
                          betas=list(np.geomspace(0.1, 10, 8)),
                          goals=[[5.0 + 3.0 * math.cos(a), 5.0 + 3.0 * math.sin(a)] for a in np.linspace(0, 6.0, 16)],
                          q=gp, grid=[100, 100, 0.1, [0.0, 0.0]], z0=[5.0, 5.0], n=2500, steps=5, dt=0.1,
                          sigma=0.1, seed=4, prefix=[2, 2], belief="random"),
        # the reference's lattice instance (test_prediction.py:32-50)
        "lattice": dict(v=lat_v, theta=lat_th, betas=[0.5, 2.0], goals=[[8.5, 4.5], [0.5, 4.5]],
                        q=dict(family="goal_progress", tau=1.0, w_v=0.0, w_th=0.0, v_threshold=None),
                        grid=[10, 10, 1.0, [0.0, 0.0]], z0=[4.5, 4.5], n=8192, steps=3, dt=1.0,
                        sigma=0.1, seed=11, prefix=[], belief="uniform"),
    }
    return cases


def _belief_for(G, space, cs, kind, seed):
    if kind == "uniform":
        return G.init_belief(space)
    r = np.random.default_rng(seed)
    if kind == "random":
        return G.JointBelief.from_probs(r.dirichlet(np.ones(space.size)))
    if kind == "zeros":
        p = r.dirichlet(np.ones(space.size))
        p[::3] = 0.0
        return G.JointBelief.from_probs(p)
    # posterior after 10 synthetic observations of a Boltzmann walker
    from gridcast.belief import update_belief
    b = G.init_belief(space)
    q = G.q_goal_progress(0.5)
    goals = space.goals.positions
    z = G.HumanState(float(np.mean(goals[:, 0])), float(np.mean(goals[:, 1])))
    for _ in range(10):
        p = G.boltzmann_policy(z, 10.0, goals[0], cs, q)
        j = min(int(np.searchsorted(np.cumsum(p), r.random(), side="right")), len(cs) - 1)
        z2 = G.human_step(z, cs[j], 0.1)
        b = update_belief(b, z, z2, 0.1, cs, q, space, snap_tol=math.inf)
        z = z2
    return b


def gen_predict(G):
    from gridcast.prediction import PredictionConfig, predict, sample_hypotheses, propagate_step, ParticleBatch
    from oracle import model
    for name, case in predict_cases().items():
        cs, space, q, spec = _spec(G, case)
        b = _belief_for(G, space, cs, case["belief"], 17)
        cfg = PredictionConfig(n=case["n"], steps=case["steps"], dt=case["dt"],
                               smoothing_sigma=case["sigma"], seed=case["seed"])
        pre = tuple(case["prefix"])
        stack = predict(G.HumanState(*case["z0"]), b, cfg, cs, q, space, spec, prefix=pre)
        hyp = sample_hypotheses(b, cfg.n, cfg.seed, prefix=pre)
        # per-step float32 positions through the public propagate_step
        batch = ParticleBatch.duplicated(G.HumanState(*case["z0"]), hyp)
        xy_steps = []
        counts = []
        from gridcast.occupancy import emplace_counts
        for t in range(1, cfg.steps + 1):
            batch = propagate_step(batch, cs, q, space, cfg.dt, cfg.seed, step=t, prefix=pre)
            xy_steps.append(batch.xy.copy())
            counts.append(emplace_counts(batch.xy, spec).astype(np.int64))
        counts = np.stack(counts)
        nz = np.nonzero(counts)
        qs = case["q"]
        tb = model.make_tables(cs.v, cs.theta, cfg.dt,
                               model.QSpec(qs["family"], qs["tau"], qs["w_v"], qs["w_th"], qs["v_threshold"]))
        keep_steps = sorted({0, cfg.steps // 2, cfg.steps - 1})
        payload = dict(
            meta=json.dumps(case),
            log_w=b.log_weights,
            hyp=hyp,
            count_idx=np.stack(nz, axis=1).astype(np.int32),
            count_val=counts[nz].astype(np.int32),
            xy_first=xy_steps[0], xy_last=xy_steps[-1],
            layer_steps=np.array(keep_steps),
            layers=stack.layers[keep_steps],
            layer_sums=stack.layers.sum(axis=(1, 2)),
            # tables as the reference host computes them (float32), so the GPU box
            # need not recompute numpy cos/sin
            sx=tb.sx, sy=tb.sy, at=tb.at, pen=tb.pen, dispx=tb.dispx, dispy=tb.dispy,
            keep=tb.keep, q_kind=np.int32(tb.q_kind),
            ref_disp=cs.displacements(cfg.dt).astype(np.float32),
        )
        np.savez_compressed(os.path.join(OUT, f"predict_{name}.npz"), **payload)
        print("predict", name, "nnz", len(nz[0]))


def naive_cases():
    v, th = _grid_cs()
    gp = dict(family="goal_progress", tau=0.5, w_v=0.0, w_th=0.0, v_threshold=None)
    return {
        # cfg1-like, two 1024-particle stream chunks (the second partial)
        "gp": dict(v=v, theta=th, betas=list(np.geomspace(0.1, 10, 5)), goals=[[8.5, 5.0], [1.5, 7.0]],
                   q=gp, grid=[100, 100, 0.1, [0.0, 0.0]], z0=[5.0, 5.0], n=1100, steps=10, dt=0.1,
                   sigma=0.0, seed=4, belief="posterior"),
        "masked_s01": dict(v=v, theta=th, betas=[0.5, 3.0], goals=[[4.0, 9.0], [9.0, 1.0]],
                           q=dict(family="goal_progress", tau=0.5, w_v=0.0, w_th=0.0, v_threshold=0.5),
                           grid=[60, 60, 0.1, [0.0, 0.0]], z0=[3.0, 3.0], n=400, steps=6, dt=0.1,
                           sigma=0.1, seed=9, belief="random"),
        "qdefault": dict(v=v, theta=th, betas=[0.3, 1.0, 3.0], goals=[[1.0, 1.0], [2.0, 3.0]],
                         q=dict(family="default", tau=0.5, w_v=0.3, w_th=2.0, v_threshold=None),
                         grid=[64, 48, 0.05, [-0.5, 0.25]], z0=[1.1, 1.3], n=300, steps=5, dt=0.05,
                         sigma=0.0, seed=11, belief="uniform"),
        # weights, start near the origin corner (edge clamping)
        "weights_edge": dict(v=v, theta=th, betas=[0.5, 2.0, 8.0], goals=[[-1.0, 0.3], [3.0, 2.9]],
                             q=dict(family="goal_progress", tau=0.3, w_v=0.2, w_th=0.1, v_threshold=None),
                             grid=[40, 30, 0.1, [0.0, 0.0]], z0=[0.35, 0.2], n=700, steps=8, dt=0.1,
                             sigma=0.0, seed=99, belief="random"),
    }


def gen_naive(G):
    from gridcast.prediction import PredictionConfig, predict_naive
    for name, case in naive_cases().items():
        cs, space, q, spec = _spec(G, case)
        b = _belief_for(G, space, cs, case["belief"], 17)
        cfg = PredictionConfig(n=case["n"], steps=case["steps"], dt=case["dt"],
                               smoothing_sigma=case["sigma"], seed=case["seed"])
        st = predict_naive(G.HumanState(*case["z0"]), b, cfg, cs, q, space, spec)
        L = st.layers
        nz = np.nonzero(L)
        np.savez_compressed(os.path.join(OUT, f"naive_{name}.npz"), meta=json.dumps(case), log_w=b.log_weights,
                            idx=np.stack(nz, axis=1).astype(np.int32), val=L[nz], shape=np.array(L.shape))
        print("naive", name, "nnz", len(nz[0]))


def gen_belief(G):
    from gridcast.belief import update_belief, mask_stationary, ControlSnapMismatch
    from oracle.model import control_grid
    v, th = control_grid(4, 24, 1.4)
    cs = G.ControlSet([G.ControlAction(float(a), float(b)) for a, b in zip(v, th)])
    r = np.random.default_rng(5)
    goals = r.uniform(0, 10, (4, 2))
    space = G.HypothesisSpace(G.RationalitySet.log_spaced(5), G.GoalSet(goals))
    chains = []
    specs = [
        dict(family="goal_progress", tau=0.5, w_v=0.0, w_th=0.0, v_threshold=None),
        dict(family="goal_progress", tau=0.5, w_v=0.0, w_th=0.0, v_threshold=0.5),
        dict(family="goal_progress", tau=0.4, w_v=0.1, w_th=0.05, v_threshold=None),
        dict(family="default", tau=0.5, w_v=1.0, w_th=1.0, v_threshold=None),
    ]
    for ci, qsd in enumerate(specs):
        if qsd["family"] == "goal_progress":
            q = G.q_goal_progress(qsd["tau"], (qsd["w_v"], qsd["w_th"]))
        else:
            q = G.q_default((qsd["w_v"], qsd["w_th"]))
        if qsd["v_threshold"] is not None:
            q = mask_stationary(q, cs, qsd["v_threshold"])
        if ci == 2:
            lw0 = np.log(r.dirichlet(np.ones(space.size)))
            lw0[[3, 7]] = -np.inf
            b = G.JointBelief(lw0 - np.log(np.exp(lw0).sum()))
        else:
            b = G.init_belief(space)
        z = (5.0, 5.0)
        heading = 0.3
        rows = []
        for k in range(30):
            if k % 7 == 3:
                zn = z  # stationary observation -> fallback heading
            elif k % 11 == 5:
                zn = (z[0] + 0.9, z[1] - 0.4)  # beyond the set: snap mismatch
            else:
                zn = (z[0] + r.uniform(-0.15, 0.15), z[1] + r.uniform(-0.15, 0.15))
            try:
                nb = update_belief(b, G.HumanState(*z), G.HumanState(*zn), 0.1, cs, q, space,
                                   fallback_theta=heading)
                status = 0
            except ControlSnapMismatch:
                nb = update_belief(b, G.HumanState(*z), G.HumanState(*zn), 0.1, cs, q, space,
                                   fallback_theta=heading, snap_tol=math.inf)
                status = 1
            rows.append(dict(z=list(z), zn=list(zn), heading=heading, status=status,
                             prior=b.log_weights.tolist(), post=nb.log_weights.tolist()))
            if math.hypot(zn[0] - z[0], zn[1] - z[1]) > 1e-9:
                heading = math.atan2(zn[1] - z[1], zn[0] - z[0])
            b, z = nb, zn
        chains.append(dict(q=qsd, rows=rows))
    np.savez_compressed(os.path.join(OUT, "belief.npz"),
                        meta=json.dumps(dict(goals=goals.tolist(), betas=list(G.RationalitySet.log_spaced(5).betas),
                                             dt=0.1, chains=chains)))


def gen_smooth(G):
    from gridcast.occupancy import GridSpec, smooth_values
    r = np.random.default_rng(9)
    items = []
    arrs = []
    outs = []
    for (w, h, res, sig) in [(37, 23, 0.1, 0.1), (50, 50, 0.1, 0.15), (16, 40, 0.25, 0.3), (9, 9, 1.0, 0.7), (30, 30, 0.1, 0.0)]:
        v = r.integers(0, 50, (h, w)).astype(float)
        v[r.random((h, w)) < 0.6] = 0
        v /= max(v.sum(), 1.0)
        spec = GridSpec(w, h, res)
        items.append([w, h, res, sig])
        arrs.append(v.ravel())
        outs.append(smooth_values(v, spec, sig).ravel())
    np.savez_compressed(os.path.join(OUT, "smooth.npz"), meta=json.dumps(items),
                        x=np.concatenate(arrs), y=np.concatenate(outs))


def gen_multi(G):
    """sim.py:489-504 pattern: per-human predict with prefix (2, i), union_max, time union."""
    from gridcast import rng
    from gridcast.prediction import PredictionConfig, predict
    from gridcast.occupancy import union_max
    from oracle.model import control_grid
    v, th = control_grid(4, 24, 1.4)
    cs = G.ControlSet([G.ControlAction(float(a), float(b)) for a, b in zip(v, th)])
    starts = [(3.0, 3.0), (6.0, 3.0), (3.0, 6.0)]
    humans = []
    stacks = []
    seed = rng.derive_seed(0, 7, 4)
    cfg = PredictionConfig(n=1500, steps=8, dt=0.1, smoothing_sigma=0.1, seed=seed)
    spec = G.GridSpec(100, 100, 0.1)
    for i, s in enumerate(starts):
        goals = np.array([[s[0] + 2.0 * math.cos(a), s[1] + 2.0 * math.sin(a)] for a in (0.0, 1.6, 3.1, 4.7)])
        space = G.HypothesisSpace(G.RationalitySet.log_spaced(5), G.GoalSet(goals))
        b = _belief_for(G, space, cs, "random", 100 + i)
        q = G.q_goal_progress(0.5)
        st = predict(G.HumanState(*s), b, cfg, cs, q, space, spec, prefix=(2, i))
        stacks.append(st)
        humans.append(dict(start=list(s), goals=goals.tolist(), log_w=b.log_weights.tolist()))
    from gridcast.occupancy import union
    layers = np.stack([union_max([s.grid(k) for s in stacks]).values for k in range(cfg.steps)])
    tu = np.maximum.accumulate(layers, axis=0)
    # the "independent" union 1 - prod(1 - p) (occupancy.py:180-184)
    ind = np.stack([union([s.grid(k) for s in stacks], mode="independent").values for k in range(cfg.steps)])
    np.savez_compressed(os.path.join(OUT, "multi.npz"),
                        meta=json.dumps(dict(humans=humans, seed=str(seed), n=cfg.n, steps=cfg.steps,
                                             dt=cfg.dt, sigma=cfg.smoothing_sigma)),
                        union=layers.astype(np.float64), time_union=tu,
                        independent=ind, independent_tu=np.maximum.accumulate(ind, axis=0))


def gen_exact(G):
    from gridcast.prediction import exact_predict
    case = predict_cases()["lattice"]
    cs, space, q, spec = _spec(G, case)
    b = G.JointBelief.from_probs([0.35, 0.35, 0.15, 0.15])
    st = exact_predict(G.HumanState(4.5, 4.5), b, 3, 1.0, cs, q, space, spec)
    np.savez_compressed(os.path.join(OUT, "exact.npz"), log_w=b.log_weights, layers=st.layers)
    # a grid control set on a 30x24 grid (largest instances within the 2e6 cap), goal
    # progress, stationary mask and q_default
    from gridcast.belief import mask_stationary
    from oracle.model import control_grid
    v, th = control_grid(3, 8, 1.2)
    cs2 = G.ControlSet([G.ControlAction(float(a), float(t)) for a, t in zip(v, th)])
    space2 = G.HypothesisSpace(G.RationalitySet((0.5, 3.0)), G.GoalSet(np.array([[2.5, 1.0], [0.4, 2.0]])))
    spec2 = G.GridSpec(30, 24, 0.1)
    r = np.random.default_rng(4)
    b2 = G.JointBelief.from_probs(r.dirichlet(np.ones(4)))
    out = {}
    for tag, q2 in (("gp", G.q_goal_progress(0.5)), ("mask", mask_stationary(G.q_goal_progress(0.5), cs2, 0.7)),
                    ("def", G.q_default((0.5, 0.2)))):
        st2 = exact_predict(G.HumanState(1.43, 1.17), b2, 6, 0.2, cs2, q2, space2, spec2)
        out[tag] = st2.layers
    np.savez_compressed(os.path.join(OUT, "exact_grid.npz"), log_w=b2.log_weights, v=v, theta=th, **out)


def gen_collision(G):
    """collision_field (occupancy.py:222-239) on random layers, several radii/resolutions."""
    from gridcast.occupancy import GridSpec, OccupancyGrid, collision_field, collision_probability
    r = np.random.default_rng(21)
    items, xs, ys = [], [], []
    for (w, h, res, rad) in [(37, 23, 0.1, 0.25), (40, 40, 0.1, 0.5), (16, 30, 0.25, 0.6), (9, 9, 1.0, 0.0),
                             (50, 20, 0.05, 0.3)]:
        v = r.random((h, w)) * 0.05
        v[r.random((h, w)) < 0.5] = 0
        g = OccupancyGrid(GridSpec(w, h, res), v)
        items.append([w, h, res, rad, collision_probability(g, (w * res * 0.4, h * res * 0.6), rad)])
        xs.append(v.ravel())
        ys.append(collision_field(g, rad).ravel())
    np.savez_compressed(os.path.join(OUT, "collision.npz"), meta=json.dumps(items),
                        x=np.concatenate(xs), y=np.concatenate(ys))


def gen_gcst(G):
    """A stack file written by the reference (gridio.py:36-51) for format round trips."""
    from gridcast.gridio import save_stack
    from gridcast.occupancy import GridSpec
    from gridcast.prediction import PredictionStack
    r = np.random.default_rng(5)
    spec = GridSpec(12, 7, 0.25, (-1.5, 2.0))
    st = PredictionStack(spec, r.random((3, 7, 12)), 4.5, 0.2)
    save_stack(st, os.path.join(OUT, "stack_ref.grd"))


def gen_mppi(G):
    """mppi_step (planners/mppi.py:149-243) with and without a prediction stack."""
    from gridcast.planners.mppi import MppiConfig, mppi_step
    from gridcast.agents import RobotState
    from gridcast.occupancy import GridSpec
    from gridcast.prediction import PredictionStack
    r = np.random.default_rng(8)
    spec = GridSpec(60, 40, 0.1)
    layers = np.zeros((12, 40, 60))
    for k in range(12):
        layers[k, 15:25, 20 + k:30 + k] = r.random((10, 10)) * 0.2
    stack = PredictionStack(spec, layers, 0.0, 0.1)
    z = RobotState(1.0, 2.0, 0.4, 0.3)
    goal = RobotState(5.0, 2.2, 0.0, 0.0)
    out = {}
    for tag, st, qc, n in (("nostack", None, False, 512), ("stack", stack, False, 700), ("quad", stack, True, 300)):
        cfg = MppiConfig(horizon=20, rollouts=n, dt=0.1, quadratic_control_cost=qc, seed=3)
        nominal = r.normal(0, 0.2, (20, 2))
        controls, diag = mppi_step(z, nominal, goal, st, cfg, seed=11)
        out[tag + "_nominal"] = nominal
        out[tag + "_controls"] = controls
        out[tag + "_costs"] = diag.costs
    np.savez_compressed(os.path.join(OUT, "mppi.npz"), layers=layers, **out)


def _sparse_counts(counts_list):
    """(T, H, W) per-step counts -> (idx (nnz, 3) int32 [t, iy, ix], val int32)."""
    idx, val = [], []
    for t, c in enumerate(counts_list):
        iy, ix = np.nonzero(c)
        idx.append(np.stack([np.full(len(iy), t), iy, ix], 1))
        val.append(c[iy, ix])
    return np.concatenate(idx).astype(np.int32), np.concatenate(val).astype(np.int32)


def _sparse_layers(layers):
    nz = np.nonzero(layers)
    return np.stack(nz, 1).astype(np.int32), layers[nz]


def _digest(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _scene_beliefs(G, sc, n_updates=10):
    """sim.py:455-485 over the scene's warm-up track: per human the posterior after
    n_updates observations (ControlSnapMismatch -> retry with snap_tol=inf), the last
    heading and the stationary flag."""
    from gridcast.belief import ControlSnapMismatch, update_belief
    cs = G.ControlSet.grid(4, 24, 1.4)
    q = G.q_goal_progress(0.5)
    out = []
    for i, sp in enumerate(sc.spaces):
        space = G.HypothesisSpace(G.RationalitySet.log_spaced(5), G.GoalSet(np.array(sp.goals.positions)))
        b = G.init_belief(space)
        heading, stationary = 0.0, False
        for k in range(1, n_updates + 1):
            prev = G.HumanState(*sc.warmup_track[k - 1][i])
            obs = G.HumanState(*sc.warmup_track[k][i])
            try:
                b = update_belief(b, prev, obs, 0.1, cs, q, space, fallback_theta=heading)
            except ControlSnapMismatch:
                b = update_belief(b, prev, obs, 0.1, cs, q, space, fallback_theta=heading, snap_tol=math.inf)
            moved = math.hypot(obs.x - prev.x, obs.y - prev.y)
            stationary = moved / 0.1 < 0.05
            if moved > 1e-9:
                heading = math.atan2(obs.y - prev.y, obs.x - prev.x)
        out.append((space, b, heading, stationary))
    return cs, q, out


def gen_cfg3_cycle(G, steps=25):
    """The headline launch shape from the live reference: the bench's cfg3 scene (8 humans,
    each its own 4-goal HypothesisSpace, 262,144 particles, 400x400 @ 0.1 m, dt 0.02), the
    10th cycle of sim.run_episode's pattern (belief after 10 updates, seed
    derive_seed(0, 7, 9), prefix (2, i), masked Q when stationary), sigma 0.1, truncated to
    ``steps`` steps; per-human counts, hypothesis/position digests, the max union and its
    time union (sim.py:489-505)."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from gridcast import rng
    from gridcast.belief import mask_stationary
    from gridcast.occupancy import emplace_counts, smooth_values, union_max
    from gridcast.prediction import (ParticleBatch, PredictionConfig, predict, propagate_step,
                                     sample_hypotheses)
    from paper_2603_01122_b200.scenario import make_scene
    sc = make_scene("cfg3", cycles=2)
    cs, q, beliefs = _scene_beliefs(G, sc)
    qm = mask_stationary(q, cs, 0.5)
    spec = G.GridSpec(400, 400, 0.1)
    n, dt, sigma = sc.n, sc.dt, 0.1
    seed = rng.derive_seed(0, 7, 9)
    humans, per_layers, payload = [], [], {}
    for i, (space, b, heading, stationary) in enumerate(beliefs):
        z0 = G.HumanState(*sc.warmup_track[10][i])
        qi = qm if stationary else q
        pre = (rng.HUMAN_PREFIX, i)
        hyp = sample_hypotheses(b, n, seed, prefix=pre)
        batch = ParticleBatch.duplicated(z0, hyp)
        counts, layers = [], np.empty((steps, spec.height, spec.width))
        for t in range(1, steps + 1):
            batch = propagate_step(batch, cs, qi, space, dt, seed, step=t, workers=8, prefix=pre)
            c = emplace_counts(batch.xy, spec)
            counts.append(c.astype(np.int64))
            layers[t - 1] = smooth_values(c / n, spec, sigma)
        if i == 0:  # the loop above is predict() (prediction.py:243-255) verbatim: check it
            cfg = PredictionConfig(n=n, steps=steps, dt=dt, smoothing_sigma=sigma, seed=seed)
            st = predict(z0, b, cfg, cs, qi, space, spec, workers=8, prefix=pre)
            assert np.array_equal(st.layers, layers)
        per_layers.append(layers)
        ci, cv = _sparse_counts(counts)
        payload[f"count_idx_{i}"], payload[f"count_val_{i}"] = ci, cv
        li, lv = _sparse_layers(layers)
        payload[f"layer_idx_{i}"], payload[f"layer_val_{i}"] = li, lv
        humans.append(dict(start=[z0.x, z0.y], goals=np.asarray(space.goals.positions).tolist(),
                           log_w=b.log_weights.tolist(), stationary=bool(stationary), heading=heading,
                           hyp_sha256=_digest(hyp.astype(np.int32)),
                           xy_sha256=_digest(batch.xy.astype(np.float32))))
        print("cfg3_cycle human", i, "nnz", len(cv), "stationary", stationary)
    u = np.stack([union_max([G.OccupancyGrid(spec, L[k]) for L in per_layers]).values for k in range(steps)])
    tu = np.maximum.accumulate(u, axis=0)
    payload["union_idx"], payload["union_val"] = _sparse_layers(u)
    payload["tunion_idx"], payload["tunion_val"] = _sparse_layers(tu)
    meta = dict(n=n, steps=steps, dt=dt, sigma=sigma, seed=str(seed), cycle=9, grid=[400, 400, 0.1, [0.0, 0.0]],
                warmup_track=np.asarray(sc.warmup_track).tolist(), humans=humans,
                betas=list(G.RationalitySet.log_spaced(5).betas))
    np.savez_compressed(os.path.join(OUT, "cfg3_cycle.npz"), meta=json.dumps(meta), **payload)


def gen_long_cfg4(G, n=4096, steps=500):
    """A cfg4 human (T = 500, dt 0.02, 400x400): its reachable windows (285 x 285 cells at the
    last step) exceed shared memory, so K2 takes the global-histogram path."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from gridcast.occupancy import emplace_counts, smooth_values
    from gridcast.prediction import ParticleBatch, propagate_step, sample_hypotheses
    from oracle import model
    from paper_2603_01122_b200.scenario import make_scene
    sc = make_scene("cfg4_rank", cycles=2, humans=1)
    cs, q, beliefs = _scene_beliefs(G, sc)
    space, b, _, _ = beliefs[0]
    spec = G.GridSpec(400, 400, 0.1)
    dt, sigma, seed, pre = sc.dt, 0.1, 5, (2, 0)
    z0 = G.HumanState(*sc.warmup_track[10][0])
    hyp = sample_hypotheses(b, n, seed, prefix=pre)
    batch = ParticleBatch.duplicated(z0, hyp)
    counts = []
    keep_steps = [0, 249, steps - 1]
    layers = []
    for t in range(1, steps + 1):
        batch = propagate_step(batch, cs, q, space, dt, seed, step=t, workers=8, prefix=pre)
        c = emplace_counts(batch.xy, spec)
        counts.append(c.astype(np.int64))
        if t - 1 in keep_steps:
            layers.append(smooth_values(c / n, spec, sigma))
    ci, cv = _sparse_counts(counts)
    tb = model.make_tables(cs.v, cs.theta, dt, model.QSpec("goal_progress", 0.5))
    meta = dict(n=n, steps=steps, dt=dt, sigma=sigma, seed=seed, prefix=list(pre), grid=[400, 400, 0.1, [0.0, 0.0]],
                z0=[z0.x, z0.y], goals=np.asarray(space.goals.positions).tolist(),
                betas=list(G.RationalitySet.log_spaced(5).betas))
    li, lv = _sparse_layers(np.stack(layers))
    np.savez_compressed(os.path.join(OUT, "long_cfg4.npz"), meta=json.dumps(meta), log_w=b.log_weights,
                        hyp=hyp.astype(np.int32), xy_last=batch.xy.astype(np.float32), count_idx=ci, count_val=cv,
                        layer_steps=np.array(keep_steps), layer_idx=li, layer_val=lv,
                        sx=tb.sx, sy=tb.sy, at=tb.at, pen=tb.pen, dispx=tb.dispx, dispy=tb.dispy, keep=tb.keep,
                        q_kind=np.int32(tb.q_kind))
    print("long_cfg4 nnz", len(cv))


def gen_uniforms(G):
    """The reference's own random draws of the cfg1_s0 case, drawn by its rng module exactly
    as sample_hypotheses (prediction.py:128-131) and propagate_step (prediction.py:186-192)
    draw them: hypothesis u (n,) float64 and per-step chunk uniforms (T, n) float32."""
    from gridcast import rng
    case = predict_cases()["cfg1_s0"]
    n, steps, seed, pre = case["n"], case["steps"], case["seed"], tuple(case["prefix"])
    hyp_u = rng.stream(seed, *pre, rng.HYPOTHESIS_DRAWS).random(n)
    u = np.empty((steps, n), dtype=np.float32)
    for t in range(1, steps + 1):
        for a, b, c in rng.chunk_ranges(n, 1024):
            u[t - 1, a:b] = rng.stream(seed, *pre, rng.STEP_DRAWS, t, c).random(b - a, dtype=np.float32)
    np.savez_compressed(os.path.join(OUT, "uniforms_cfg1.npz"), hyp_u=hyp_u, step_u=u)


GENERATORS = dict(philox=lambda G: gen_philox(G), exp=lambda G: gen_exp(), predict=gen_predict, belief=gen_belief,
                  smooth=gen_smooth, multi=gen_multi, exact=gen_exact, collision=gen_collision, gcst=gen_gcst,
                  mppi=gen_mppi, naive=gen_naive, cfg3_cycle=gen_cfg3_cycle, long_cfg4=gen_long_cfg4,
                  uniforms=gen_uniforms)


def main():
    os.makedirs(OUT, exist_ok=True)
    G = _ref()
    names = sys.argv[1:] or list(GENERATORS)
    for name in names:
        GENERATORS[name](G)
    import platform
    with open(os.path.join(OUT, "PROVENANCE.txt"), "w") as f:
        f.write(f"generated by oracle/gen_golden.py from {REF}\n")
        f.write(f"numpy {np.__version__}; python {platform.python_version()}; {platform.machine()}\n")


if __name__ == "__main__":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    main()
