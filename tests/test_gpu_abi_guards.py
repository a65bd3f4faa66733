"""GPU: the C ABI's own validation (the drop-in boundary must not trust its caller) and the
engine's reference semantics for a first, unprimed observation (sim.py:462-485)."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2603_01122_b200 as G  # noqa: E402
from paper_2603_01122_b200 import _lib  # noqa: E402
from paper_2603_01122_b200 import prediction as PR  # noqa: E402


def _args(n_hyp_per_human, max_win_cells=None, steps=6, n=512):
    """A reference-mode gc_predict launch of len(n_hyp_per_human) humans through ctypes."""
    dev = torch.device("cuda")
    cs = G.ControlSet.grid(4, 24, 1.4)
    q = G.q_goal_progress(0.5)
    tab = PR.action_tables(cs, q, 0.1, dev)
    spec = G.GridSpec(60, 60, 0.1)
    geo = PR.geometry(spec, steps, tab.max_step, 0.0, dev)
    H = len(n_hyp_per_human)
    off = np.concatenate([[0], np.cumsum(n_hyp_per_human)]).astype(np.int32)
    tot = max(int(off[-1]), 1)
    up = lambda a, t: torch.as_tensor(np.array(a, dtype=t), device=dev)  # noqa: E731
    keep = dict(
        start=up([[3.0, 3.0]] * H, np.float32), off=up(off, np.int32),
        beta=up(np.ones(tot), np.float32), goal=up(np.tile([[5.0, 5.0]], (tot, 1)), np.float32),
        cdf=up(np.linspace(1.0 / tot, 1.0, tot), np.float64), seed=up(np.zeros(H), np.uint64),
        pre=up(np.zeros((H, 4)), np.uint32), plen=up(np.zeros(H), np.int32), tid=up(np.zeros(H), np.int32),
        counts=torch.zeros(H * geo.human_stride, dtype=torch.int32, device=dev),
        err=torch.zeros(1, dtype=torch.int32, device=dev))
    a = _lib.PredictArgs()
    a.n_humans, a.n, a.steps, a.rng_mode = H, n, steps, _lib.GC_RNG_REFERENCE
    a.grid_w, a.grid_h, a.res32 = spec.width, spec.height, float(np.float32(0.1))
    a.d_start_xy, a.d_hyp_off = keep["start"].data_ptr(), keep["off"].data_ptr()
    a.d_beta32, a.d_goal32, a.d_cdf = keep["beta"].data_ptr(), keep["goal"].data_ptr(), keep["cdf"].data_ptr()
    a.d_seed, a.d_prefix, a.d_prefix_len = keep["seed"].data_ptr(), keep["pre"].data_ptr(), keep["plen"].data_ptr()
    keep["tarr"] = (_lib.ActionTable * 1)(tab.struct)
    a.h_tables, a.n_tables, a.d_table_id = keep["tarr"], 1, keep["tid"].data_ptr()
    a.d_step_r, a.d_step_off = geo.d_step_r.data_ptr(), geo.d_step_off.data_ptr()
    a.human_stride = geo.human_stride
    a.max_win_cells = geo.max_win_cells if max_win_cells is None else max_win_cells
    a.d_counts, a.d_error = keep["counts"].data_ptr(), keep["err"].data_ptr()
    return a, keep


def _run(a, keep):
    _lib.check(_lib.lib().gc_predict(ctypes.byref(a), None), "gc_predict")
    torch.cuda.synchronize()
    return int(keep["err"].item()) & 0xFFFFFFFF, int(keep["counts"].sum().item())


def test_predict_rejects_hypothesis_counts_outside_1_to_256():
    for ok in ([4, 4], [256, 1]):  # both ends of the range
        a, keep = _args(ok)
        word, total = _run(a, keep)
        assert word == 0 and total == 2 * 512 * 6
    for bad in ([4, 0], [257, 4]):
        a, keep = _args(bad)
        word, _ = _run(a, keep)
        assert word & _lib.GC_ERRBIT_HYPOTHESES
        with pytest.raises(ValueError):
            _lib.check_error_word(word)


def test_predict_rejects_underreported_window_capacity():
    a, keep = _args([4], max_win_cells=0)
    a.hist_path = _lib.GC_HIST_SMEM  # the shared-memory window is sized from max_win_cells
    word, total = _run(a, keep)
    assert word & _lib.GC_ERRBIT_WINDOW_CAPACITY and total == 0
    with pytest.raises(ValueError):
        _lib.check_error_word(word)


@pytest.mark.parametrize("bad", [1, -1, 7])
def test_predict_rejects_table_ids_outside_the_launch(bad):
    """A human whose table id does not name one of the launch's tables is not predicted
    (no read past the parameter bank's tables) and the launch reports it."""
    a, keep = _args([4, 4])
    keep["tid"][1] = bad
    word, total = _run(a, keep)
    assert word & _lib.GC_ERRBIT_TABLE_ID and total == 512 * 6  # human 0 only
    with pytest.raises(ValueError):
        _lib.check_error_word(word)


def test_engine_stage_rejects_non_finite_observations():
    from paper_2603_01122_b200.engine import CycleEngine, EngineConfig
    from paper_2603_01122_b200.scenario import make_scene
    sc = make_scene("cfg2", cycles=2, humans=2)
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, EngineConfig(n=1024, steps=8, dt=sc.dt))
    bad = np.array(sc.warmup_track[1], dtype=float)
    bad[1, 0] = np.nan
    with pytest.raises(ValueError):
        eng.stage(bad)
    with pytest.raises(ValueError):
        eng.stage(sc.warmup_track[1][:1])


def test_belief_update_rejects_too_many_hypotheses():
    from paper_2603_01122_b200.belief import belief_tables, launch_belief_update
    dev = torch.device("cuda")
    cs = G.ControlSet.grid(4, 24, 1.4)
    btab = belief_tables(cs, G.q_goal_progress(0.5), dev)
    nh = _lib.GC_MAX_HYPOTHESES + 2
    off = torch.tensor([0, nh], dtype=torch.int32, device=dev)
    beta = torch.ones(nh, dtype=torch.float64, device=dev)
    goal = torch.full((nh, 2), 5.0, dtype=torch.float64, device=dev)
    obs = torch.tensor([[1.0, 1.0, 1.1, 1.0]], dtype=torch.float64, device=dev)
    fb = torch.zeros(1, dtype=torch.float64, device=dev)
    lw = torch.full((nh,), -np.log(nh), dtype=torch.float64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    launch_belief_update(btab, off, beta, goal, obs, fb, lw, lw, st, 0.1, np.inf, 1, 1)
    torch.cuda.synchronize()
    assert int(st.item()) == _lib.GC_BAD_ARG


def test_engine_unprimed_first_cycle_predicts_without_update():
    """stage() before prime(): no belief update, unmasked table, then normal cycles."""
    from paper_2603_01122_b200.engine import CycleEngine, EngineConfig
    from paper_2603_01122_b200.scenario import make_scene
    sc = make_scene("cfg1", cycles=4)
    cfg = EngineConfig(n=sc.n, steps=sc.steps, dt=sc.dt, mode="reference")
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, cfg)
    prior = eng.posterior(0).copy()
    eng.stage(sc.track[0], buf=0)
    assert int(eng.h_tid[0]) == 0
    eng.run_cycle(buf=0)
    np.testing.assert_array_equal(eng.posterior(0), prior)  # no update on the first observation
    with pytest.raises(RuntimeError):
        eng.capture(buf=0)  # a graph always contains the update
    eng.stage(sc.track[1], buf=1)  # now primed: the update runs
    eng.run_cycle(buf=1)
    b = G.update_belief(G.JointBelief(prior), G.HumanState(*sc.track[0][0]), G.HumanState(*sc.track[1][0]),
                        cfg.obs_dt, sc.control_set, sc.q, sc.spaces[0], snap_tol=np.inf)
    np.testing.assert_allclose(np.exp(eng.posterior(0)), np.exp(b.log_weights), rtol=1e-9, atol=0)
    eng.check_errors()


def test_assume_qg_fast_kernel_is_bit_identical_and_guarded(monkeypatch):
    """Production launches whose hypotheses admit the top-speed normalisation run the kernel
    without the max-shift fallback (gc_predict_args.assume_qg, set by the mirror): its
    outputs equal the general kernel's bit for bit; a launch that claims assume_qg for a
    hypothesis that needs the fallback (beta = 300) is reported, not silently wrong."""
    import paper_2603_01122_b200.prediction as PRm
    cs = G.ControlSet.grid(4, 24, 1.4)
    q = G.q_goal_progress(0.5)
    tab = PR.action_tables(cs, q, 0.1, torch.device("cuda"))
    spec = G.GridSpec(200, 200, 0.1)

    def run(betas, force=None):
        space = G.HypothesisSpace(G.RationalitySet(betas), G.GoalSet(np.array([[15.0, 12.0], [4.0, 14.0]])))
        lw = np.log(np.full(len(space.beta_of), 1.0 / len(space.beta_of)))
        job = PR.HumanJob(G.HumanState(9.0, 9.0), lw, space.beta_of, space.goal_xy_of, 7, (2, 0), 0)
        if force is not None:
            monkeypatch.setattr(PRm, "assume_qg", lambda *a: force)
        out = PR.run_predict([job] * 3, [tab], 200000, 30, 0.1, 0.1, spec, "production", per_human_layers=False,
                             union64=True)
        monkeypatch.undo()
        return out

    betas = (0.1, 1.0, 10.0)
    from paper_2603_01122_b200.tables import assume_qg
    assert assume_qg([tab], [np.array(betas)]) and not assume_qg([tab], [np.array([300.0])])
    fast, general = run(betas), run(betas, force=False)
    assert torch.equal(fast["counts"], general["counts"]) and torch.equal(fast["union64"], general["union64"])
    with pytest.raises(ValueError, match="assume_qg"):
        run((300.0,), force=True)


def test_predict_and_update_reject_control_sets_above_the_action_limit():
    """GC_MAX_ACTIONS + 1 actions: gc_predict and gc_belief_update refuse the launch with
    GC_BAD_ARG (a ValueError in the mirror) instead of overrunning the shared tables."""
    m = _lib.GC_MAX_ACTIONS + 1
    r = np.random.default_rng(0)
    cs = G.ControlSet([G.ControlAction(float(v), float(t))
                       for v, t in zip(r.uniform(0.1, 1.5, m), r.uniform(-3.1, 3.1, m))])
    q = G.q_goal_progress(0.5)
    space = G.HypothesisSpace(G.RationalitySet((1.0,)), G.GoalSet(np.array([[5.0, 5.0]])))
    belief = G.init_belief(space)
    cfg = G.PredictionConfig(n=256, steps=2, dt=0.1, smoothing_sigma=0.0, seed=0, mode="production")
    with pytest.raises(ValueError, match="512 actions"):
        G.predict(G.HumanState(1.0, 1.0), belief, cfg, cs, q, space, G.GridSpec(40, 40, 0.1))
    with pytest.raises(ValueError, match="512 actions"):
        G.update_belief(belief, G.HumanState(1.0, 1.0), G.HumanState(1.05, 1.0), 0.1, cs, q, space)
