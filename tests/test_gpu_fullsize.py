"""GPU, BASELINE.json full sizes: size-independent properties of the whole cycle.

The oracle cannot run these sizes in seconds, so the checks are the properties the domain
guarantees for any size: every particle lands in exactly one cell per step (the u32 count
windows of each (human, step) sum to n -- nothing lost or double-counted by the shared-
memory windows, the touched-word flush or the global-atomics path), the horizon chunking
is bit-identical to one launch, unions are finite and within [0, 1], and a stationary
human propagates with the stationary-masked table.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2603_01122_b200.engine import CycleEngine, EngineConfig  # noqa: E402
from paper_2603_01122_b200.scenario import make_scene  # noqa: E402


def window_sums(eng):
    """(humans, steps) sums of the windowed u32 counts."""
    geo = eng.geo
    c = eng.counts.cpu().numpy().view(np.uint32).astype(np.int64)
    out = np.zeros((eng.n_humans, eng.cfg.steps), dtype=np.int64)
    start = eng.d_start.cpu().numpy().reshape(-1, 2)
    for h in range(eng.n_humans):
        for t in range(eng.cfg.steps):
            _, _, w, hh = geo.window(start[h], t)
            base = h * geo.human_stride + geo.step_off[t]
            out[h, t] = c[base:base + w * hh].sum()
    return out


def run(name, mode="production", chunks=0, humans=8, n=None, stationary=(), budget_kb=0.0, hist_path="global"):
    sc = make_scene(name, cycles=2, humans=humans)
    n = n or sc.n
    cfg = EngineConfig(n=n, steps=sc.steps, dt=sc.dt, smoothing_sigma=0.1, seed=3, mode=mode,
                       window_budget_kb=budget_kb, hist_path=hist_path)
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, cfg)
    eng.prime(sc.prev_xy)
    obs = sc.track[0].copy()
    for i in stationary:
        obs[i] = sc.prev_xy[i]  # did not move -> stationary-masked Q (sim.py:480, :495)
    eng.stage(obs, buf=0)
    if chunks > 0:
        # capture() runs one warm-up cycle before capturing, so the replayed cycle is the
        # second belief update -- the same for every chunk count
        host = torch.empty(eng.unions[0].shape, dtype=eng.unions[0].dtype).pin_memory() if chunks > 1 else None
        eng.capture(buf=0, chunks=chunks, d2h=host).replay()
    else:
        eng.run_cycle(buf=0)
    torch.cuda.synchronize()
    eng.check_errors()
    return eng


@pytest.mark.parametrize("hist_path", ["global", "smem"])
def test_cfg3_production_cycle_conserves_particles_and_bounds(hist_path):
    """cfg3: 8 humans x 262,144 particles x 250 steps (both histogram paths)."""
    eng = run("cfg3", hist_path=hist_path)
    np.testing.assert_array_equal(window_sums(eng), eng.cfg.n)
    u = eng.unions[0]
    assert torch.isfinite(u).all() and float(u.min()) >= 0.0 and float(u.max()) <= 1.0
    # every layer holds mass: the max union of 8 normalised layers has sum in [1, 8]
    s = u.double().sum(dim=(1, 2)).cpu().numpy()
    assert np.all(s > 0.99) and np.all(s < 8.01)


@pytest.mark.parametrize("mode", ["production", "reference"])
def test_cfg3_chunked_equals_single_launch(mode):
    """Full-size horizon chunking (6 tapered chunks) is bit-identical to one launch."""
    kw = dict(humans=2) if mode == "reference" else {}
    a = run("cfg3", mode=mode, chunks=1, **kw)
    ua = a.unions[0].cpu().numpy()
    del a
    b = run("cfg3", mode=mode, chunks=6, **kw)
    np.testing.assert_array_equal(b.unions[0].cpu().numpy(), ua)


def test_cfg4_shard_global_histogram_path_conserves_particles():
    """cfg4's per-GPU shard (8 humans x 1,048,576 particles x 500 steps): the late reachable
    windows exceed shared memory, so K2 adds those steps straight into the L2 count windows."""
    eng = run("cfg4_rank")
    np.testing.assert_array_equal(window_sums(eng), eng.cfg.n)
    u = eng.unions[0]
    assert torch.isfinite(u).all() and float(u.max()) <= 1.0


@pytest.mark.parametrize("mode", ["production", "reference"])
def test_long_horizon_window_split_equals_global_path(mode):
    """T = 500 (cfg4 shape): with hist_path="smem" the engine runs steps 1..264 on shared-
    memory windows and the rest on global reductions (two launches, particle state handed
    over); bit-identical to the whole horizon on the (default) global path."""
    n = 65536 if mode == "production" else 4096
    a = run("cfg4_rank", mode=mode, humans=2, n=n, budget_kb=46.0, hist_path="smem")
    assert a.window_bounds() == [(1, 265), (265, 501)]
    np.testing.assert_array_equal(window_sums(a), n)
    ua = a.unions[0].cpu().numpy()
    del a
    b = run("cfg4_rank", mode=mode, humans=2, n=n, budget_kb=0)
    assert b.window_bounds() == [(1, 501)]
    np.testing.assert_array_equal(b.unions[0].cpu().numpy(), ua)


def test_stationary_human_uses_masked_table_and_ragged_n():
    """A human who did not move propagates with mask_stationary(v <= 0.5) in the same
    launch as moving humans (per-human table ids); ragged n (partial CTA)."""
    eng = run("cfg3", humans=3, n=3333, stationary=(1,))
    assert list(eng.h_tid) == [0, 1, 0]
    np.testing.assert_array_equal(window_sums(eng), 3333)
    # with v <= 0.467 m/s the stationary human covers at most 0.467 * 5 s = 2.3 m
    geo = eng.geo
    c = eng.counts.cpu().numpy().view(np.uint32)
    start = eng.d_start.cpu().numpy().reshape(-1, 2)
    t = eng.cfg.steps - 1
    x0, y0, w, hh = geo.window(start[1], t)
    base = 1 * geo.human_stride + geo.step_off[t]
    win = c[base:base + w * hh].reshape(hh, w)
    ys, xs = np.nonzero(win)
    cx, cy = start[1] / 0.1
    reach = np.hypot(xs + x0 + 0.5 - cx, ys + y0 + 0.5 - cy).max() * 0.1
    assert reach < 0.467 * eng.cfg.steps * eng.cfg.dt + 0.3


def test_cfg3_production_tv_within_reference_seed_spread():
    """The north star's production-mode criterion at the headline size: per (human, step)
    layers of the production sampler vs the bit-exact reference mode on the same inputs,
    TV bounded by the reference's own seed-to-seed TV (1.5x + 0.005), all 8 x 250 layers."""
    sc = make_scene("cfg3", cycles=2, humans=8)
    layers = {}
    for tag, seed, mode in (("a", 1, "reference"), ("b", 2, "reference"), ("p", 3, "production")):
        cfg = EngineConfig(n=sc.n, steps=sc.steps, dt=sc.dt, smoothing_sigma=0.1, seed=seed, mode=mode,
                           per_human_layers=True)
        eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, cfg)
        eng.prime(sc.prev_xy)
        eng.stage(sc.track[0], buf=0)
        eng.run_cycle(buf=0)
        torch.cuda.synchronize()
        eng.check_errors()
        layers[tag] = eng.layers.clone()
        del eng
        torch.cuda.empty_cache()

    def tv(u, v):  # (humans, steps) total variation
        return 0.5 * (u - v).abs().sum(dim=(2, 3))

    spread = tv(layers["a"], layers["b"])
    got = torch.maximum(tv(layers["p"], layers["a"]), tv(layers["p"], layers["b"]))
    print(f"cfg3 per-layer TV: production vs reference max {float(got.max()):.4f} mean {float(got.mean()):.4f}; "
          f"reference seed spread max {float(spread.max()):.4f} mean {float(spread.mean()):.4f}")
    assert bool((got <= 1.5 * spread + 0.005).all()), (float(got.max()), float(spread.max()))
    # and every layer is a probability distribution
    mass = layers["p"].sum(dim=(2, 3))
    assert float((mass - 1).abs().max()) < 1e-9


def test_cfg3_graph_replays_are_bitwise_reproducible():
    """The captured cycle replayed twice on the same inputs (same cycle seed) gives the same
    fused union bit for bit: production streams are counter-based, counts are integer
    atomics, the union is an order-independent max."""
    sc = make_scene("cfg3", cycles=2, humans=8)
    cfg = EngineConfig(n=sc.n, steps=sc.steps, dt=sc.dt, smoothing_sigma=0.1, seed=3, mode="production")
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, cfg)
    eng.prime(sc.prev_xy)
    eng.stage(sc.track[0], buf=0)
    g = eng.capture(buf=0, with_h2d=True, with_update=False)
    g.replay()
    torch.cuda.synchronize()
    first = eng.unions[0].cpu().numpy()
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(eng.unions[0].cpu().numpy(), first)
    assert first.max() > 0
