"""GPU: gc_union_tiles, the gather / scatter of the sparse cross-GPU max-reduce of the fused
grid (engine.sparse_max_reduce), against a torch restatement -- partial edge tiles, both
dtypes -- and the sparse merge of two engines' unions (human shards) against one engine's
union over all humans."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2603_01122_b200.engine import CycleEngine, EngineConfig, union_tiles  # noqa: E402
from paper_2603_01122_b200.scenario import make_scene  # noqa: E402


def _ref_pack(u, ids):
    T, H, W = u.shape
    ntx, nty = -(-W // 32), -(-H // 32)
    out = torch.zeros((len(ids), 32, 32), dtype=u.dtype)
    for i, tid in enumerate(ids):
        t, rem = divmod(int(tid), ntx * nty)
        ty, tx = divmod(rem, ntx)
        blk = u[t, ty * 32:(ty + 1) * 32, tx * 32:(tx + 1) * 32]
        out[i, :blk.shape[0], :blk.shape[1]] = blk
    return out


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_union_tiles_gather_scatter(dtype):
    g = torch.Generator().manual_seed(5)
    T, H, W = 7, 100, 70  # 4 x 3 tiles per layer, partial edge tiles
    u = torch.rand((T, H, W), generator=g, dtype=torch.float64).to(dtype)
    u[u < 0.5] = 0
    ntiles = T * 4 * 3
    ids = torch.randperm(ntiles, generator=g)[:30].sort().values.to(torch.int32)
    du = u.cuda()
    packed = torch.full((len(ids), 32, 32), -1.0, dtype=dtype, device="cuda")
    union_tiles(du, ids.cuda(), packed, unpack=False)
    torch.testing.assert_close(packed.cpu(), _ref_pack(u, ids), rtol=0, atol=0)
    # scatter: every listed tile's in-grid cells overwritten, everything else untouched
    dst = torch.full_like(du, 3.0)
    union_tiles(dst, ids.cuda(), packed, unpack=True)
    want = torch.full_like(u, 3.0)
    ntx, nty = 3, 4
    for tid in ids.tolist():
        t, rem = divmod(tid, ntx * nty)
        ty, tx = divmod(rem, ntx)
        want[t, ty * 32:(ty + 1) * 32, tx * 32:(tx + 1) * 32] = u[t, ty * 32:(ty + 1) * 32, tx * 32:(tx + 1) * 32]
    torch.testing.assert_close(dst.cpu(), want, rtol=0, atol=0)


def test_sparse_merge_of_human_shards_equals_one_engine():
    """Two engines with disjoint humans (the multi-GPU human sharding, global human ids in
    the streams) merged by OR-ing their union-tile flags, packing the flagged tiles, taking
    the max and scattering back -- what sparse_max_reduce does over NCCL -- equal one
    engine's fused union over all humans, bit for bit."""
    sc = make_scene("cfg2", cycles=4, humans=4)
    cfg = EngineConfig(n=8192, steps=24, dt=sc.dt, union_dtype="float64")
    track = np.concatenate([sc.warmup_track[1:], sc.track])

    def run(ids):
        eng = CycleEngine(sc.control_set, sc.q, [sc.spaces[i] for i in ids], sc.spec, cfg, human_ids=ids)
        eng.prime(sc.warmup_track[0][ids])
        for k in range(3):
            eng.stage(track[k][ids], buf=0)
            eng.run_cycle(buf=0)
        torch.cuda.synchronize()
        eng.check_errors()
        return eng

    full = run([0, 1, 2, 3])
    a, b = run([0, 2]), run([1, 3])
    flags = torch.maximum(a.utile[0], b.utile[0])
    ids = torch.nonzero(flags.reshape(-1)).reshape(-1).to(torch.int32)
    pa = torch.empty((len(ids), 32, 32), dtype=torch.float64, device="cuda")
    pb = torch.empty_like(pa)
    union_tiles(a.unions[0], ids, pa, unpack=False)
    union_tiles(b.unions[0], ids, pb, unpack=False)
    merged = a.unions[0].clone()
    union_tiles(merged, ids, torch.maximum(pa, pb), unpack=True)
    torch.cuda.synchronize()
    assert torch.equal(merged, full.unions[0])
    assert torch.equal(flags, full.utile[0])
    assert 0 < len(ids) < flags.numel()


@pytest.mark.parametrize("sigma", [0.03, 0.05, 0.1, 0.13, 0.2])
def test_epilogue_radii_match_the_standalone_smoother(sigma):
    """K3 for every radius the dispatch distinguishes (k_epilogue_r<1..3>, the runtime-radius
    kernel for 4 and 6): the fused epilogue's layers equal the standalone smoother
    (gc_smooth_layers, itself pinned to the reference's smooth_values) applied to the
    unsmoothed layers of the same predict, and the max union equals the max of the layers."""
    import paper_2603_01122_b200 as G
    from paper_2603_01122_b200 import prediction as PR
    from paper_2603_01122_b200.occupancy import smooth_values
    cs, q = G.ControlSet.grid(4, 24, 1.4), G.q_goal_progress(0.5)
    tab = PR.action_tables(cs, q, 0.1, torch.device("cuda"))
    spec = G.GridSpec(90, 70, 0.1)
    space = G.HypothesisSpace(G.RationalitySet((0.5, 3.0)), G.GoalSet(np.array([[7.0, 5.0], [1.0, 1.0]])))
    lw = np.log(np.array([0.4, 0.1, 0.3, 0.2]))
    jobs = [PR.HumanJob(G.HumanState(4.0 + i, 3.0), lw, space.beta_of, space.goal_xy_of, 11, (2, i), 0)
            for i in range(2)]
    raw = PR.run_predict(jobs, [tab], 20000, 12, 0.1, 0.0, spec, "production")["layers"].cpu().numpy()
    out = PR.run_predict(jobs, [tab], 20000, 12, 0.1, sigma, spec, "production", union64=True)
    lay = out["layers"].cpu().numpy()
    for h in range(2):
        for t in (0, 5, 11):
            np.testing.assert_allclose(lay[h, t], smooth_values(raw[h, t], spec, sigma), rtol=0, atol=1e-15)
    np.testing.assert_array_equal(out["union64"].cpu().numpy(), lay.max(axis=0))


@pytest.mark.parametrize("sigma", [0.13, 0.186])
def test_large_smoothing_radii_match_the_reference_operator(sigma):
    """Radii far above the bench's 3 cells (39 and 56 = GC_MAX_SMOOTH_RADIUS on a 1 cm grid):
    the fused epilogue's layers and the standalone smoother both equal the oracle's dense
    restatement of smooth_values (bit-identical to the reference, tests/test_oracle_golden.py)
    within 1e-15; one radius more raises NotImplementedError like any unsupported input."""
    import paper_2603_01122_b200 as G
    from paper_2603_01122_b200 import prediction as PR
    from paper_2603_01122_b200.occupancy import smooth_layers_device
    from oracle import predict as OP
    cs, q = G.ControlSet.grid(4, 24, 1.4), G.q_goal_progress(0.5)
    tab = PR.action_tables(cs, q, 0.05, torch.device("cuda"))
    spec = G.GridSpec(200, 160, 0.01)
    space = G.HypothesisSpace(G.RationalitySet((0.5, 3.0)), G.GoalSet(np.array([[1.7, 1.2], [0.2, 0.3]])))
    lw = np.log(np.array([0.4, 0.1, 0.3, 0.2]))
    jobs = [PR.HumanJob(G.HumanState(1.0, 0.8), lw, space.beta_of, space.goal_xy_of, 5, (2, 0), 0)]
    raw = PR.run_predict(jobs, [tab], 20000, 4, 0.05, 0.0, spec, "production")["layers"]
    out = PR.run_predict(jobs, [tab], 20000, 4, 0.05, sigma, spec, "production", union64=True)
    lay = out["layers"].cpu().numpy()
    alone = smooth_layers_device(raw[0].contiguous(), spec, sigma).cpu().numpy()
    g = OP.Grid(spec.width, spec.height, spec.resolution)
    for t in range(4):
        want = OP.smooth_dense(raw[0, t].cpu().numpy(), g, sigma)
        np.testing.assert_allclose(lay[0, t], want, rtol=0, atol=1e-15)
        np.testing.assert_allclose(alone[t], want, rtol=0, atol=1e-15)
    np.testing.assert_array_equal(out["union64"].cpu().numpy(), lay.max(axis=0))
    with pytest.raises(NotImplementedError):
        smooth_layers_device(raw[0].contiguous(), spec, 0.19)
