"""CPU, world_size 2 over gloo: the multi-GPU decomposition of a scene.

Humans are sharded across ranks with their GLOBAL index in the random-stream prefix
(HUMAN_PREFIX, i) (sim.py:493-499), each rank merges its own humans by max, and the
per-rank unions are merged into one fused grid by a max reduction
(engine.fused_reduce -- NCCL on the GPU box, gloo here).  The fused grid must equal the
single-process union over all humans for any partition (checked with the oracle, which
stands in for the per-rank CUDA predict on this GPU-less host).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import model
from oracle import predict as OP

N, T, DT, SIG, SEED = 600, 6, 0.1, 0.1, 12345
GRID = OP.Grid(60, 60, 0.1)


def humans():
    r = np.random.default_rng(3)
    out = []
    for i in range(5):
        s = r.uniform(1.5, 4.5, 2)
        goals = s + 2.0 * np.stack([np.cos(np.arange(4) * 1.57), np.sin(np.arange(4) * 1.57)], 1)
        beta_of, goal_of = model.hypothesis_tables(np.geomspace(0.1, 10, 5), goals)
        lw = np.log(r.dirichlet(np.ones(20)))
        out.append((s, lw - np.log(np.exp(lw).sum()), beta_of, goal_of))
    return out


def layers_of(i, hm, tb):
    s, lw, b, g = hm
    return OP.predict(s, lw, N, T, DT, SIG, SEED, tb, b, g, GRID, prefix=(2, i))["layers"]


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, shards, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_01122_b200.engine import fused_reduce
    v, th = model.control_grid(4, 24, 1.4)
    tb = model.make_tables(v, th, DT, model.QSpec())
    hs = humans()
    local = np.zeros((T, GRID.height, GRID.width))
    for i in shards[rank]:
        np.maximum(local, layers_of(i, hs[i], tb), out=local)
    u = torch.from_numpy(local)
    fused_reduce(u, dst=0)
    # timing rule of bench.py: the step time is the max over ranks
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        np.save(result_path, u.numpy())
        assert float(t.item()) == world
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("shards", [([0, 1, 2], [3, 4]), ([4, 0], [2, 1, 3])])
def test_fused_grid_equals_single_process_union(tmp_path, shards):
    path = str(tmp_path / "fused.npy")
    mp.spawn(_worker, args=(2, _free_port(), shards, path), nprocs=2, join=True)
    fused = np.load(path)
    v, th = model.control_grid(4, 24, 1.4)
    tb = model.make_tables(v, th, DT, model.QSpec())
    hs = humans()
    ref = OP.union_max([layers_of(i, h, tb) for i, h in enumerate(hs)])
    np.testing.assert_array_equal(fused, ref)


def test_scene_shards_are_disjoint_and_sized():
    from paper_2603_01122_b200.scenario import make_scene
    a = make_scene("cfg3", cycles=1, humans=8, human_offset=0)
    b = make_scene("cfg3", cycles=1, humans=8, human_offset=8)
    assert len(a.spaces) == len(b.spaces) == 8
    assert not np.allclose(a.starts, b.starts)
    assert a.n == 262144 and a.steps == 250


def _shard_worker(rank, world, port, result_path):
    """Each rank runs its block of one human's particles (streams keyed by the global
    particle index) and the u32 counts are summed across ranks (the particle-sharded
    path of engine.CycleEngine(particle_shard=...), counts_reduce = all_reduce(sum))."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    v, th = model.control_grid(4, 24, 1.4)
    tb = model.make_tables(v, th, DT, model.QSpec())
    s, lw, b, g = humans()[0]
    n_total = 3000
    hyp = OP.sample_hypotheses(lw, n_total, SEED, prefix=(2, 0))
    lo, hi = rank * n_total // world, (rank + 1) * n_total // world
    uni = np.stack([OP.step_uniforms(SEED, (2, 0), t, n_total)[lo:hi] for t in range(1, T + 1)])
    part = OP.predict(s, lw, hi - lo, T, DT, 0.0, SEED, tb, b, g, GRID, prefix=(2, 0), uniforms=uni,
                      hyp=hyp[lo:hi])["counts"]
    c = torch.from_numpy(part.astype(np.int64))
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    if rank == 0:
        np.save(result_path, c.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_particle_sharded_counts_sum_to_single_process(tmp_path):
    path = str(tmp_path / "counts.npy")
    mp.spawn(_shard_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    v, th = model.control_grid(4, 24, 1.4)
    tb = model.make_tables(v, th, DT, model.QSpec())
    s, lw, b, g = humans()[0]
    full = OP.predict(s, lw, 3000, T, DT, 0.0, SEED, tb, b, g, GRID, prefix=(2, 0))["counts"]
    np.testing.assert_array_equal(np.load(path), full)


def _independent_worker(rank, world, port, result_path):
    """Independent union across ranks: each rank holds prod(1 - p) of its humans
    (EngineConfig(union_partial=True)); fused_reduce(mode="independent") multiplies the
    partials (ReduceOp.PRODUCT); the receiving rank finishes 1 - prod on the GPU."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_01122_b200.engine import fused_reduce
    r = np.random.default_rng(7)
    layers = r.uniform(0.0, 0.3, size=(5, T, 12, 12))
    mine = layers[rank::world]
    miss = np.prod(1.0 - np.clip(mine, 0.0, 1.0), axis=0)
    u = torch.from_numpy(miss.copy())
    fused_reduce(u, dst=0, mode="independent", finish=False)
    if rank == 0:
        np.save(result_path, u.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_independent_union_partials_multiply_across_ranks(tmp_path):
    path = str(tmp_path / "miss.npy")
    mp.spawn(_independent_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    r = np.random.default_rng(7)
    layers = r.uniform(0.0, 0.3, size=(5, T, 12, 12))
    ref = OP.union_independent(list(layers))
    np.testing.assert_allclose(1.0 - np.load(path), ref, rtol=0, atol=1e-15)


def _torch_tile_op(union, ids, packed, unpack):
    """CPU restatement of gc_union_tiles (test infrastructure): tile id
    (t * nty + ty) * ntx + tx, 32 x 32 blocks, zeros outside the grid."""
    T, H, W = union.shape
    ntx, nty = -(-W // 32), -(-H // 32)
    for i, tid in enumerate(ids.tolist()):
        t, rem = divmod(tid, ntx * nty)
        ty, tx = divmod(rem, ntx)
        y0, x0 = ty * 32, tx * 32
        h, w = min(32, H - y0), min(32, W - x0)
        if unpack:
            union[t, y0:y0 + h, x0:x0 + w] = packed[i, :h, :w]
        else:
            packed[i].zero_()
            packed[i, :h, :w] = union[t, y0:y0 + h, x0:x0 + w]


def _tile_flags(u):
    T, H, W = u.shape
    ntx, nty = -(-W // 32), -(-H // 32)
    f = torch.zeros((T, nty, ntx), dtype=torch.uint8)
    for ty in range(nty):
        for tx in range(ntx):
            f[:, ty, tx] = (u[:, ty * 32:(ty + 1) * 32, tx * 32:(tx + 1) * 32] > 0).flatten(1).any(1).to(torch.uint8)
    return f


def _sparse_worker(rank, world, port, shards, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_01122_b200.engine import sparse_max_reduce
    v, th = model.control_grid(4, 24, 1.4)
    tb = model.make_tables(v, th, DT, model.QSpec())
    hs = humans()
    local = np.zeros((T, GRID.height, GRID.width))
    for i in shards[rank]:
        np.maximum(local, layers_of(i, hs[i], tb), out=local)
    u = torch.from_numpy(local)
    flags = _tile_flags(u)
    own = flags.clone()
    sparse_max_reduce(u, flags, dst=0, tile_op=_torch_tile_op)
    # the flags are OR-ed over the ranks: they cover this rank's own tiles
    assert bool((flags >= own).all())
    if rank == 0:
        np.save(result_path, u.numpy())
        np.save(result_path + ".flags.npy", flags.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("shards", [([0, 1, 2], [3, 4]), ([4], [0, 1, 2, 3])])
def test_sparse_tile_reduce_equals_single_process_union(tmp_path, shards):
    """engine.sparse_max_reduce (OR of the tile flags, pack the flagged tiles, max-reduce the
    packed buffers, scatter back) gives rank 0 the same fused grid as the dense reduce --
    the single-process union over all humans -- with a 60 x 60 grid whose edge tiles are
    partial (28 cells)."""
    path = str(tmp_path / "fused_sparse.npy")
    mp.spawn(_sparse_worker, args=(2, _free_port(), shards, path), nprocs=2, join=True)
    fused = np.load(path)
    v, th = model.control_grid(4, 24, 1.4)
    tb = model.make_tables(v, th, DT, model.QSpec())
    ref = OP.union_max([layers_of(i, h, tb) for i, h in enumerate(humans())])
    np.testing.assert_array_equal(fused, ref)
    np.testing.assert_array_equal(np.load(path + ".flags.npy"), _tile_flags(torch.from_numpy(ref)).numpy())
