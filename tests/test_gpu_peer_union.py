"""GPU, two processes on cuda:0: the peer-memory fused union (peer.PeerUnion).

Each rank runs a CycleEngine over its shard of the humans (global ids in the random
streams, sim.py:493-499) whose K3 atomicMax-es straight into the grid owned by rank 0
through a CUDA IPC mapping -- the multi-GPU fused grid without an NCCL reduce.  Two
processes on one GPU exercise the same IPC export/import and the same kernels; no kernel
waits on another rank (the ranks meet only at host barriers, gloo).  The fused grid must be
bit-identical to one engine's union over all humans (max is exact and order-independent),
in both RNG modes, for two consecutive cycles on alternating buffers.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

HUMANS = 4


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _engine(sc, mode, ids, peer=None):
    from paper_2603_01122_b200.engine import CycleEngine, EngineConfig
    cfg = EngineConfig(n=8192, steps=24, dt=sc.dt, smoothing_sigma=0.1, seed=5, mode=mode)
    eng = CycleEngine(sc.control_set, sc.q, [sc.spaces[i] for i in ids], sc.spec, cfg,
                      human_ids=ids, peer=peer)
    eng.prime(sc.warmup_track[0][ids])
    return eng


def _worker(rank, world, port, mode, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_01122_b200.peer import PeerUnion
        from paper_2603_01122_b200.scenario import make_scene
        sc = make_scene("cfg2", cycles=4, humans=HUMANS)
        ids = list(range(rank * HUMANS // world, (rank + 1) * HUMANS // world))
        peer = PeerUnion((24, sc.spec.height, sc.spec.width), torch.float32)
        eng = _engine(sc, mode, ids, peer)
        fused = []
        for k in range(1, 3):
            b = k % 2
            peer.zero(b)
            peer.barrier()
            eng.stage(sc.warmup_track[k][ids], buf=b)
            eng.run_cycle(buf=b)
            peer.barrier()
            if peer.is_owner:
                fused.append(peer.tensor(b).cpu().numpy().copy())
        if rank == 0:
            ref = _engine(sc, mode, list(range(HUMANS)))
            want = []
            for k in range(1, 3):
                ref.stage(sc.warmup_track[k], buf=k % 2)
                want.append(ref.run_cycle(buf=k % 2).cpu().numpy().copy())
            np.savez(out_path, fused=np.stack(fused), want=np.stack(want))
        peer.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["production", "reference"])
def test_peer_union_equals_single_process_union(tmp_path, mode):
    out = str(tmp_path / "r.npz")
    mp.start_processes(_worker, args=(2, _free_port(), mode, out), nprocs=2, join=True, start_method="spawn")
    r = np.load(out)
    assert r["want"].max() > 0
    assert np.array_equal(r["fused"], r["want"])
