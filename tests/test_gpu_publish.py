"""GPU: tile-sparse D2H of the fused union (gc_publish_tiles).

The e2e cycle ships only the 32 x 32 union tiles that are nonzero now, or that the host
stack still holds from its previous cycle (zeroed), by kernel stores into the pinned host
stack.  After every cycle the host stack must equal the device union bit for bit --
whatever the tiles did in between (humans move, tiles appear and vanish, buffers alternate).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2603_01122_b200.engine import CycleEngine, EngineConfig  # noqa: E402
from paper_2603_01122_b200.scenario import make_scene  # noqa: E402


@pytest.mark.parametrize("dtype,chunks,time_union,mode", [
    ("float64", 1, False, "production"), ("float64", 3, False, "production"), ("float32", 3, True, "production"),
    ("float64", 2, True, "reference")])
def test_host_stack_equals_device_union_every_cycle(dtype, chunks, time_union, mode):
    sc = make_scene("cfg2", cycles=8, humans=3)
    cfg = EngineConfig(n=8192, steps=40, dt=sc.dt, mode=mode, union_dtype=dtype, time_union=time_union,
                       chunk_taper=0.6)
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, cfg)
    eng.prime(sc.warmup_track[0])
    tdt = torch.float64 if dtype == "float64" else torch.float32
    host = [torch.zeros(eng.unions[0].shape, dtype=tdt).pin_memory() for _ in range(2)]
    host[1].fill_(7.0)  # a dirty host stack is zeroed on its first use
    cp = torch.cuda.Stream()
    track = np.concatenate([sc.warmup_track[1:], sc.track])
    # large jumps between some cycles: whole tiles vanish and appear elsewhere
    track[4] += 3.0
    for k in range(len(track)):
        b = k % 2
        eng.stage(track[k], buf=b)
        eng.run_cycle(buf=b, chunks=chunks, d2h=host[b], copy_stream=cp)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(host[b].numpy(), eng.unions[b].cpu().numpy())
    assert host[0].numpy().max() > 0
    eng.check_errors()


def test_graph_replay_with_tile_publication():
    """The captured e2e cycle (H2D, update, chunked predict, tile publication on the copy
    stream) leaves the host stack equal to the device union on every replay."""
    sc = make_scene("cfg2", cycles=6, humans=2)
    cfg = EngineConfig(n=4096, steps=32, dt=sc.dt, union_dtype="float64")
    eng = CycleEngine(sc.control_set, sc.q, sc.spaces, sc.spec, cfg)
    eng.prime(sc.warmup_track[0])
    host = [torch.zeros(eng.unions[0].shape, dtype=torch.float64).pin_memory() for _ in range(2)]
    for k in range(1, 3):
        eng.stage(sc.warmup_track[k], buf=k % 2)
        eng.run_cycle(buf=k % 2)
    torch.cuda.synchronize()
    g = [eng.capture(buf=b, with_h2d=True, chunks=3, d2h=host[b]) for b in (0, 1)]
    for k in range(3, 9):
        b = k % 2
        eng.stage(sc.warmup_track[k] if k <= 10 else sc.track[k - 11], buf=b)
        g[b].replay()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(host[b].numpy(), eng.unions[b].cpu().numpy())

