"""CPU: host-side scheduling logic of the CycleEngine (no device work)."""

import pytest

from paper_2603_01122_b200.engine import CycleEngine, EngineConfig


class _Cfg:
    def __init__(self, steps, taper):
        self.cfg = EngineConfig(steps=steps, chunk_taper=taper)


@pytest.mark.parametrize("steps", [1, 2, 5, 22, 100, 250, 500])
@pytest.mark.parametrize("chunks", [1, 2, 3, 6, 8, 12, 200])
@pytest.mark.parametrize("taper", [0.4, 0.5, 1.0])
def test_chunk_bounds_partition_the_horizon_on_philox_phase(steps, chunks, taper):
    b = CycleEngine.chunk_bounds(_Cfg(steps, taper), chunks)
    assert b[0][0] == 1 and b[-1][1] == steps + 1
    assert all(t0 < t1 for t0, t1 in b)
    assert all(b[i][1] == b[i + 1][0] for i in range(len(b) - 1))
    # production streams draw one Philox block per 4 steps: every chunk starts on a block
    assert all((t0 - 1) % 4 == 0 for t0, _ in b)
    assert len(b) <= max(1, chunks)


def test_tapered_chunks_shrink_toward_the_end():
    sizes = [t1 - t0 for t0, t1 in CycleEngine.chunk_bounds(_Cfg(250, 0.5), 6)]
    assert sizes == sorted(sizes, reverse=True) and sizes[-1] <= 8 and sum(sizes) == 250
