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
    # chunks start on 4-step boundaries (the K < 4 production path takes turns over up to
    # 4 steps; the engine keeps this phase for every launch shape)
    assert all((t0 - 1) % 4 == 0 for t0, _ in b)
    assert len(b) <= max(1, chunks)


class _Geo:
    def __init__(self, steps, budget_kb, cells=400, res=0.1, dt=0.02, reduce=None):
        from paper_2603_01122_b200.occupancy import GridSpec
        from paper_2603_01122_b200.tables import Geometry
        self.cfg = EngineConfig(steps=steps, window_budget_kb=budget_kb, hist_path="smem")
        self.geo = Geometry(GridSpec(cells, cells, res), steps, 1.4 * dt, 0.1, "cpu")
        self.counts_reduce = reduce


@pytest.mark.parametrize("steps", [1, 4, 100, 248, 250, 500, 1000])
@pytest.mark.parametrize("budget", [0.0, 46.0, 64.0])
def test_window_bounds_split_long_horizons_on_4_step_boundaries(steps, budget):
    e = _Geo(steps, budget)
    b = CycleEngine.window_bounds(e)
    assert b[0][0] == 1 and b[-1][1] == steps + 1 and len(b) <= 2
    if len(b) == 2:
        t = b[0][1]
        assert (t - 1) % 4 == 0 and budget > 0
        cells = e.geo.win_cells

        def kb(c):
            return (((int(c) + 1) // 2 + 3) // 4 * 16) / 1024
        assert kb(cells[t - 2]) <= budget < kb(cells[steps - 1])   # the prefix fits, the whole does not
    if budget == 0.0 or steps <= 264:
        assert b == [(1, steps + 1)]
    # particle sharding keeps one launch (its counts are reduced across GPUs before K3)
    assert CycleEngine.window_bounds(_Geo(steps, budget, reduce=lambda c: c)) == [(1, steps + 1)]


def test_tapered_chunks_shrink_toward_the_end():
    sizes = [t1 - t0 for t0, t1 in CycleEngine.chunk_bounds(_Cfg(250, 0.5), 6)]
    assert sizes == sorted(sizes, reverse=True) and sizes[-1] <= 8 and sum(sizes) == 250


def test_bench_reference_arm_json_contract():
    """`bench.py --impl reference` (the driver's reference arm) prints one JSON line with the
    contract's keys; tiny sample (1 step of one human) so it runs in seconds on CPU."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3", "--ref-t", "1"], capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["warmup"] >= 3
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
