"""GPU: bench.py's JSON contract on both of its code paths (short runs).

* the single-GPU path (device cycle, chunked e2e, roofline, clocks, CPU baseline);
* the multi-GPU path (NCCL process group, fused max-reduce, overlapped rank-0 D2H) through
  torchrun with one rank (--force-dist): the branch the driver's scaling run takes; and
  the same branch with the peer-memory fused grid (--fused-path peer).
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks")


def _line(cmd):
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _check(d):
    for k in KEYS:
        assert k in d, k
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["warmup"] >= 3 and "workload" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0 < r["frac"] < 1.5
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0


def test_bench_single_gpu_contract():
    d = _line([sys.executable, "bench.py", "--steps", "5", "--warmup", "3", "--lat-cycles", "20", "--cpu-t", "1",
               "--no-ref-mode"])
    _check(d)
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("port", "reference")
    assert d["p99_ms"] >= d["p50_ms"] > 0 and d["latency_cycles"] >= 20


def test_bench_distributed_path_one_rank():
    d = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
               "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--gpus", "1", "--force-dist",
               "--steps", "5", "--warmup", "3", "--lat-cycles", "10", "--no-cpu-baseline", "--no-ref-mode"])
    _check(d)
    assert d["config"]["fused_grid"] == "nccl"


def test_bench_distributed_path_one_rank_peer_union():
    d = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
               "--master-addr", "127.0.0.1", "--master-port", "29543", "bench.py", "--gpus", "1", "--force-dist",
               "--fused-path", "peer", "--steps", "5", "--warmup", "3", "--lat-cycles", "10", "--no-cpu-baseline",
               "--no-ref-mode"])
    _check(d)
    assert d["config"]["fused_grid"] == "peer"
