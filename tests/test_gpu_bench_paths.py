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
               "--cpu-runs", "1", "--no-ref-mode"])
    _check(d)
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("port", "reference")
    assert cb["host"]["nproc"] >= 1 and "numpy" in cb["host"] and cb["extrapolation"]["sampled_steps"] == 1
    assert d["p99_ms"] >= d["p50_ms"] > 0 and d["latency_cycles"] >= 20
    # the headline e2e is the reference's float64 layout, the float32 one beside it
    assert d["e2e"]["dtype"] == "f64" and d["e2e_f32"]["dtype"] == "f32"
    assert d["e2e"]["d2h_bytes_per_step"] == 2 * d["e2e_f32"]["d2h_bytes_per_step"]
    # K2 timed inside the replayed graph: a share of the cycle, never more than it
    assert 0 < d["kernels_ms"]["k_predict"] < d["ms_per_step"]


def test_bench_gpus_beyond_the_box_fails_loudly():
    import torch
    n = torch.cuda.device_count() + 1
    out = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--steps", "3"], capture_output=True,
                         text=True, timeout=300, cwd=ROOT)
    assert out.returncode != 0 and "CUDA device" in out.stderr
    assert not [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]


def test_bench_distributed_path_one_rank():
    d = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
               "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--gpus", "1", "--force-dist",
               "--steps", "5", "--warmup", "3", "--lat-cycles", "10", "--no-cpu-baseline", "--no-ref-mode",
               "--no-e2e-alt"])
    _check(d)
    assert d["fused_grid"] == "nccl" and d["n_gpus"] == 1


def test_bench_distributed_path_one_rank_peer_union():
    d = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
               "--master-addr", "127.0.0.1", "--master-port", "29543", "bench.py", "--gpus", "1", "--force-dist",
               "--fused-path", "peer", "--steps", "5", "--warmup", "3", "--lat-cycles", "10", "--no-cpu-baseline",
               "--no-ref-mode", "--no-e2e-alt"])
    _check(d)
    assert d["fused_grid"] == "peer" and d["n_gpus"] == 1


def test_bench_distributed_path_one_rank_dense_reduce():
    d = _line([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
               "--master-addr", "127.0.0.1", "--master-port", "29545", "bench.py", "--gpus", "1", "--force-dist",
               "--fused-path", "nccl-dense", "--steps", "5", "--warmup", "3", "--lat-cycles", "10",
               "--no-cpu-baseline", "--no-ref-mode", "--no-e2e-alt"])
    _check(d)
    assert d["fused_grid"] == "nccl-dense" and d["n_gpus"] == 1
