"""CPU: bench.py's reference arm (the timed CPU path, oracle/port.py) and the contract the
driver compares the two arms on: identical workload config dicts, an explicit
extrapolation, the host description BASELINE.md 5 asks for."""

import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _args(**kw):
    a = argparse.Namespace(config="cfg1", goal_radius=None, gpus=1)
    for k, v in kw.items():
        setattr(a, k, v)
    return a


def test_reference_arm_line_and_identical_config():
    import bench
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "cfg1", "--steps", "2",
                          "--warmup", "3", "--ref-t", "2"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "particle-steps/s"
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "port" and cb["cores"] >= 1 and cb["value"] == d["value"]
    for k in ("cpu_model", "nproc", "numpy", "OPENBLAS_NUM_THREADS"):
        assert k in cb["host"], k
    assert d["extrapolated"] and d["extrapolation"]["sampled_steps"] == 2
    assert d["extrapolation"]["factor_steps"] == 20 / 2
    # our arm builds its config with the same function from the same arguments
    scene = bench.scene_for(_args(), 0, cycles=2)
    assert d["config"] == json.loads(json.dumps(bench.workload_config(_args(), scene, 1)))


def test_reference_arm_other_ranks_exit_without_work():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0 and not out.stdout.strip()


def test_worker_choices_follow_baseline_protocol():
    import bench
    ch = bench.worker_choices()
    assert ch[0] is None and (os.cpu_count() or 1) in ch or os.cpu_count() == 1
    assert all(w is None or w >= 2 for w in ch)
