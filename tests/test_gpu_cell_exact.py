"""GPU: K2's production cell map is the reference's floor(fl(fl(x - ox) / res)) exactly.

Production particles keep the reference's float32 world coordinates, and their cell is
computed from the correctly rounded reciprocal with one residual correction
(gc_common.cuh div_rn_recip) instead of the IEEE division's slow path.  This checks that
quotient bit for bit against __fdiv_rn on every float32 |t| <= 4096 res for a set of grid
resolutions (tools/cuda_checks/div_recip.cu)."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_div_rn_recip_equals_ieee_division_exhaustively(tmp_path):
    exe = str(tmp_path / "div_recip")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-ftz=false", "-prec-div=true",
                    "-I", os.path.join(ROOT, "paper_2603_01122_b200", "csrc"),
                    os.path.join(ROOT, "tools", "cuda_checks", "div_recip.cu"), "-o", exe], check=True,
                   capture_output=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("cell mismatches: 0 of") >= 12
