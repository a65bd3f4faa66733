"""GPU: the packed FP32x2 numpy-exp (exp_np2, used by the bit-exact reference mode) equals
the scalar restatement exp_np lane by lane on 16.7 M floats in [-110, 0] (the oracle pins
exp_np to numpy; tests/test_oracle_golden.py::test_numpy_exp_restatement_bit_exact)."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exp_np2_bit_identical_to_exp_np(tmp_path):
    exe = str(tmp_path / "exp2_vs_exp")
    src = os.path.join(ROOT, "tools", "cuda_checks", "exp2_vs_exp.cu")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-ftz=false", "-prec-div=true",
                    "-prec-sqrt=true", "--fmad=false", "-I", os.path.join(ROOT, "paper_2603_01122_b200", "csrc"),
                    src, "-o", exe], check=True, capture_output=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches: 0 of" in out.stdout
