"""GPU: the device restatements of numpy's float32 exp.

* exp_np2 (packed FP32x2, used by the bit-exact reference mode) equals the scalar exp_np
  lane by lane on every float in [-110, 0] (tools/cuda_checks/exp2_vs_exp.cu);
* exp_np and exp_np2 equal numpy's own np.exp(float32) -- this box's numpy -- bit for bit
  on EVERY float32 input of the propagation's domain [-110, 0] and on a sweep of positive
  inputs up to overflow.  (The oracle's restatement is pinned to numpy on a fixture in
  tests/test_oracle_golden.py; this is the exhaustive device-side pin.)
"""

import ctypes
import os
import subprocess

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
         "--fmad=false", "-I", os.path.join(ROOT, "paper_2603_01122_b200", "csrc")]


def test_exp_np2_bit_identical_to_exp_np(tmp_path):
    exe = str(tmp_path / "exp2_vs_exp")
    subprocess.run(["nvcc", *FLAGS, os.path.join(ROOT, "tools", "cuda_checks", "exp2_vs_exp.cu"), "-o", exe],
                   check=True, capture_output=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches: 0 of" in out.stdout


def test_device_exp_equals_numpy_on_every_float(tmp_path):
    so = str(tmp_path / "libexp.so")
    subprocess.run(["nvcc", *FLAGS, "-shared", "-Xcompiler", "-fPIC",
                    os.path.join(ROOT, "tools", "cuda_checks", "exp_lib.cu"), "-o", so], check=True, capture_output=True)
    lib = ctypes.CDLL(so)
    lib.exp_np_batch.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_longlong, ctypes.c_void_p]

    def check(bits):
        x = bits.view(np.float32)
        with np.errstate(over="ignore", under="ignore"):
            ref = np.exp(x)
        dx = torch.from_numpy(x).cuda()
        dy, dy2 = torch.empty_like(dx), torch.empty_like(dx)
        assert lib.exp_np_batch(dx.data_ptr(), dy.data_ptr(), dy2.data_ptr(), len(x),
                                torch.cuda.current_stream().cuda_stream) == 0
        for d in (dy, dy2):
            got = d.cpu().numpy()
            bad = np.flatnonzero(got.view(np.uint32) != ref.view(np.uint32))
            assert len(bad) == 0, (x[bad[:4]], got[bad[:4]], ref[bad[:4]])

    # every float in [-110, 0]: bit patterns 0x80000000 .. 0xC2DC0000, in 64 M slabs
    lo, hi, step = 0x80000000, 0xC2DC0000, 1 << 26
    for s in range(lo, hi, step):
        check(np.arange(s, min(s + step, hi), dtype=np.uint32))
    # positive inputs up to past the overflow threshold (88.72), strided
    check(np.linspace(0, 0x42C00000, 1 << 24).astype(np.uint32))
