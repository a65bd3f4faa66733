"""Device plumbing: the CUDA device/stream every entry point runs on.

PyTorch supplies device memory and streams; the compute is the library's own kernels.
There is deliberately no CPU path: without a CUDA device the product raises.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib


class NoCudaDevice(RuntimeError):
    """A CUDA device (B200) is required; the predictor has no CPU fallback."""


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise NoCudaDevice("gridcast_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    _lib.lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream=None) -> ctypes.c_void_p:
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def upload(a, dev, dtype=None):
    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    return torch.from_numpy(arr).to(dev, non_blocking=False)


_TORCH_DT = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
             np.dtype(np.int32): torch.int32, np.dtype(np.uint32): torch.int32, np.dtype(np.uint64): torch.int64}


def upload_packed(dev, arrays):
    """Copy several small host arrays to the device in one transfer; returns device views
    (16-byte aligned, same shapes; unsigned types are viewed as their signed twins, which
    the C ABI reads as the unsigned bits)."""
    arrays = [np.ascontiguousarray(a) for a in arrays]
    offs, total = [], 0
    for a in arrays:
        total = (total + 15) // 16 * 16
        offs.append(total)
        total += a.nbytes
    host = np.zeros((total + 15) // 16 * 16 or 16, dtype=np.uint8)
    for a, o in zip(arrays, offs):
        host[o:o + a.nbytes] = a.reshape(-1).view(np.uint8)
    d = torch.as_tensor(host, device=dev)
    return [d[o:o + a.nbytes].view(_TORCH_DT[a.dtype]).view(a.shape) for a, o in zip(arrays, offs)]
