"""Device plumbing: the CUDA device/stream every entry point runs on.

PyTorch supplies device memory and streams; the compute is the library's own kernels.
There is deliberately no CPU path: without a CUDA device the product raises.
"""

from __future__ import annotations

import ctypes

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
    import numpy as np
    arr = np.ascontiguousarray(a if dtype is None else np.asarray(a, dtype=dtype))
    return torch.from_numpy(arr).to(dev, non_blocking=False)
