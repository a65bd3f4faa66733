"""Stream namespaces and key derivation (reference rng.py:1-47).

The draws themselves are generated inside the kernels (GC_RNG_REFERENCE regenerates the
reference's Philox4x64-10 streams in-register); this module keeps the namespace
constants and the host-side key helpers, implemented by the C ABI (gc_derive_seed,
gc_stream_f32) rather than numpy.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

HYPOTHESIS_DRAWS = 0
STEP_DRAWS = 1
HUMAN_PREFIX = 2
SIM_HUMAN = 3
SIM_OBSERVE = 4
MPPI_NOISE = 5
SIM_PREDICT = 7  # sim.py per-cycle prediction seed namespace

_MASK64 = (1 << 64) - 1


def _path(path):
    arr = (ctypes.c_uint32 * max(1, len(path)))(*[int(p) & 0xFFFFFFFF for p in path])
    return arr, len(path)


def derive_seed(seed: int, *path: int) -> int:
    """SeedSequence(seed, spawn_key=path).generate_state(2, u64) folded by xor."""
    arr, n = _path(path)
    return int(_lib.lib().gc_derive_seed(int(seed) & _MASK64, arr, n))


def stream(seed: int, *path: int) -> np.random.Generator:
    """The generator of stream (seed, *path) (rng.py:27-31): numpy's Philox4x64-10 keyed by
    SeedSequence(seed, spawn_key=path) -- the host-side object for callers that draw from
    a stream directly; the kernels regenerate the same streams in-register."""
    ss = np.random.SeedSequence(entropy=int(seed) & _MASK64, spawn_key=tuple(int(p) & 0xFFFFFFFF for p in path))
    return np.random.Generator(np.random.Philox(ss))


def stream_f32(seed: int, path, n: int) -> np.ndarray:
    """``rng.stream(seed, *path).random(n, dtype=float32)`` computed by the C ABI."""
    arr, k = _path(path)
    out = np.empty(n, dtype=np.float32)
    _lib.lib().gc_stream_f32(int(seed) & _MASK64, arr, k, out.ctypes.data_as(ctypes.c_void_p), n)
    return out


def chunk_ranges(n: int, chunk: int):
    index = 0
    for start in range(0, n, chunk):
        yield start, min(start + chunk, n), index
        index += 1
