"""ORACLE (test infrastructure only): ctypes binding of ``oracle/c/oracle.c``."""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

Q_GOAL_PROGRESS = 0
Q_GOAL_PROGRESS_FULL = 1
Q_DEFAULT = 2


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "c", "oracle.c")
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        L.or_exp_np_f32.argtypes = [P, P, ctypes.c_long]
        L.or_exp_np_f32.restype = None
        L.or_propagate.argtypes = [P, P, P, ctypes.c_long, P, P, P, P, P, P, ctypes.c_int,
                                   P, P, P, ctypes.c_int, P, P, P]
        L.or_propagate.restype = None
        L.or_cells.argtypes = [P, ctypes.c_long, ctypes.c_float, ctypes.c_float,
                               ctypes.c_float, ctypes.c_int, ctypes.c_int, P]
        L.or_cells.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def exp_np_f32(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.empty_like(x)
    lib().or_exp_np_f32(_p(x), _p(y), x.size)
    return y


def propagate(xy, hyp, beta32, goal32, tables, u01, return_picked=False):
    """One reference step (prediction.py:147-162) for all particles, exact float32."""
    xy = np.ascontiguousarray(xy, dtype=np.float32)
    hyp = np.ascontiguousarray(hyp, dtype=np.int32)
    beta32 = np.ascontiguousarray(beta32, dtype=np.float32)
    goal32 = np.ascontiguousarray(goal32, dtype=np.float32)
    u01 = np.ascontiguousarray(u01, dtype=np.float32)
    out = np.empty_like(xy)
    keep = np.ascontiguousarray(tables.keep, dtype=np.int32)
    work = np.empty(len(keep), dtype=np.float32)
    picked = np.empty(len(hyp), dtype=np.int32) if return_picked else None
    lib().or_propagate(
        _p(xy), _p(out), _p(hyp), len(hyp), _p(beta32), _p(goal32),
        _p(tables.sx), _p(tables.sy), _p(tables.at), _p(tables.pen), int(tables.q_kind),
        _p(tables.dispx), _p(tables.dispy), _p(keep), len(keep), _p(u01), _p(work),
        _p(picked) if picked is not None else None,
    )
    return (out, picked) if return_picked else out


def cells(xy, grid) -> np.ndarray:
    """Flat clamped cell index iy*W+ix of every particle (occupancy.py:43-51)."""
    xy = np.ascontiguousarray(xy, dtype=np.float32)
    flat = np.empty(xy.shape[0], dtype=np.int64)
    lib().or_cells(_p(xy), xy.shape[0], np.float32(grid.origin[0]), np.float32(grid.origin[1]),
                   np.float32(grid.resolution), int(grid.width), int(grid.height), _p(flat))
    return flat
