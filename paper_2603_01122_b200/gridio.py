"""Layered-grid stack files (reference gridio.py:1-72, "GCST" format).

    magic b"GCST" | version u32 = 1 | width, height, steps u32 |
    resolution, origin_x, origin_y, dt, base_time f64 | steps*height*width f64 row-major

``save_stack`` streams a device-resident stack (float32 union or float64 layers) to disk
in layer chunks: each chunk is widened to float64 on the GPU and copied to pinned host
memory while the previous chunk is written, so a 250-layer 400x400 stack never needs a
full host copy.  ``load_stack`` returns a host-backed PredictionStack (reference layout).
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from .occupancy import GridSpec
from .prediction import PredictionStack

MAGIC = b"GCST"
VERSION = 1
HEADER = struct.Struct("<4sIIII5d")


def _header(spec, steps, dt, base_time) -> bytes:
    return HEADER.pack(MAGIC, VERSION, spec.width, spec.height, steps, spec.resolution,
                       spec.origin[0], spec.origin[1], dt, base_time)


def save_stack(stack: PredictionStack, path, chunk_layers: int = 16) -> None:
    src = stack._dev if getattr(stack, "_dev", None) is not None else None
    with open(path, "wb") as f:
        f.write(_header(stack.spec, stack.steps, stack.dt, stack.base_time))
        if src is None:
            f.write(np.ascontiguousarray(stack.layers, dtype="<f8").tobytes())
            return
        T = src.shape[0]
        hw = src.shape[1] * src.shape[2]
        bufs = [torch.empty((chunk_layers, hw), dtype=torch.float64).pin_memory() for _ in range(2)]
        copy = torch.cuda.Stream()
        done = [None, None]
        pending = None
        for i, k0 in enumerate(range(0, T, chunk_layers)):
            k1 = min(T, k0 + chunk_layers)
            b = i % 2
            if done[b] is not None:
                done[b].synchronize()
            with torch.cuda.stream(copy):
                copy.wait_stream(torch.cuda.current_stream())
                wide = src[k0:k1].reshape(k1 - k0, hw).to(torch.float64)
                bufs[b][: k1 - k0].copy_(wide, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            if pending is not None:
                pb, pn, pev = pending
                pev.synchronize()
                f.write(bufs[pb][:pn].numpy().astype("<f8", copy=False).tobytes())
            pending = (b, k1 - k0, ev)
            done[b] = ev
        if pending is not None:
            pb, pn, pev = pending
            pev.synchronize()
            f.write(bufs[pb][:pn].numpy().astype("<f8", copy=False).tobytes())


def load_stack(path) -> PredictionStack:
    with open(path, "rb") as f:
        raw = f.read(HEADER.size)
        if len(raw) != HEADER.size:
            raise ValueError(f"{path}: truncated layered-grid header")
        magic, version, width, height, steps, res, ox, oy, dt, base_time = HEADER.unpack(raw)
        if magic != MAGIC:
            raise ValueError(f"{path}: not a layered-grid file (bad magic {magic!r})")
        if version != VERSION:
            raise ValueError(f"{path}: unsupported layered-grid version {version}")
        count = steps * height * width
        data = np.frombuffer(f.read(count * 8), dtype="<f8")
        if data.size != count:
            raise ValueError(f"{path}: truncated layer data")
    spec = GridSpec(width=width, height=height, resolution=res, origin=(ox, oy))
    return PredictionStack(spec, data.reshape(steps, height, width), base_time, dt)


def grid_to_csv(grid, path) -> None:
    """One grid as comma-separated rows, row 0 = lowest y, 17 significant digits
    (gridio.py:75-77) -- a round trip reproduces every float64 exactly."""
    np.savetxt(path, np.asarray(grid.values, dtype=float), delimiter=",", fmt="%.17g")


def grid_from_csv(path, spec: GridSpec):
    """Inverse of grid_to_csv (gridio.py:80-82)."""
    from .occupancy import OccupancyGrid
    return OccupancyGrid(spec, np.loadtxt(path, delimiter=",", ndmin=2))
