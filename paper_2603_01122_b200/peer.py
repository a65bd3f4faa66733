"""Fused multi-GPU union over NVLink peer memory (the union of sim.py:500-502 /
occupancy.py:162-192 across the ranks of one node).

``engine.fused_reduce`` merges per-rank (T, H, W) unions with an NCCL max-reduce of the
dense grids every cycle (cfg3 shape: 160 MB float32).  ``PeerUnion`` instead lets every
rank's epilogue (K3, ``gc_grid_epilogue``) atomicMax its humans' smoothed layers straight
into the owning rank's grid through a CUDA IPC mapping: the transfer is the sparse K3 write
stream itself (only tiles with particles), overlapped tile by tile with the smoothing, and
no reduction kernel runs at all.  The max of non-negative IEEE values is exact and
order-independent, so the fused grid is bit-identical to the single-GPU union.

Protocol per cycle on buffer b (``buffers`` = 2 lets cycle k+1 compute while the owner
reads cycle k):

    owner: zero(b) ──► barrier ──► every rank: cycle with ``CycleEngine(peer=...)`` writing b
                                   ──► barrier ──► owner reads / time-unions b

``barrier`` is stream-ordered: a 4-byte NCCL all-reduce on the current stream (CUDA-graph
capturable) when the process group is NCCL, else a host barrier after a device sync (gloo;
used by the single-GPU, two-process test).
"""

from __future__ import annotations

import ctypes
import math
from typing import Optional, Sequence

import torch

from . import _lib

_TYPESTR = {torch.float32: "<f4", torch.float64: "<f8"}


class _CudaArray:
    """Zero-copy ``__cuda_array_interface__`` view of a raw device allocation."""

    def __init__(self, ptr: int, shape, dtype: torch.dtype):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": _TYPESTR[dtype],
                                         "data": (int(ptr), False), "version": 3, "strides": None}


class PeerUnion:
    """(T, H, W) union grids owned by rank ``owner`` of ``group`` and mapped into every rank.

    ``ptr(b)`` is the device address this rank passes as the epilogue's union pointer;
    ``tensor(b)`` (owner only) is a torch view of buffer b for reading / copying it out."""

    def __init__(self, shape: Sequence[int], dtype: torch.dtype = torch.float32, group=None,
                 owner: int = 0, buffers: int = 2):
        import torch.distributed as dist
        if dtype not in _TYPESTR:
            raise ValueError("PeerUnion holds float32 or float64 grids")
        self.shape, self.dtype, self.group, self.owner = tuple(shape), dtype, group, owner
        self.rank = dist.get_rank(group)
        self.is_owner = self.rank == owner
        self.nbytes = math.prod(self.shape) * torch.tensor([], dtype=dtype).element_size()
        self._nccl = dist.get_backend(group) == "nccl"
        self._flag = torch.zeros(1, dtype=torch.int32, device="cuda") if self._nccl else None
        L = _lib.lib()
        self._ptrs, self._owned, self._tensors = [], [], []
        handles = None
        if self.is_owner:
            for _ in range(buffers):
                p = ctypes.c_void_p()
                _lib.check(L.gc_peer_alloc(self.nbytes, ctypes.byref(p)), "gc_peer_alloc")
                self._owned.append(p.value)
                self._ptrs.append(p.value)
                t = torch.as_tensor(_CudaArray(p.value, self.shape, dtype), device="cuda")
                t.zero_()
                self._tensors.append(t)
            handles = []
            for p in self._ptrs:
                h = (ctypes.c_uint8 * 64)()
                _lib.check(L.gc_peer_export(ctypes.c_void_p(p), h), "gc_peer_export")
                handles.append(bytes(h))
            torch.cuda.synchronize()
        obj = [handles]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, owner) if group is not None else owner,
                                   group=group)
        if not self.is_owner:
            for hb in obj[0]:
                p = ctypes.c_void_p()
                h = (ctypes.c_uint8 * 64).from_buffer_copy(hb)
                _lib.check(L.gc_peer_import(h, ctypes.byref(p)), "gc_peer_import")
                self._ptrs.append(p.value)
        self.buffers = buffers

    def ptr(self, b: int) -> int:
        return self._ptrs[b % self.buffers]

    def tensor(self, b: int) -> torch.Tensor:
        if not self.is_owner:
            raise RuntimeError("only the owning rank holds the fused union as a tensor")
        return self._tensors[b % self.buffers]

    def zero(self, b: int):
        """Owner: clear buffer b on the current stream (before the barrier that opens a cycle)."""
        if self.is_owner:
            self._tensors[b % self.buffers].zero_()

    def barrier(self):
        """Every rank: all writes issued before it (any rank) precede all work issued after it."""
        import torch.distributed as dist
        if self._nccl:
            dist.all_reduce(self._flag, group=self.group)
        else:
            torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.group)

    def finish(self, b: int, time_union: bool = False):
        """Owner, after the closing barrier: the conservative time union (sim.py:503-504)."""
        if self.is_owner and time_union:
            t = self._tensors[b % self.buffers]
            hw = t.shape[-1] * t.shape[-2]
            sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            _lib.check(_lib.lib().gc_time_union(ctypes.c_void_p(t.data_ptr()), t.element_size(), 0, t.shape[0],
                                                hw, sh), "gc_time_union")

    def close(self):
        """Collective: importers unmap first, then the owner frees."""
        import torch.distributed as dist
        L = _lib.lib()
        torch.cuda.synchronize()
        if not self.is_owner:
            for p in self._ptrs:
                _lib.check(L.gc_peer_close(ctypes.c_void_p(p)), "gc_peer_close")
        dist.barrier(group=self.group)
        if self.is_owner:
            self._tensors = []
            for p in self._owned:
                _lib.check(L.gc_peer_free(ctypes.c_void_p(p)), "gc_peer_free")
        self._ptrs, self._owned = [], []
