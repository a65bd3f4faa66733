// gc_peer.cu -- device buffers shared between the ranks of one node over CUDA IPC, so the
// epilogue (K3) of every rank can atomicMax its humans' layers straight into the fused
// union held by the owning rank (NVLink peer memory) instead of each rank writing a local
// union that an NCCL max-reduce then merges (engine.fused_reduce; sim.py:500-502 is the
// reference's single-process union).  The max is order-independent and exact, so the
// fused grid is bit-identical to the single-GPU one.
//
// An exported buffer is a whole cudaMalloc allocation (IPC handles name allocations, not
// interior pointers).  Opening uses cudaIpcMemLazyEnablePeerAccess, so a rank on another
// GPU maps it through NVLink; a second process on the same GPU maps it directly.
#include <cstring>
#include "gc_common.cuh"
#include "gc_internal.h"

using namespace gc;

extern "C" gc_status gc_peer_alloc(int64_t bytes, void **d_out) {
    GC_CHECK_ARG(d_out && bytes > 0, "gc_peer_alloc: need bytes > 0 and an output pointer");
    *d_out = nullptr;
    GC_CUDA(cudaMalloc(d_out, (size_t)bytes));
    return GC_OK;
}

extern "C" gc_status gc_peer_free(void *d) {
    if (d) GC_CUDA(cudaFree(d));
    return GC_OK;
}

extern "C" gc_status gc_peer_export(const void *d, uint8_t *h_handle) {
    GC_CHECK_ARG(d && h_handle, "gc_peer_export: null buffer or handle");
    static_assert(sizeof(cudaIpcMemHandle_t) == GC_PEER_HANDLE_BYTES, "IPC handle size");
    cudaIpcMemHandle_t h;
    GC_CUDA(cudaIpcGetMemHandle(&h, const_cast<void *>(d)));
    memcpy(h_handle, &h, sizeof(h));
    return GC_OK;
}

extern "C" gc_status gc_peer_import(const uint8_t *h_handle, void **d_out) {
    GC_CHECK_ARG(h_handle && d_out, "gc_peer_import: null handle or output pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, h_handle, sizeof(h));
    *d_out = nullptr;
    GC_CUDA(cudaIpcOpenMemHandle(d_out, h, cudaIpcMemLazyEnablePeerAccess));
    return GC_OK;
}

extern "C" gc_status gc_peer_close(void *d) {
    if (d) GC_CUDA(cudaIpcCloseMemHandle(d));
    return GC_OK;
}
