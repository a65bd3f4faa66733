// gc_abi.cu -- error state, version, launch counter and host-side RNG utilities.
#include <cstring>
#include <string>
#include "gc_common.cuh"
#include "gc_internal.h"

namespace gc {
static thread_local std::string g_err;
static std::atomic<uint64_t> g_launches{0};

void set_error(const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}
void count_launch(uint64_t k) { g_launches += k; }
}  // namespace gc

extern "C" {

const char *gc_last_error(void) { return gc::g_err.c_str(); }
int32_t gc_abi_version(void) { return GC_ABI_VERSION; }
uint64_t gc_launch_count(void) { return gc::g_launches.load(); }

// stream-ordered zero fill of a device buffer (graph-capturable memset node)
gc_status gc_fill_zero(void *d_ptr, int64_t bytes, void *stream) {
    GC_CHECK_ARG(d_ptr != nullptr && bytes >= 0, "gc_fill_zero: bad buffer");
    if (bytes == 0) return GC_OK;
    return gc::cuda_check(cudaMemsetAsync(d_ptr, 0, (size_t)bytes, (cudaStream_t)stream), "gc_fill_zero");
}

// rng.derive_seed (rng.py:34-39)
uint64_t gc_derive_seed(uint64_t seed, const uint32_t *h_path, int32_t path_len) {
    gc::SSPool s = gc::ss_pool_init(seed);
    for (int i = 0; i < path_len; ++i) gc::ss_absorb(s, h_path[i]);
    uint64_t k0, k1;
    gc::ss_key(s, k0, k1);
    return k0 ^ k1;
}

// rng.stream(seed, *path).random(n, dtype=float32) (rng.py:27-31)
void gc_stream_f32(uint64_t seed, const uint32_t *h_path, int32_t path_len, float *h_out, int64_t n) {
    gc::SSPool s = gc::ss_pool_init(seed);
    for (int i = 0; i < path_len; ++i) gc::ss_absorb(s, h_path[i]);
    uint64_t k0, k1;
    gc::ss_key(s, k0, k1);
    for (int64_t j = 0; j < n; ++j) h_out[j] = gc::philox64_f32(k0, k1, (uint64_t)j);
}

}  // extern "C"
