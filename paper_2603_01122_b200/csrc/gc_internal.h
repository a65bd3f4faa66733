// gc_internal.h -- host-side helpers shared by the gridcast_b200 translation units.
#pragma once
#include <cstdarg>
#include <cstdio>
#include <cstdint>
#include <atomic>
#include <cuda_runtime.h>
#include "../../include/gridcast_b200.h"

namespace gc {

void set_error(const char *fmt, ...);
void count_launch(uint64_t k = 1);

inline gc_status cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return GC_CUDA_ERROR;
    }
    return GC_OK;
}

#define GC_TRY(expr)                           \
    do {                                       \
        gc_status _s = (expr);                 \
        if (_s != GC_OK) return _s;            \
    } while (0)

#define GC_CUDA(call) GC_TRY(::gc::cuda_check((call), #call))

#define GC_CHECK_ARG(cond, ...)                \
    do {                                       \
        if (!(cond)) {                         \
            ::gc::set_error(__VA_ARGS__);      \
            return GC_BAD_ARG;                 \
        }                                      \
    } while (0)

}  // namespace gc
