// Check: the error of the reference-mode filter weight w~(x) = ex2.approx.ftz(fl(x * log2e))
// (gc_predict.cu ref_pick's fast pass) against the true e^x, over EVERY float32 x in
// [-104, 0] (~1.1e9 inputs, exhaustive).  The filter's margin (GC_REF_FILTER_* in
// gc_predict.cu) assumes
//     |w~(x) - e^x| <= EPS_W * e^x + A_W        for every such x
// and this tool prints the measured worst cases the constants must dominate:
//   * max relative error over x with e^x >= 2^-125 (normal results), per |x| decade bin,
//   * max of |w~ - e^x| - EPS_W e^x over all x (the additive part; FTZ and the argument
//     rounding |x| 2^-24 e^x live here),
// and exits 1 when the stated (EPS_W, A_W) are violated anywhere.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false
//        -I paper_2603_01122_b200/csrc tools/cuda_checks/ex2_filter_err.cu -o /tmp/ex && /tmp/ex
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "gc_common.cuh"
using namespace gc;

#ifndef EPS_W
#define EPS_W 3.0e-7  // EPS_MUFU: gc_predict.cu GC_REF_FILTER_EPS_W = EPS_MUFU + numpy (2.13e-7) + slack
#endif
#ifndef A_W
#define A_W 1.0e-9
#endif

__device__ __forceinline__ void amax(unsigned *p, double v) {
    // positive floats order as their bit patterns
    atomicMax(p, __float_as_uint((float)v));
}

__global__ void kall(unsigned lo, unsigned long long count, unsigned *relbin, unsigned *addmax,
                     unsigned long long *viol) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const float x = __uint_as_float(lo + (unsigned)i);  // negative floats: lo = 0x80000000
        const float t = __fmul_rn(x, 1.4426950408889634f);
        const double w = (double)ex2_approx(t);
        const double e = exp((double)x);
        const double err = fabs(w - e);
        if (e >= 0x1p-125) {
            const int b = min(104, (int)(-x));
            amax(&relbin[b], err / e);
        }
        const double add = err - EPS_W * e;
        if (add > 0) amax(addmax, add);
        if (err > EPS_W * e + A_W) atomicAdd(viol, 1ull);
    }
}

int main() {
    const unsigned lo = 0x80000000u, hi = 0xC2D00000u;  // -0 .. -104
    const unsigned long long count = (unsigned long long)(hi - lo) + 1;
    unsigned *d_rel, *d_add;
    unsigned long long *d_v;
    cudaMalloc(&d_rel, 105 * 4);
    cudaMalloc(&d_add, 4);
    cudaMalloc(&d_v, 8);
    cudaMemset(d_rel, 0, 105 * 4);
    cudaMemset(d_add, 0, 4);
    cudaMemset(d_v, 0, 8);
    kall<<<148 * 16, 256>>>(lo, count, d_rel, d_add, d_v);
    unsigned rel[105], add;
    unsigned long long v;
    cudaMemcpy(rel, d_rel, sizeof(rel), cudaMemcpyDeviceToHost);
    cudaMemcpy(&add, d_add, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&v, d_v, 8, cudaMemcpyDeviceToHost);
    if (cudaGetLastError() != cudaSuccess) { printf("cuda error\n"); return 2; }
    float worst = 0.f;
    for (int b = 0; b <= 104; ++b) {
        float r;
        memcpy(&r, &rel[b], 4);
        worst = r > worst ? r : worst;
        if (b < 4 || b % 10 == 0 || b >= 85) printf("|x| in [%3d,%3d): max rel err %.3e\n", b, b + 1, r);
    }
    float a;
    memcpy(&a, &add, 4);
    printf("inputs %llu; max rel err (normal) %.4e; max additive excess over EPS_W=%.2e: %.4e (A_W=%.2e); violations %llu\n",
           count, worst, (double)EPS_W, a, (double)A_W, v);
    return v ? 1 : 0;
}
