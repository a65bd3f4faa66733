// Check: exp_np2 (packed FP32x2, fast division, branch-free scaling) is bit-identical to
// exp_np lane by lane over EVERY float in [-110, 0] (exhaustive, ~1.1e9 inputs, plus a
// strided pairing so both lanes see different values).  Build and run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -ftz=false -prec-div=true --fmad=false
//        -I paper_2603_01122_b200/csrc tools/cuda_checks/exp2_vs_exp.cu -o /tmp/e2 && /tmp/e2
#include <cstdio>
#include <cstring>
#include "gc_common.cuh"
using namespace gc;

__global__ void k(const float *x, int n, unsigned *bad, float *ex) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i + 1 >= n) return;
    const float2 v = make_float2(x[2 * i], x[2 * i + 1]);
    const float2 y2 = exp_np2(v);
    const float a = exp_np(v.x), b = exp_np(v.y);
    if (__float_as_uint(a) != __float_as_uint(y2.x)) { unsigned j = atomicAdd(bad, 1u); if (j < 8) { ex[4*j] = v.x; ex[4*j+1] = a; ex[4*j+2] = y2.x; ex[4*j+3] = v.y; } }
    if (__float_as_uint(b) != __float_as_uint(y2.y)) { unsigned j = atomicAdd(bad, 1u); if (j < 8) { ex[4*j] = v.y; ex[4*j+1] = b; ex[4*j+2] = y2.y; ex[4*j+3] = v.x; } }
}

__global__ void kall(unsigned lo, unsigned count, unsigned *bad, float *ex) {
    // consecutive float bit patterns lo + 2i, lo + 2i + 1 as the two lanes
    const unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i + 1 >= count) return;
    const float2 v = make_float2(__uint_as_float(lo + (unsigned)(2 * i)), __uint_as_float(lo + (unsigned)(2 * i + 1)));
    const float2 y2 = exp_np2(v);
    const float a = exp_np(v.x), b = exp_np(v.y);
    if (__float_as_uint(a) != __float_as_uint(y2.x)) { unsigned j = atomicAdd(bad, 1u); if (j < 8) { ex[4*j] = v.x; ex[4*j+1] = a; ex[4*j+2] = y2.x; ex[4*j+3] = v.y; } }
    if (__float_as_uint(b) != __float_as_uint(y2.y)) { unsigned j = atomicAdd(bad, 1u); if (j < 8) { ex[4*j] = v.y; ex[4*j+1] = b; ex[4*j+2] = y2.y; ex[4*j+3] = v.x; } }
}

int main() {
    float *ex; unsigned *bad;
    cudaMalloc(&bad, 4); cudaMalloc(&ex, 32 * 4); cudaMemset(bad, 0, 4);
    // every float from -0.0 (0x80000000) to -110.0 (0xC2DC0000), in slabs
    const unsigned lo = 0x80000000u, hi = 0xC2DC0000u;
    unsigned long long total = 0;
    for (unsigned long long s = lo; s < hi; s += (1ull << 28)) {
        const unsigned cnt = (unsigned)((hi - s) < (1ull << 28) ? (hi - s) : (1ull << 28));
        kall<<<(unsigned)((cnt / 2 + 255) / 256), 256>>>((unsigned)s, cnt, bad, ex);
        total += cnt;
    }
    // and a strided pairing (different magnitudes in the two lanes)
    const int n = 1 << 24;
    float *h = new float[n];
    for (int i = 0; i < n; ++i) { unsigned b = lo + (unsigned)((double)(hi - lo) * i / n); memcpy(&h[i], &b, 4); }
    float *d;
    cudaMalloc(&d, n * 4);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice);
    k<<<(n / 2 + 255) / 256, 256>>>(d, n, bad, ex);
    unsigned nb; float e[32];
    cudaMemcpy(&nb, bad, 4, cudaMemcpyDeviceToHost); cudaMemcpy(e, ex, 128, cudaMemcpyDeviceToHost);
    printf("mismatches: %u of %llu\n", nb, total + n);
    for (unsigned j = 0; j < nb && j < 8; ++j) {
        unsigned bx, by; memcpy(&bx, &e[4*j], 4); memcpy(&by, &e[4*j+3], 4);
        printf("  x=%.9g (%08x) exp_np=%.9g exp_np2=%.9g  other lane %.9g (%08x)\n", e[4*j], bx, e[4*j+1], e[4*j+2], e[4*j+3], by);
    }
    return nb != 0;
}
