// Check: exp_np2 (packed FP32x2) is bit-identical to exp_np lane by lane over every float
// in [lo, hi] (strided), plus logits-shaped differences.  Build and run on the GPU box:
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

int main() {
    const int n = 1 << 24;
    float *h = new float[n];
    // all floats from -110 to 0 sampled evenly in the bit pattern space
    unsigned lo = 0x80000000u, hi = 0xC2DC0000u;  // -0.0 .. -110.0
    for (int i = 0; i < n; ++i) { unsigned b = lo + (unsigned)((double)(hi - lo) * i / n); memcpy(&h[i], &b, 4); }
    float *d, *ex; unsigned *bad;
    cudaMalloc(&d, n * 4); cudaMalloc(&bad, 4); cudaMalloc(&ex, 32 * 4);
    cudaMemcpy(d, h, n * 4, cudaMemcpyHostToDevice); cudaMemset(bad, 0, 4);
    k<<<(n / 2 + 255) / 256, 256>>>(d, n, bad, ex);
    unsigned nb; float e[32];
    cudaMemcpy(&nb, bad, 4, cudaMemcpyDeviceToHost); cudaMemcpy(e, ex, 128, cudaMemcpyDeviceToHost);
    printf("mismatches: %u of %d\n", nb, n);
    for (unsigned j = 0; j < nb && j < 8; ++j) {
        unsigned bx, by; memcpy(&bx, &e[4*j], 4); memcpy(&by, &e[4*j+3], 4);
        printf("  x=%.9g (%08x) exp_np=%.9g exp_np2=%.9g  other lane %.9g (%08x)\n", e[4*j], bx, e[4*j+1], e[4*j+2], e[4*j+3], by);
    }
    return nb != 0;
}
