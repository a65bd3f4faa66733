// Check: K2's production cell map floor_clamp(div_rn_recip(t, res, recip_nr(res)), W - 1)
// (gc_common.cuh) equals the reference's clamp(floor(fl(t / res)), 0, W - 1) for EVERY
// float32 t with |t| <= 4096 res (W = 4096 cells), for each resolution given on the command
// line (default: a set of usual grid resolutions).  Also counts quotient bit mismatches
// where |t / res| >= 2^-100 (the correction step is exact there; below, residuals are
// subnormal but every such quotient is in cell 0 either way).  Prints
// "cell mismatches: N of M" per resolution; exit 1 on any cell mismatch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -ftz=false -prec-div=true
//        -I paper_2603_01122_b200/csrc tools/cuda_checks/div_recip.cu -o /tmp/dr && /tmp/dr
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "gc_common.cuh"
using namespace gc;

__global__ void kall(unsigned lo, unsigned long long count, float res, unsigned long long *bad, float *ex) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    const float y = recip_nr(res);
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const float t = __uint_as_float(lo + (unsigned)i);
        const float a = __fdiv_rn(t, res), b = div_rn_recip(t, res, y);
        const float fa = floorf(a);
        const int ca = fa < 0.f ? 0 : (fa > 4095.f ? 4095 : (int)fa);  // the reference's cell
        const int cb = floor_clamp(b, 4095.f);                         // K2's
        if (ca != cb) {
            unsigned long long j = atomicAdd(bad, 1ull);
            if (j < 4) { ex[3 * j] = t; ex[3 * j + 1] = a; ex[3 * j + 2] = b; }
        }
        if (__float_as_uint(a) != __float_as_uint(b) && fabsf(a) >= 7.88860905e-31f) atomicAdd(bad + 1, 1ull);
    }
}

int main(int argc, char **argv) {
    float def[] = {0.1f, 0.05f, 0.2f, 0.25f, 0.5f, 1.0f, 0.3f, 0.15f, 0.02f, 0.07f, 0.125f, 0.033f};
    int nres = argc > 1 ? argc - 1 : (int)(sizeof(def) / sizeof(def[0]));
    unsigned long long *bad;
    float *ex;
    cudaMalloc(&bad, 16);
    cudaMalloc(&ex, 64);
    int fail = 0;
    for (int r = 0; r < nres; ++r) {
        const float res = argc > 1 ? (float)atof(argv[r + 1]) : def[r];
        const float lim = 4096.0f * res;
        unsigned hi;
        memcpy(&hi, &lim, 4);
        unsigned long long total = 0, nbad = 0, nbits = 0;
        for (int sign = 0; sign < 2; ++sign) {  // [0, lim] and [-lim, -0]
            const unsigned lo = sign ? 0x80000000u : 0u;
            const unsigned long long count = (unsigned long long)hi + 1;
            cudaMemset(bad, 0, 16);
            kall<<<148 * 16, 256>>>(lo, count, res, bad, ex);
            unsigned long long bb[2] = {0, 0};
            cudaMemcpy(bb, bad, 16, cudaMemcpyDeviceToHost);
            const unsigned long long b = bb[0];
            nbits += bb[1];
            if (b) {
                float e[12];
                cudaMemcpy(e, ex, sizeof(e), cudaMemcpyDeviceToHost);
                printf("  e.g. t=%.9g ieee=%.9g recip=%.9g\n", e[0], e[1], e[2]);
            }
            nbad += b;
            total += count;
        }
        printf("res %.9g: cell mismatches: %llu of %llu (quotient bit mismatches above 2^-100: %llu)\n", res, nbad,
               total, nbits);
        fail |= nbad != 0;
    }
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(err)); return 2; }
    return fail;
}
