// Check: div_rn_recip(t, res, fl(1/res)) (gc_common.cuh; K2's production cell map) is
// bit-identical to the IEEE quotient __fdiv_rn(t, res) for EVERY float32 t with
// |t| <= 4096 res, for each resolution given on the command line (default: a set of usual
// grid resolutions).  Prints "mismatches: N of M" per resolution; exit 1 on any mismatch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -ftz=false -prec-div=true
//        -I paper_2603_01122_b200/csrc tools/cuda_checks/div_recip.cu -o /tmp/dr && /tmp/dr
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include "gc_common.cuh"
using namespace gc;

__global__ void kall(unsigned lo, unsigned long long count, float res, float inv, unsigned long long *bad, float *ex) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
        const float t = __uint_as_float(lo + (unsigned)i);
        const float a = __fdiv_rn(t, res), b = div_rn_recip(t, res, inv);
        if (__float_as_uint(a) != __float_as_uint(b)) {
            unsigned long long j = atomicAdd(bad, 1ull);
            if (j < 4) { ex[3 * j] = t; ex[3 * j + 1] = a; ex[3 * j + 2] = b; }
        }
    }
}

int main(int argc, char **argv) {
    float def[] = {0.1f, 0.05f, 0.2f, 0.25f, 0.5f, 1.0f, 0.3f, 0.15f, 0.02f, 0.07f, 0.125f, 0.033f};
    int nres = argc > 1 ? argc - 1 : (int)(sizeof(def) / sizeof(def[0]));
    unsigned long long *bad;
    float *ex;
    cudaMalloc(&bad, 8);
    cudaMalloc(&ex, 64);
    int fail = 0;
    for (int r = 0; r < nres; ++r) {
        const float res = argc > 1 ? (float)atof(argv[r + 1]) : def[r];
        const float inv = 1.0f / res;  // host IEEE division, as gc_predict computes it
        const float lim = 4096.0f * res;
        unsigned hi;
        memcpy(&hi, &lim, 4);
        unsigned long long total = 0, nbad = 0;
        for (int sign = 0; sign < 2; ++sign) {  // [0, lim] and [-lim, -0]
            const unsigned lo = sign ? 0x80000000u : 0u;
            const unsigned long long count = (unsigned long long)hi + 1;
            cudaMemset(bad, 0, 8);
            kall<<<148 * 16, 256>>>(lo, count, res, inv, bad, ex);
            unsigned long long b = 0;
            cudaMemcpy(&b, bad, 8, cudaMemcpyDeviceToHost);
            if (b) {
                float e[12];
                cudaMemcpy(e, ex, sizeof(e), cudaMemcpyDeviceToHost);
                printf("  e.g. t=%.9g ieee=%.9g recip=%.9g\n", e[0], e[1], e[2]);
            }
            nbad += b;
            total += count;
        }
        printf("res %.9g: mismatches: %llu of %llu\n", res, nbad, total);
        fail |= nbad != 0;
    }
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(err)); return 2; }
    return fail;
}
