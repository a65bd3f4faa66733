// Test harness: the device numpy-exp restatements over a device array, for an exhaustive
// comparison with numpy's own float32 exp (tests/test_gpu_exp_packed.py).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -ftz=false -prec-div=true --fmad=false
//        -shared -Xcompiler -fPIC -I paper_2603_01122_b200/csrc tools/cuda_checks/exp_lib.cu -o libexp.so
#include "gc_common.cuh"
using namespace gc;

__global__ void k_exp(const float *x, float *y, float *y2, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * i + 1 < n) {
        const float2 r = exp_np2(make_float2(x[2 * i], x[2 * i + 1]));
        y2[2 * i] = r.x;
        y2[2 * i + 1] = r.y;
    } else if (2 * i < n) {
        y2[2 * i] = exp_np(x[2 * i]);
    }
    for (long long j = 2 * i; j < 2 * i + 2 && j < n; ++j) y[j] = exp_np(x[j]);
}

extern "C" int exp_np_batch(const float *d_x, float *d_y, float *d_y2, long long n, void *stream) {
    k_exp<<<(unsigned)((n / 2 + 256) / 256), 256, 0, (cudaStream_t)stream>>>(d_x, d_y, d_y2, n);
    return (int)cudaGetLastError();
}
