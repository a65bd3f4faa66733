// D2H bandwidth: cudaMemcpyAsync (copy engine) vs a kernel storing straight into mapped
// pinned host memory (zero-copy over PCIe / C2C), for the e2e union sizes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/cuda_checks/zerocopy_bw.cu -o /tmp/zc && /tmp/zc
#include <cstdio>

__global__ void kstore(const float4 *src, float4 *dst, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const size_t sizes[] = {16u << 20, 64u << 20, 320u << 20};
    for (size_t bytes : sizes) {
        void *d, *h, *hm;
        cudaMalloc(&d, bytes);
        cudaMemset(d, 1, bytes);
        cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
        cudaHostAlloc(&hm, bytes, cudaHostAllocMapped);
        float4 *hdev;
        cudaHostGetDevicePointer((void **)&hdev, hm, 0);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int w = 0; w < 2; ++w) cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%4zu MB memcpy D2H: %.1f GB/s\n", bytes >> 20, 5 * bytes / (ms * 1e6));
        for (int blocks : {16, 64, 148, 296, 592}) {
            kstore<<<blocks, 512>>>((const float4 *)d, hdev, bytes / 16);
            cudaEventRecord(a);
            for (int r = 0; r < 5; ++r) kstore<<<blocks, 512>>>((const float4 *)d, hdev, bytes / 16);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
            printf("%4zu MB kernel stores to mapped host memory, %3d CTAs: %.1f GB/s\n", bytes >> 20, blocks,
                   5 * bytes / (ms * 1e6));
        }
        cudaFree(d);
        cudaFreeHost(h);
        cudaFreeHost(hm);
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
