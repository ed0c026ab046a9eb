// Pinned H2D bandwidth: default pinned vs write-combined vs mapped host memory (1 GiB, best of 5).
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const size_t n = 1ull << 30;
    void* d; cudaMalloc(&d, n);
    const unsigned flags[] = {cudaHostAllocDefault, cudaHostAllocPortable, cudaHostAllocWriteCombined,
                              cudaHostAllocPortable | cudaHostAllocWriteCombined, cudaHostAllocMapped};
    const char* names[] = {"default", "portable", "write-combined", "portable|wc", "mapped"};
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int f = 0; f < 5; ++f) {
        void* h; cudaHostAlloc(&h, n, flags[f]);
        memset(h, 1, n);
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a, s);
            cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        float best2 = 1e9;  // D2H
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(a, s);
            cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (ms < best2) best2 = ms;
        }
        printf("%-16s H2D %.1f GB/s  D2H %.1f GB/s\n", names[f], n / best / 1e6, n / best2 / 1e6);
        cudaFreeHost(h);
    }
}
