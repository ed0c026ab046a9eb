// Micro-probe: MUFU.EX2 throughput per SM for f32 vs f16x2 vs bf16x2 inputs
// (results per clock per SM). Build + run: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/mufu mufu_probe.cu && /tmp/mufu
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
template <int MODE>
__global__ void k(float* out, int iters, long long* clk) {
    float a[16];
    unsigned h[16];
    for (int i = 0; i < 16; ++i) { a[i] = -0.001f * (threadIdx.x + i); h[i] = 0x3c003c00u ^ (threadIdx.x + i); }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            else if (MODE == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
            else asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[i]));
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 16; ++i) s += a[i] + __uint_as_float(h[i]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
int main() {
    float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 8);
    const int iters = 4096;
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) k<0><<<148, 1024>>>(o, iters, c);
            if (mode == 1) k<1><<<148, 1024>>>(o, iters, c);
            if (mode == 2) k<2><<<148, 1024>>>(o, iters, c);
            cudaDeviceSynchronize();
        }
        long long clk; cudaMemcpy(&clk, c, 8, cudaMemcpyDeviceToHost);
        double ops = 1024.0 * iters * 16;  // MUFU instructions (lanes) per SM
        double res = ops * (mode == 0 ? 1 : 2);
        printf("mode %s: %.2f lane-ops/clk/SM, %.2f results/clk/SM (%s)\n", mode == 0 ? "f32" : mode == 1 ? "f16x2" : "bf16x2",
               ops / clk, res / clk, cudaGetErrorString(cudaGetLastError()));
    }
}
