// Probe: tcgen05.mma kind::f16 with the B operand MN-major (N contiguous,
// SWIZZLE_128B: 64-element N chunks of 8 K-rows x 128 B) — finds the smem
// descriptor LBO / SBO that reproduce C = A·B (A K-major) for M = 128,
// N = 128, K = 64. Build + run:
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2405_16283_b200/csrc/kernels -o /tmp/mn tools/probes/mn_major_probe.cu -lcuda && /tmp/mn
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "tc_common.cuh"

namespace tn::k {
void set_pdl(bool) {}
bool pdl_enabled() { return false; }
}  // namespace tn::k
using namespace tn::k;

constexpr int M = 128, N = 128, K = 64;

__device__ __forceinline__ std::uint64_t desc_gen(std::uint32_t saddr, std::uint32_t lbo, std::uint32_t sbo) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((saddr & 0x3FFFF) >> 4);
    d |= static_cast<std::uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<std::uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<std::uint64_t>(1) << 46;
    d |= static_cast<std::uint64_t>(2) << 61;
    return d;
}

__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* C, int lbo, int sbo, int kstep) {
    extern __shared__ __align__(1024) std::uint8_t smem[];
    const std::uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
    std::uint8_t* gbase = smem + (base - smem_u32(smem));
    const std::uint32_t sA = base, sB = base + M * 128;
    const std::uint32_t bar = sB + 2 * 8192, slot = bar + 8;
    // A: K-major SW128: row m (128 B = 64 K elems), 16-byte chunk c at (c ^ (m & 7))
    for (int i = threadIdx.x; i < M * 8; i += blockDim.x) {
        const int m = i / 8, c = i % 8;
        uint4 v = *reinterpret_cast<const uint4*>(A + m * K + c * 8);
        *reinterpret_cast<uint4*>(gbase + m * 128 + ((c ^ (m & 7)) * 16)) = v;
    }
    // B (K x N, N contiguous): box b (64 N cols) at b*8192, K-row k at k*128, chunk c at (c ^ (k & 7))
    for (int i = threadIdx.x; i < K * (N / 8); i += blockDim.x) {
        const int k = i / (N / 8), cc = i % (N / 8), b = cc / 8, c = cc % 8;
        uint4 v = *reinterpret_cast<const uint4*>(B + k * N + cc * 8);
        *reinterpret_cast<uint4*>(gbase + M * 128 + b * 8192 + k * 128 + ((c ^ (k & 7)) * 16)) = v;
    }
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_async_smem();
    if (threadIdx.x / 32 == 0) tmem_alloc(slot, 128);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    std::uint32_t tmem;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(slot));
    if (threadIdx.x / 32 == 0) {
        const std::uint32_t idesc = make_idesc(1u, M, N) | (1u << 16);  // b_major = MN
        for (int kk = 0; kk < K / 16; ++kk)
            tc_mma(tmem, sdesc(sA + kk * 32), desc_gen(sB + kk * kstep, lbo, sbo), idesc, kk != 0, false);
        tc_commit(bar);
        mbar_wait(bar, 0);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (w < 4) {
        for (int c0 = 0; c0 < N; c0 += 32) {
            std::uint32_t r[32];
            TN_LD32(tmem + (static_cast<std::uint32_t>(w * 32) << 16) + c0, r);
            tc_wait_ld();
            for (int j = 0; j < 32; ++j) C[(w * 32 + lane) * N + c0 + j] = __uint_as_float(r[j]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x / 32 == 0) tmem_free(tmem, 128);
}

int main() {
    std::vector<__nv_bfloat16> hA(M * K), hB(K * N);
    std::vector<float> fA(M * K), fB(K * N);
    srand(1);
    for (int i = 0; i < M * K; ++i) { fA[i] = (rand() % 17 - 8) / 8.0f; hA[i] = __float2bfloat16(fA[i]); }
    for (int i = 0; i < K * N; ++i) { fB[i] = (rand() % 13 - 6) / 4.0f; hB[i] = __float2bfloat16(fB[i]); }
    std::vector<float> ref(M * N, 0.f);
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            float s = 0;
            for (int k = 0; k < K; ++k) s += fA[m * K + k] * fB[k * N + n];
            ref[m * N + n] = s;
        }
    __nv_bfloat16 *dA, *dB;
    float* dC;
    cudaMalloc(&dA, M * K * 2);
    cudaMalloc(&dB, K * N * 2);
    cudaMalloc(&dC, M * N * 4);
    cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), K * N * 2, cudaMemcpyHostToDevice);
    const int smem = 1024 + M * 128 + 2 * 8192 + 64;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int cand[][3] = {{8192, 1024, 2048}, {1024, 8192, 2048}, {8192, 1024, 256}, {1024, 8192, 256}};
    for (auto& c : cand) {
        cudaMemset(dC, 0, M * N * 4);
        probe<<<1, 128, smem>>>(dA, dB, dC, c[0], c[1], c[2]);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> hC(M * N);
        cudaMemcpy(hC.data(), dC, M * N * 4, cudaMemcpyDeviceToHost);
        double err = 0, nrm = 0;
        for (int i = 0; i < M * N; ++i) { err += (hC[i] - ref[i]) * (hC[i] - ref[i]); nrm += ref[i] * ref[i]; }
        printf("{\"lbo\": %d, \"sbo\": %d, \"kstep\": %d, \"rel_err\": %.3e, \"err\": \"%s\"}\n", c[0], c[1], c[2],
               std::sqrt(err / nrm), cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
