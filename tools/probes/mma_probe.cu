// Micro-probe: tcgen05.mma (kind::f16, cta_group::1, M = 128) issue-to-completion
// cycles per instruction for the shapes the attention kernel uses, operands
// from shared memory (SS) or A from tensor memory (TS), with 1 or 2 CTAs per
// SM issuing concurrently. Floor (tcgen05 pacing): 128 * N / 256 clk per MMA.
// Build + run:
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2405_16283_b200/csrc/kernels -o /tmp/mma_probe tools/probes/mma_probe.cu -lcuda && /tmp/mma_probe
#include <cstdio>

#include "tc_common.cuh"

namespace tn::k {
void set_pdl(bool) {}
bool pdl_enabled() { return false; }
}  // namespace tn::k

using namespace tn::k;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 2) probe(int iters, long long* out) {
    extern __shared__ __align__(1024) std::uint8_t smem[];
    // A: 128 rows x 128 B, B: N rows x 128 B (SW128 K-major atoms), then barrier + TMEM slot
    const std::uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
    const std::uint32_t sA = base, sB = base + 128 * 128;
    const std::uint32_t bar = sB + N * 128, slot = bar + 8;
    for (int i = threadIdx.x; i < (128 + N) * 128 / 16; i += blockDim.x)
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(base + i * 16), "r"(0x3c003c00u));
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_async_smem();
    if (threadIdx.x / 32 == 0) tmem_alloc(slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    std::uint32_t tmem;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(slot));
    if (threadIdx.x / 32 == 0) {
        const std::uint32_t idesc = make_idesc(1u, 128, N);
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (TS)
                    tc_mma_ts(tmem, tmem + 128 + kk * 8, sdesc(sB + kk * 32), idesc, (it | kk) != 0);
                else
                    tc_mma(tmem, sdesc(sA + kk * 32), sdesc(sB + kk * 32), idesc, (it | kk) != 0, false);
            }
        }
        tc_commit(bar);
        mbar_wait(bar, 0);
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x / 32 == 0) tmem_free(tmem, 256);
}

template <int N, bool TS>
void run(int cps) {
    const int grid = 148 * cps, iters = 2048;
    long long* d;
    cudaMalloc(&d, grid * sizeof(long long));
    const int smem = 1024 + (128 + N) * 128 + 64;
    cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) probe<N, TS><<<grid, 128, smem>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[296];
    cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < grid; ++i) avg += h[i];
    avg /= grid;
    const double per = avg / (iters * 4.0), floor = 128.0 * N / 256.0;
    printf("{\"N\": %d, \"a_operand\": \"%s\", \"ctas_per_sm\": %d, \"clk_per_mma\": %.1f, \"floor_clk\": %.0f, "
           "\"frac_of_floor\": %.3f, \"err\": \"%s\"}\n",
           N, TS ? "tmem" : "smem", cps, per, floor, floor * cps / per, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    for (int cps = 1; cps <= 2; ++cps) {
        run<64, false>(cps);
        run<64, true>(cps);
        run<128, false>(cps);
        run<128, true>(cps);
    }
    run<256, false>(1);
    return 0;
}
