// Micro-probe: tcgen05.mma.cta_group::2 (kind::f16, M = 256 over a CTA pair)
// throughput (back-to-back) and batch latency (8 MMAs issued, commit, wait)
// for N = 64/128/256, A from shared memory (SS) or tensor memory (TS).
// Build + run:
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a \
//        -I paper_2405_16283_b200/csrc/kernels -o /tmp/mma2_probe tools/probes/mma2_probe.cu -lcuda && /tmp/mma2_probe
#include <cstdio>

#include "tc_common.cuh"

namespace tn::k {
void set_pdl(bool) {}
bool pdl_enabled() { return false; }
}  // namespace tn::k

using namespace tn::k;

template <int N, bool TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(int iters, long long* out) {
    extern __shared__ __align__(1024) std::uint8_t smem[];
    const std::uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
    const std::uint32_t sA = base, sB = base + 128 * 128;  // A: 128 rows x 128 B; B: N/2 rows x 128 B per CTA
    const std::uint32_t bar = sB + N * 128, slot = bar + 8;
    for (int i = threadIdx.x; i < (128 + N) * 128 / 16; i += blockDim.x)
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(base + i * 16), "r"(0x3c003c00u));
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    fence_async_smem();
    if (threadIdx.x / 32 == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot), "r"(512) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    std::uint32_t tmem;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem) : "r"(slot));
    const bool leader = cluster_rank() == 0;
    long long thr = 0, lat = 0;
    if (threadIdx.x / 32 == 0 && leader) {
        const std::uint32_t idesc = make_idesc(1u, 256, N);
        std::uint32_t ph = 0;
        // throughput: iters x 4 MMAs back to back
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (TS) tc_mma_ts_2sm(tmem, tmem + 256 + kk * 8, sdesc(sB + kk * 32), idesc, (it | kk) != 0);
                else tc_mma_2sm(tmem, sdesc(sA + kk * 32), sdesc(sB + kk * 32), idesc, (it | kk) != 0, false);
            }
        }
        tc_commit_2sm(bar);
        mbar_wait(bar, ph);
        ph ^= 1;
        thr = clock64() - t0;
        // latency: 8 MMAs + commit + wait, repeated
        long long t1 = clock64();
        for (int r = 0; r < 64; ++r) {
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                if (TS) tc_mma_ts_2sm(tmem, tmem + 256 + (kk & 3) * 8, sdesc(sB + (kk & 3) * 32), idesc, kk != 0);
                else tc_mma_2sm(tmem, sdesc(sA + (kk & 3) * 32), sdesc(sB + (kk & 3) * 32), idesc, kk != 0, false);
            }
            tc_commit_2sm(bar);
            mbar_wait(bar, ph);
            ph ^= 1;
        }
        lat = clock64() - t1;
        if (threadIdx.x == 0) {
            out[2 * (blockIdx.x / 2)] = thr;
            out[2 * (blockIdx.x / 2) + 1] = lat;
        }
    } else if (threadIdx.x / 32 == 0) {
        // the peer's barrier also receives the multicast commits: consume them
        for (int r = 0; r < 65; ++r) mbar_wait(bar, r & 1);
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (threadIdx.x / 32 == 0)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

template <int N, bool TS>
void run() {
    const int grid = 148, iters = 1024;
    long long* d;
    cudaMalloc(&d, grid * sizeof(long long));
    const int smem = 1024 + (128 + N) * 128 + 64;
    cudaFuncSetAttribute(probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 2; ++rep) probe<N, TS><<<grid, 128, smem>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double thr = 0, lat = 0;
    for (int i = 0; i < grid / 2; ++i) thr += h[2 * i], lat += h[2 * i + 1];
    thr /= grid / 2;
    lat /= grid / 2;
    const double per = thr / (iters * 4.0), floor = 128.0 * N / 256.0;
    printf("{\"cta_group\": 2, \"N\": %d, \"a_operand\": \"%s\", \"clk_per_mma\": %.1f, \"floor_clk\": %.0f, "
           "\"batch8_latency_clk\": %.0f, \"err\": \"%s\"}\n",
           N, TS ? "tmem" : "smem", per, floor, lat / 64.0, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<64, false>();
    run<128, false>();
    run<128, true>();
    run<256, false>();
    run<256, true>();
    return 0;
}
