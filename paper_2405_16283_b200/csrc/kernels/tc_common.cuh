// Device-side helpers shared by the tcgen05 kernels: mbarriers, TMA, tcgen05
// (MMA / commit / fences / TMEM loads+stores) and UMMA smem descriptors.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "kernels.hpp"

namespace tn::k {

// PDL: let the next kernel on the stream launch once every CTA of this one
// has started (pdl_trigger at entry), and wait for the previous kernel's
// completion + memory visibility before touching global memory (pdl_wait).
// Both are no-ops when the launch carries no PDL attribute.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint32_t bar, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint32_t bar, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(std::uint32_t bar, std::uint32_t parity) {
    std::uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(0x989680u)  // suspend-time hint: sleep in HW instead of spinning
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ bool mbar_test(std::uint32_t bar, std::uint32_t parity) {  // non-blocking
    std::uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(std::uint32_t bar, std::uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ void tma_load_3d(std::uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            std::uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
// MMA issue helpers: called by a whole converged warp; one elected lane
// issues. Warp-wide calls let ptxas keep the descriptors in uniform
// registers — issuing from a single divergent lane costs ~40 instructions per
// MMA (ELECT/R2UR broadcast loops), more than a short MMA's execution time.
__device__ __forceinline__ void tc_commit(std::uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
        : "memory");
}
__device__ __forceinline__ void tc_mma(std::uint32_t d, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                       std::uint32_t accum, bool tf32) {
    if (tf32) {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(accum)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(accum)
            : "memory");
    }
}
// A operand from tensor memory (rows = lanes, K packed two 16-bit values per
// 32-bit column), B from shared memory.
__device__ __forceinline__ void tc_mma_ts(std::uint32_t d, std::uint32_t a_tmem, std::uint64_t b, std::uint32_t idesc,
                                          std::uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum)
        : "memory");
}
// K-major operand in a SWIZZLE_128B layout: rows of 128 B, 8-row groups
// 1024 B apart (SBO), LBO unused, descriptor version 1 (sm_100).
__device__ __forceinline__ std::uint64_t sdesc(std::uint32_t saddr) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((saddr & 0x3FFFF) >> 4);
    d |= static_cast<std::uint64_t>(1) << 16;
    d |= static_cast<std::uint64_t>(1024 >> 4) << 32;
    d |= static_cast<std::uint64_t>(1) << 46;
    d |= static_cast<std::uint64_t>(2) << 61;
    return d;
}

#define TN_LD32(taddr, r)                                                                                     \
    asm volatile(                                                                                             \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                   \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),     \
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),            \
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),          \
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),          \
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                                                               \
        : "r"(taddr))


#define TN_ST32(taddr, r)                                                                                     \
    asm volatile(                                                                                             \
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16," \
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),                    \
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),   \
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),       \
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),      \
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])                   \
        : "memory")

#define TN_ST16(taddr, r)                                                                                     \
    asm volatile(                                                                                             \
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" \
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),  \
        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])           \
        : "memory")

// max(a, b, c) in one instruction (FMNMX3, sm_100).
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// 2^x on the SFU (MUFU.EX2), flushing denormal results to zero.
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Packed fp32 pairs (FFMA2 / FADD2, sm_100): each lane is rounded exactly
// like the scalar fmaf / fadd, at half the issue cost.
__device__ __forceinline__ void fma2(float& a, float& b, float m, float c) {  // a = a*m + c, b = b*m + c
    asm("{\n\t.reg .b64 t, u, v;\n\tmov.b64 t, {%0, %1};\n\tmov.b64 u, {%2, %2};\n\tmov.b64 v, {%3, %3};\n\t"
        "fma.rn.f32x2 t, t, u, v;\n\tmov.b64 {%0, %1}, t;\n\t}"
        : "+f"(a), "+f"(b)
        : "f"(m), "f"(c));
}
__device__ __forceinline__ void fma2v(float& a, float& b, float x, float y, float c) {  // a = a*x + c, b = b*y + c
    asm("{\n\t.reg .b64 t, u, v;\n\tmov.b64 t, {%0, %1};\n\tmov.b64 u, {%2, %3};\n\tmov.b64 v, {%4, %4};\n\t"
        "fma.rn.f32x2 t, t, u, v;\n\tmov.b64 {%0, %1}, t;\n\t}"
        : "+f"(a), "+f"(b)
        : "f"(x), "f"(y), "f"(c));
}
__device__ __forceinline__ void add2(float& a, float& b, float x, float y) {  // a += x, b += y
    asm("{\n\t.reg .b64 t, u;\n\tmov.b64 t, {%0, %1};\n\tmov.b64 u, {%2, %3};\n\t"
        "add.rn.f32x2 t, t, u;\n\tmov.b64 {%0, %1}, t;\n\t}"
        : "+f"(a), "+f"(b)
        : "f"(x), "f"(y));
}

__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tmem_alloc(std::uint32_t slot_smem, std::uint32_t cols) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(slot_smem), "r"(cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_free(std::uint32_t taddr, std::uint32_t cols) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}
// Instruction descriptor: D fp32, A/B format (1 bf16, 2 tf32), both K-major, M x N.
__host__ __device__ constexpr std::uint32_t make_idesc(std::uint32_t fmt, int M, int N) {
    return (1u << 4) | (fmt << 7) | (fmt << 10) | (static_cast<std::uint32_t>(N >> 3) << 17) |
           (static_cast<std::uint32_t>(M >> 4) << 24);
}

// CTA-pair (cta_group::2) helpers: cluster rank, peer smem addresses, TMA
// loads that signal the leader CTA's barrier, pair MMAs and multicast commits.
__device__ __forceinline__ std::uint32_t cluster_rank() {
    std::uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ std::uint32_t mapa(std::uint32_t addr, std::uint32_t rank) {
    std::uint32_t out;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
    return out;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d_2sm(std::uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                std::uint32_t leader_bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<std::uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(leader_bar)
        : "memory");
}
__device__ __forceinline__ void tc_mma_2sm(std::uint32_t d, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                           std::uint32_t accum, bool tf32) {
    if (tf32) {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(accum)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc), "r"(accum)
            : "memory");
    }
}
__device__ __forceinline__ void tc_commit_2sm(std::uint32_t bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(bar),
        "h"(static_cast<unsigned short>(3))
        : "memory");
}
// Arrive on a barrier in a peer CTA's shared memory (mapa address). Default
// .release.cta semantics: the arrivals here only publish tensor-memory
// accesses, which the tcgen05 fences order; .release.cluster would add a
// MEMBAR.ALL.GPU to every arrive.
__device__ __forceinline__ void mbar_arrive_remote(std::uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// Pair MMA with the A operand from tensor memory (each CTA's TMEM holds its
// 128 rows of A at the same address), B from shared memory.
__device__ __forceinline__ void tc_mma_ts_2sm(std::uint32_t d, std::uint32_t a_tmem, std::uint64_t b,
                                              std::uint32_t idesc, std::uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 r;\n\telect.sync r|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(accum)
        : "memory");
}

// Kernel launch with the PDL attribute when the dispatcher enabled it.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t s,
                       Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

}  // namespace tn::k
