// Fused blockwise causal attention task: for one head and
// one 128-query block, O = softmax(scale · Q Kᵀ) V with an online softmax over
// 128-key blocks — the S/P tiles never leave the SM.
//
//   warp 0     TMA: Q once, then K_j / Vᵀ_j into a 2-stage ring
//   warp 1     one thread issues tcgen05.mma: S_j = Q·K_jᵀ into TMEM cols
//              [0,128), O += P_j·V_j into TMEM cols [128,256); S_{j+1} is issued
//              as soon as the softmax warps have pulled S_j into registers
//   warps 2-5  softmax/correction, one query row per thread: tcgen05.ld S_j,
//              running max/sum in fp32 (exp2 with log2e-folded scale), rescale O
//              in TMEM when the row max grows, P_j as bf16 into a 128B-swizzled
//              K-major smem tile (the A operand of the P·V MMA), final O / l
// Deterministic: fixed block order, fixed per-row reductions.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"
#include "tc_common.cuh"

namespace tn::k {
namespace {

constexpr int kB = 128;      // query rows / keys per block
constexpr int kHd = 128;     // head dim of the fused path
constexpr int kAtomB = 16384;  // one 128-row x 128-byte swizzle atom
constexpr int kTile = 2 * kAtomB;  // 128 x 128 bf16 = two atoms along K
constexpr int kThreads = 192;

struct AttnParams {
    __nv_bfloat16* O;
    int heads, seq, nblk;
    std::int64_t ldo;
    float scale_log2;
    int causal;
};

__device__ __forceinline__ void load_tile(std::uint32_t dst, const CUtensorMap* map, int inner0, int row0, int h,
                                          std::uint32_t bar) {
    tma_load_3d(dst, map, inner0, row0, h, bar);
    tma_load_3d(dst + kAtomB, map, inner0 + 64, row0, h, bar);
}

// P row r, keys [c0, c0+8) as one 16-byte chunk into the swizzled K-major tile.
__device__ __forceinline__ std::uint32_t p_chunk_addr(std::uint32_t base, int r, int key) {
    const int atom = key >> 6, chunk = (key & 63) >> 3;
    return base + atom * kAtomB + r * 128 + ((chunk ^ (r & 7)) << 4);
}

__global__ void __launch_bounds__(kThreads, 1)
    attention_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                     const __grid_constant__ CUtensorMap tv, const AttnParams p) {
    extern __shared__ std::uint8_t smem_raw[];
    const std::uint32_t raw = smem_u32(smem_raw);
    const std::uint32_t base = (raw + 1023) & ~1023u;
    // P is double-buffered so the softmax of block j+1 overlaps the P·V MMA of
    // block j (p_full / o_done are per-buffer barriers: each completes every
    // other block, so no waiter can fall two phases behind).
    const std::uint32_t sQ = base;
    const std::uint32_t sP[2] = {base + kTile, base + 2 * kTile};
    const std::uint32_t sK[2] = {base + 3 * kTile, base + 4 * kTile};
    const std::uint32_t sV[2] = {base + 5 * kTile, base + 6 * kTile};
    std::uint8_t* gen_base = smem_raw + (base - raw);
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(gen_base + 7 * kTile);
    const std::uint32_t b0 = smem_u32(bars);
    const std::uint32_t q_full = b0, kv_full = b0 + 8, kv_empty = b0 + 24, s_full = b0 + 40, s_free = b0 + 48,
                        p_full = b0 + 56, o_done = b0 + 72;  // p_full[2], o_done[2]
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 12);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // Heavy (late) query blocks first: blockIdx.x enumerates (qb desc, head).
    const int h = blockIdx.x % p.heads;
    const int qb = p.nblk - 1 - static_cast<int>(blockIdx.x / p.heads);
    const int nkv = p.causal ? qb + 1 : p.nblk;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tq)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tk)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tv)) : "memory");
        mbar_init(q_full, 1);
        mbar_init(kv_full, 1);
        mbar_init(kv_full + 8, 1);
        mbar_init(kv_empty, 1);
        mbar_init(kv_empty + 8, 1);
        mbar_init(s_full, 1);
        mbar_init(s_free, 4);
        mbar_init(p_full, 4);
        mbar_init(p_full + 8, 4);
        mbar_init(o_done, 1);
        mbar_init(o_done + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) tmem_alloc(smem_u32(tmem_slot), 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const std::uint32_t tmem = *tmem_slot;
    const std::uint32_t tS = tmem, tO = tmem + 128;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(q_full, kTile);
            load_tile(sQ, &tq, 0, qb * kB, h, q_full);
            for (int j = 0; j < nkv; ++j) {
                const int st = j & 1;
                mbar_wait(kv_empty + 8 * st, ((j >> 1) & 1) ^ 1);
                mbar_expect_tx(kv_full + 8 * st, 2 * kTile);
                load_tile(sK[st], &tk, 0, j * kB, h, kv_full + 8 * st);
                load_tile(sV[st], &tv, j * kB, 0, h, kv_full + 8 * st);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const std::uint32_t idesc = make_idesc(1u, kB, kB);
            auto issue_s = [&](int j) {
                const int st = j & 1;
                mbar_wait(kv_full + 8 * st, (j >> 1) & 1);
                if (j > 0) mbar_wait(s_free, (j - 1) & 1);  // softmax pulled S_{j-1}
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < kHd / 16; ++kk) {
                    const std::uint32_t off = (kk >> 2) * kAtomB + (kk & 3) * 32;
                    tc_mma(tS, sdesc(sQ + off), sdesc(sK[st] + off), idesc, kk != 0, false);
                }
                tc_commit(s_full);
            };
            mbar_wait(q_full, 0);
            issue_s(0);
            for (int j = 0; j < nkv; ++j) {
                if (j + 1 < nkv) issue_s(j + 1);
                const int pb = j & 1;
                mbar_wait(p_full + 8 * pb, (j >> 1) & 1);
                tc_fence_after();
                const int st = j & 1;
#pragma unroll
                for (int kk = 0; kk < kB / 16; ++kk) {
                    const std::uint32_t off = (kk >> 2) * kAtomB + (kk & 3) * 32;
                    tc_mma(tO, sdesc(sP[pb] + off), sdesc(sV[st] + off), idesc, (j | kk) != 0, false);
                }
                tc_commit(o_done + 8 * pb);
                tc_commit(kv_empty + 8 * st);
            }
        }
    } else {
        const int lane_base = (warp % 4) * 32;
        const int r = lane_base + lane;  // query row within the block
        const std::uint32_t trow = static_cast<std::uint32_t>(lane_base) << 16;
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nkv; ++j) {
            mbar_wait(s_full, j & 1);
            tc_fence_after();
            float s[kB];
#pragma unroll
            for (int c = 0; c < kB; c += 32) {
                std::uint32_t u[32];
                TN_LD32(tS + trow + c, u);
#pragma unroll
                for (int i = 0; i < 32; ++i) s[c + i] = __uint_as_float(u[i]);
            }
            tc_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(s_free);

            const bool diag = p.causal && j == qb;
            // 8 independent max / sum chains (a fixed tree, so still
            // deterministic): one warp per SMSP cannot hide a 128-long chain.
            // Max is taken on raw scores (scale > 0), then p = 2^(s*scale - m)
            // is one FFMA + one MUFU.EX2 per element.
            constexpr int kW = 8;
            float pm[kW];
#pragma unroll
            for (int w = 0; w < kW; ++w) pm[w] = -INFINITY;
            if (diag) {
#pragma unroll
                for (int c = 0; c < kB; ++c) {
                    if (c > r) s[c] = -INFINITY;
                    pm[c % kW] = fmaxf(pm[c % kW], s[c]);
                }
            } else {
#pragma unroll
                for (int c = 0; c < kB; ++c) pm[c % kW] = fmaxf(pm[c % kW], s[c]);
            }
#pragma unroll
            for (int w = kW / 2; w > 0; w /= 2)
#pragma unroll
                for (int i = 0; i < w; ++i) pm[i] = fmaxf(pm[i], pm[i + w]);
            const float mx = fmaxf(m, pm[0] * p.scale_log2);
            const float corr = ex2(m - mx);  // 0 on the first block (m = -inf)
            float ps[kW];
#pragma unroll
            for (int w = 0; w < kW; ++w) ps[w] = 0.f;
#pragma unroll
            for (int c = 0; c < kB; ++c) {
                s[c] = ex2(fmaf(s[c], p.scale_log2, -mx));
                ps[c % kW] += s[c];
            }
#pragma unroll
            for (int w = kW / 2; w > 0; w /= 2)
#pragma unroll
                for (int i = 0; i < w; ++i) ps[i] += ps[i + w];
            const float sum = ps[0];
            l = l * corr + sum;
            const bool grew = mx > m;
            m = mx;

            const int pb = j & 1;
            if (j >= 2) mbar_wait(o_done + 8 * pb, ((j - 2) >> 1) & 1);  // P_{j-2}·V done: buffer pb free
            if (j > 0 && __any_sync(0xffffffffu, grew)) {
                mbar_wait(o_done + 8 * ((j - 1) & 1), ((j - 1) >> 1) & 1);  // P_{j-1}·V done: O stable
                tc_fence_after();
                {
#pragma unroll 1
                    for (int c = 0; c < kB; c += 32) {
                        std::uint32_t u[32];
                        TN_LD32(tO + trow + c, u);
                        tc_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * corr);
                        TN_ST32(tO + trow + c, u);
                    }
                    tc_wait_st();
                }
            }
#pragma unroll
            for (int c = 0; c < kB; c += 8) {
                uint4 v;
                __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
                for (int i = 0; i < 4; ++i) hv[i] = __floats2bfloat162_rn(s[c + 2 * i], s[c + 2 * i + 1]);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(p_chunk_addr(sP[pb], r, c)), "r"(v.x),
                             "r"(v.y), "r"(v.z), "r"(v.w)
                             : "memory");
            }
            fence_async_smem();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full + 8 * pb);
        }
        // Epilogue: O / l -> bf16 rows of the [seq, heads*hd] output.
        mbar_wait(o_done + 8 * ((nkv - 1) & 1), ((nkv - 1) >> 1) & 1);
        tc_fence_after();
        const float inv = 1.0f / l;
        __nv_bfloat16* orow = p.O + static_cast<std::int64_t>(qb * kB + r) * p.ldo + static_cast<std::int64_t>(h) * kHd;
#pragma unroll 1
        for (int c = 0; c < kHd; c += 32) {
            std::uint32_t u[32];
            TN_LD32(tO + trow + c, u);
            tc_wait_ld();
            uint4* dst = reinterpret_cast<uint4*>(orow + c);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                uint4 v;
                __nv_bfloat162* hv = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    hv[i] = __floats2bfloat162_rn(__uint_as_float(u[q * 8 + 2 * i]) * inv,
                                                  __uint_as_float(u[q * 8 + 2 * i + 1]) * inv);
                dst[q] = v;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_free(tmem, 256);
}

constexpr int kSmem = 7 * kTile + 128 + 1024;

// --- SIMT fallback (any seq / head dim): one warp per query row, fp32 online
// softmax over all keys in order. Slow; only for shapes the fused path rejects.
__global__ void attention_simt(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                               const __nv_bfloat16* __restrict__ vt, __nv_bfloat16* __restrict__ O, int heads, int seq,
                               int hd, std::int64_t ldo, float scale_log2, int causal) {
    const std::int64_t w = (static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (w >= static_cast<std::int64_t>(heads) * seq) return;
    const int h = static_cast<int>(w / seq), i = static_cast<int>(w % seq);
    const __nv_bfloat16* qi = q + (static_cast<std::int64_t>(h) * seq + i) * hd;
    const int nk = causal ? i + 1 : seq;
    float m = -INFINITY, l = 0.f;
    float acc[8];  // hd <= 256: lane owns columns lane, lane+32, ...
    for (int c = 0; c < 8; ++c) acc[c] = 0.f;
    for (int j = 0; j < nk; ++j) {
        const __nv_bfloat16* kj = k + (static_cast<std::int64_t>(h) * seq + j) * hd;
        float d = 0.f;
        for (int c = lane; c < hd; c += 32) d += __bfloat162float(qi[c]) * __bfloat162float(kj[c]);
        for (int o = 16; o > 0; o /= 2) d += __shfl_xor_sync(0xffffffffu, d, o);
        const float x = d * scale_log2;
        const float mx = fmaxf(m, x), corr = exp2f(m - mx), pj = exp2f(x - mx);
        l = l * corr + pj;
        for (int c = 0; c < 8; ++c) {
            const int col = lane + 32 * c;
            if (col < hd) acc[c] = acc[c] * corr + pj * __bfloat162float(vt[(static_cast<std::int64_t>(h) * hd + col) * seq + j]);
        }
        m = mx;
    }
    for (int c = 0; c < 8; ++c) {
        const int col = lane + 32 * c;
        if (col < hd) O[static_cast<std::int64_t>(i) * ldo + static_cast<std::int64_t>(h) * hd + col] = __float2bfloat16_rn(acc[c] / l);
    }
}

}  // namespace

cudaError_t attention_prepare(const AttnArgs& a, AttnPlan* plan) {
    plan->args = a;
    auto al16 = [](const void* x) { return (reinterpret_cast<std::uintptr_t>(x) & 15) == 0; };
    bool ok = a.hd == kHd && a.seq % kB == 0 && a.seq >= kB && al16(a.q) && al16(a.k) && al16(a.vt) && al16(a.out) &&
              (a.ldo * 2) % 16 == 0;
    if (ok)
        ok = encode_tma_3d(&plan->tq, a.q, 2, a.hd, a.seq, a.hd, a.heads, static_cast<std::int64_t>(a.seq) * a.hd, 64,
                           kB) &&
             encode_tma_3d(&plan->tk, a.k, 2, a.hd, a.seq, a.hd, a.heads, static_cast<std::int64_t>(a.seq) * a.hd, 64,
                           kB) &&
             encode_tma_3d(&plan->tv, a.vt, 2, a.seq, a.hd, a.seq, a.heads, static_cast<std::int64_t>(a.seq) * a.hd, 64,
                           kHd);
    plan->path = ok ? 0 : 1;
    if (ok) {
        static unsigned long long attr_set = 0;
        int dev = 0;
        cudaGetDevice(&dev);
        if (!((attr_set >> dev) & 1ULL)) {
            cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
            attr_set |= 1ULL << dev;
        }
    }
    return cudaSuccess;
}

cudaError_t attention_launch(const AttnPlan& plan, cudaStream_t s) {
    const AttnArgs& a = plan.args;
    const float sl2 = a.scale * 1.4426950408889634f;
    if (plan.path == 1) {
        const std::int64_t warps = static_cast<std::int64_t>(a.heads) * a.seq;
        attention_simt<<<static_cast<unsigned>((warps * 32 + 255) / 256), 256, 0, s>>>(
            static_cast<const __nv_bfloat16*>(a.q), static_cast<const __nv_bfloat16*>(a.k),
            static_cast<const __nv_bfloat16*>(a.vt), static_cast<__nv_bfloat16*>(a.out), a.heads, a.seq, a.hd, a.ldo,
            sl2, a.causal);
        return cudaGetLastError();
    }
    AttnParams p;
    p.O = static_cast<__nv_bfloat16*>(a.out);
    p.heads = a.heads;
    p.seq = a.seq;
    p.nblk = a.seq / kB;
    p.ldo = a.ldo;
    p.scale_log2 = sl2;
    p.causal = a.causal;
    attention_kernel<<<p.heads * p.nblk, kThreads, kSmem, s>>>(plan.tq, plan.tk, plan.tv, p);
    return cudaGetLastError();
}

double attention_flops(const AttnArgs& a) {
    double f = 4.0 * a.heads * static_cast<double>(a.seq) * a.seq * a.hd;
    return a.causal ? f * 0.5 * (1.0 + 1.0 / a.seq) : f;
}

}  // namespace tn::k
