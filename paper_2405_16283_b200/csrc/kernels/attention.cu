// Fused blockwise causal attention task: for one head and
// one 128-query block, O = softmax(scale · Q Kᵀ) V with an online softmax over
// 64-key blocks — the S/P tiles never leave the SM. 96 KB of smem and 256
// TMEM columns per CTA, two CTAs per SM.
//
//   warp 0     TMA: Q once, then K_j (2-stage ring) and Vᵀ_j
//   warp 1     one thread issues tcgen05.mma: S_j = Q·K_jᵀ (M=128, N=64) into
//              TMEM cols [0,64), O += P_j·V_j (M=128, N=128, K=64) into cols
//              [128,256); S_{j+1} is issued as soon as the softmax warps have
//              pulled S_j into registers
//   warps 2-5  softmax/correction, one query row per thread: tcgen05.ld S_j,
//              running max/sum in fp32 (exp2 with log2e-folded scale), rescale O
//              in TMEM when the row max grows, P_j as bf16 into a 128B-swizzled
//              K-major smem tile (the A operand of the P·V MMA), final O / l
// Deterministic: fixed block order, fixed per-row reductions.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "kernels.hpp"
#include "tc_common.cuh"

namespace tn::k {
namespace {

constexpr int kB = 128;          // query rows per CTA
constexpr int kN = 64;           // keys per KV block
constexpr int kHd = 128;         // head dim of the fused path
constexpr int kThreads = 192;

// 2^x for a pair on the FMA pipe (packed FFMA2/FADD2): x = j + f with
// j = round(x), degree-3 minimax polynomial for 2^f on [-0.5, 0.5] (max rel.
// error 7.6e-5, far below the bf16 rounding P gets), j added into the
// exponent bits. x < -126 clamps to 2^-126 * 2^f (a denormal: a masked key
// contributes < 1.7e-38); -127 would let 2^f < 1 borrow into the sign bit.
__device__ __forceinline__ void ex2_poly2(float& a, float& b) {
    a = fmaxf(a, -126.0f);
    b = fmaxf(b, -126.0f);
    float ta = a, tb = b;
    add2(ta, tb, 12582912.0f, 12582912.0f);  // 1.5 * 2^23: low mantissa bits hold round(x)
    float ja = ta, jb = tb;
    add2(ja, jb, -12582912.0f, -12582912.0f);
    float fa = a, fb = b;
    add2(fa, fb, -ja, -jb);
    float pa = 0.05517027f, pb = 0.05517027f;
    fma2v(pa, pb, fa, fb, 0.24260795f);
    fma2v(pa, pb, fa, fb, 0.6932609f);
    fma2v(pa, pb, fa, fb, 0.9999283f);
    a = __int_as_float(__float_as_int(pa) + (__float_as_int(ta) << 23));
    b = __int_as_float(__float_as_int(pb) + (__float_as_int(tb) << 23));
}
// smem (bytes): Q 128x128 (2 atoms of 16 KB), K 2 stages x 64x128 (2 atoms of
// 8 KB each), V 2 stages x 128(hd)x64(keys) (1 atom, 16 KB): 96 KB, so two
// CTAs share an SM and interleave their MMA and softmax phases (the softmax
// of one hides the MMAs / loads of the other). P never touches shared
// memory: the softmax warps write it as packed bf16 into TMEM and the P·V
// MMA reads its A operand from there.
// TMEM (256 columns per CTA): S [0, 64), P [64, 96), O [128, 256).
// Two CTAs fit without alignment slack: the dynamic window starts on a 1 KB
// boundary (the per-CTA system reservation precedes it), checked below.
constexpr int kQ = 32768, kKst = 16384, kV = 16384;

struct AttnParams {
    __nv_bfloat16* O;
    float* lse;  // optional [heads][seq]: (m + log2 l) * ln 2 of each row
    int heads, seq, nblk;
    std::int64_t ldo;
    float scale_log2;
    int causal;
    long long* dbg;  // TN_ATTN_DBG timeline (pair kernel: cluster 0, its first item), else nullptr
};

// EMU of every 4 column pairs take 2^x on the FMA pipe (ex2_poly2), the rest
// on MUFU.EX2: MUFU does 16 ex2/clk/SM, the same rate the two MMAs consume
// scores at hd 128, so a quarter on the FMA pipe relieves it (measured:
// EMU=1 131.9 us, 0 134.5, 2 133.3, 3 143.0 per 7B layer). Splitting each row
// over two softmax threads (8 softmax warps) was measured slower (138-141 us).
template <int EMU>
__global__ void __launch_bounds__(kThreads, 2)
    attention_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                     const __grid_constant__ CUtensorMap tv, const AttnParams p) {
    constexpr int CW = kN;  // score columns per softmax thread
    extern __shared__ std::uint8_t smem_raw[];
    const std::uint32_t raw = smem_u32(smem_raw);
    if (raw & 1023u) __trap();  // SW128 tiles need 1 KB alignment
    const std::uint32_t base = raw;
    const std::uint32_t sQ = base, sK0 = base + kQ, sV = sK0 + 2 * kKst;
    std::uint8_t* gen_base = smem_raw + (base - raw);
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(gen_base + kQ + 2 * kKst + 2 * kV);
    const std::uint32_t b0 = smem_u32(bars);
    const std::uint32_t q_full = b0, k_full = b0 + 8, k_empty = b0 + 24, v_full = b0 + 40, v_empty = b0 + 56,
                        s_full = b0 + 72, p_full = b0 + 88, o_done = b0 + 96;  // s_full[2]
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 13);

    pdl_trigger();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int h = blockIdx.x % p.heads;
    const int qb = p.nblk - 1 - static_cast<int>(blockIdx.x / p.heads);  // heavy blocks first
    const int nkv = p.causal ? (qb + 1) * (kB / kN) : p.nblk * (kB / kN);

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tq)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tk)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tv)) : "memory");
        mbar_init(q_full, 1);
        mbar_init(k_full, 1);
        mbar_init(k_full + 8, 1);
        mbar_init(k_empty, 1);
        mbar_init(k_empty + 8, 1);
        mbar_init(v_full, 1);
        mbar_init(v_full + 8, 1);
        mbar_init(v_empty, 1);
        mbar_init(v_empty + 8, 1);
        mbar_init(s_full, 1);
        mbar_init(s_full + 8, 1);
        mbar_init(p_full, 4);
        mbar_init(o_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) tmem_alloc(smem_u32(tmem_slot), 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();  // the previous kernel's outputs (q, k, vT) are complete and visible
    const std::uint32_t tmem = *tmem_slot;
    // S double-buffered: S_j in columns [64*(j%2), +64), and P_j (bf16, 32
    // columns) written over S_j once the softmax has it in registers. S_{j+1}
    // is computed while the softmax works on S_j; S_{j+2} reuses buffer j%2
    // after P_j·V (MMAs of one issuer execute in order).
    const std::uint32_t tS = tmem, tO = tmem + 128;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(q_full, kQ);
            tma_load_3d(sQ, &tq, 0, qb * kB, h, q_full);
            tma_load_3d(sQ + kQ / 2, &tq, 64, qb * kB, h, q_full);
            for (int j = 0; j < nkv; ++j) {
                const int st = j & 1;
                mbar_wait(k_empty + 8 * st, ((j >> 1) & 1) ^ 1);
                mbar_expect_tx(k_full + 8 * st, kKst);
                const std::uint32_t dk = sK0 + st * kKst;
                tma_load_3d(dk, &tk, 0, j * kN, h, k_full + 8 * st);
                tma_load_3d(dk + kKst / 2, &tk, 64, j * kN, h, k_full + 8 * st);
                mbar_wait(v_empty + 8 * st, ((j >> 1) & 1) ^ 1);
                mbar_expect_tx(v_full + 8 * st, kV);
                tma_load_3d(sV + st * kV, &tv, j * kN, 0, h, v_full + 8 * st);
            }
        }
    } else if (warp == 1) {
        {  // whole warp: one elected lane issues (tc_mma)
            const std::uint32_t idesc_s = make_idesc(1u, kB, kN);
            const std::uint32_t idesc_o = make_idesc(1u, kB, kHd);
            auto issue_s = [&](int j) {  // K stage and S buffer are both j % 2
                const int st = j & 1;
                mbar_wait(k_full + 8 * st, (j >> 1) & 1);
                tc_fence_after();
                const std::uint32_t dk = sK0 + st * kKst;
#pragma unroll
                for (int kk = 0; kk < kHd / 16; ++kk)
                    tc_mma(tS + 64 * st, sdesc(sQ + (kk >> 2) * (kQ / 2) + (kk & 3) * 32),
                           sdesc(dk + (kk >> 2) * (kKst / 2) + (kk & 3) * 32), idesc_s, kk != 0, false);
                tc_commit(s_full + 8 * st);
                tc_commit(k_empty + 8 * st);
            };
            mbar_wait(q_full, 0);
            issue_s(0);
            if (nkv > 1) issue_s(1);
            for (int j = 0; j < nkv; ++j) {
                mbar_wait(p_full, j & 1);
                mbar_wait(v_full + 8 * (j & 1), (j >> 1) & 1);
                tc_fence_after();
                const std::uint32_t dv = sV + (j & 1) * kV;
                const std::uint32_t tPj = tS + 64 * (j & 1);
#pragma unroll
                for (int kk = 0; kk < kN / 16; ++kk)
                    tc_mma_ts(tO, tPj + kk * 8, sdesc(dv + kk * 32), idesc_o, (j | kk) != 0);
                tc_commit(o_done);
                tc_commit(v_empty + 8 * (j & 1));
                if (j + 2 < nkv) issue_s(j + 2);  // into buffer j%2, after P_j·V
            }
        }
    } else {
        const int lane_base = (warp % 4) * 32;
        const int r = lane_base + lane;  // query row within the block
        const int qrow = qb * kB + r;
        const std::uint32_t trow = static_cast<std::uint32_t>(lane_base) << 16;
        float m = -INFINITY, l = 0.f;
        constexpr int kW = 8;
        for (int j = 0; j < nkv; ++j) {
            const std::uint32_t tSj = tS + 64 * (j & 1);
            mbar_wait(s_full + 8 * (j & 1), (j >> 1) & 1);
            tc_fence_after();
            float s[CW];
#pragma unroll
            for (int c = 0; c < CW; c += 32) {
                std::uint32_t u[32];
                TN_LD32(tSj + trow + c, u);
#pragma unroll
                for (int i = 0; i < 32; ++i) s[c + i] = __uint_as_float(u[i]);
            }
            tc_wait_ld();

            // masked keys: key index j*kN + c > query row (causal)
            const int lim = p.causal ? qrow - j * kN : CW;  // columns c <= lim are valid
            float pm[kW];
#pragma unroll
            for (int w = 0; w < kW; ++w) pm[w] = -INFINITY;
            if (lim < CW - 1) {
#pragma unroll
                for (int c = 0; c < CW; ++c) {
                    if (c > lim) s[c] = -INFINITY;
                    pm[c % kW] = fmaxf(pm[c % kW], s[c]);
                }
            } else {
#pragma unroll
                for (int c = 0; c < CW; ++c) pm[c % kW] = fmaxf(pm[c % kW], s[c]);
            }
#pragma unroll
            for (int w = kW / 2; w > 0; w /= 2)
#pragma unroll
                for (int i = 0; i < w; ++i) pm[i] = fmaxf(pm[i], pm[i + w]);
            // Lazy rescale: the running max only moves (and O is only
            // rescaled) when the block max exceeds it by more than 2^8, so
            // P <= 256 stays well inside bf16/fp32 range and most blocks skip
            // the TMEM read-modify-write of O. Final O / l is unchanged.
            const float cand = fmaxf(m, pm[0] * p.scale_log2);  // a fully masked block keeps m
            const bool grew = cand > m + 8.0f;
            const float mx = grew ? cand : m;
            const float corr = ex2(m - mx);
            float ps[kW];
#pragma unroll
            for (int w = 0; w < kW; ++w) ps[w] = 0.f;
            // x = s*scale - mx, 2^x, per-column-class partial sums: packed
            // FFMA2/FADD2 (bitwise the same as the scalar fmaf / += chain)
#pragma unroll
            for (int c = 0; c < CW; c += 2) {
                fma2(s[c], s[c + 1], p.scale_log2, -mx);
                if ((c % 8) < 2 * EMU) {
                    ex2_poly2(s[c], s[c + 1]);
                } else {
                    s[c] = ex2(s[c]);
                    s[c + 1] = ex2(s[c + 1]);
                }
                add2(ps[c % kW], ps[c % kW + 1], s[c], s[c + 1]);
            }
#pragma unroll
            for (int w = kW / 2; w > 0; w /= 2)
#pragma unroll
                for (int i = 0; i < w; ++i) ps[i] += ps[i + w];
            l = l * corr + ps[0];
            m = mx;

            if (j > 0) {
                mbar_wait(o_done, (j - 1) & 1);  // P_{j-1}·V done: O stable, P tile free
                tc_fence_after();
                if (__any_sync(0xffffffffu, grew)) {
#pragma unroll 1
                    for (int c = 0; c < kHd; c += 32) {
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
            {
                std::uint32_t pw[CW / 2];
#pragma unroll
                for (int i = 0; i < CW / 2; ++i) {
                    __nv_bfloat162 v2 = __floats2bfloat162_rn(s[2 * i], s[2 * i + 1]);
                    pw[i] = *reinterpret_cast<std::uint32_t*>(&v2);
                }
                TN_ST32(tSj + trow, pw);  // P_j over S_j (already in registers)
                tc_wait_st();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_full);
        }
        // Epilogue: O / l -> bf16 rows of the [seq, heads*hd] output.
        mbar_wait(o_done, (nkv - 1) & 1);
        tc_fence_after();
        const float inv = 1.0f / l;
        if (p.lse) p.lse[static_cast<std::int64_t>(h) * p.seq + qrow] = (m + __log2f(l)) * 0.6931471805599453f;
        __nv_bfloat16* orow = p.O + static_cast<std::int64_t>(qrow) * p.ldo + static_cast<std::int64_t>(h) * kHd;
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

constexpr int kSmem = kQ + 2 * kKst + 2 * kV + 128;

// ---------------------------------------------------------------------------
// CTA-pair kernel (cta_group::2, a cluster of two CTAs on one TPC), the fast
// path for seq % 256 == 0. A work item is 512 consecutive query rows of one
// head, as TWO Q tiles of 256 rows (each tile = M 256 MMAs issued by the
// leader; a CTA holds 128 rows of each tile), walking 128-key blocks.
// Persistent: one cluster per TPC walks its items (heaviest first, snake
// order over the clusters for balance); the next item's Q load and first
// S MMAs overlap the current item's last blocks and O epilogue.
// Each CTA stages HALF of every K block (64 keys) and HALF of every Vᵀ block
// (64 of the 128 head-dim rows), so per 128x128 score tile an SM moves 80 KB
// through shared memory (vs 192 KB in the 1-CTA kernel) and the tensor pipe,
// not shared-memory bandwidth, bounds the MMAs.
// TMEM (512 columns per CTA): S0/P0 [0,128), S1/P1 [128,256), O0 [256,384),
// O1 [384,512). smem: Q0, Q1 (32 KB each), 3 stages of K and Vᵀ halves.
//   warp 0     TMA (both CTAs; .cta_group::2 loads signal the leader's barriers)
//   warp 1     leader only, one in-order issuer: per item S0_0, S1_0, then per
//              block j P0_j·V_j, S0_{j+1}, P1_j·V_j, S1_{j+1}. The single
//              issuer staggers the two tiles: tile 0's softmax runs while the
//              pipe executes tile 1's MMAs and vice versa. Each P·V is issued
//              in two halves (keys [0,64) as soon as the softmax stored them).
//              In-order execution makes S_t,j+1 overwrite P_t,j only after
//              P_t,j·V read it, and S_t,j+1 complete implies P_t,j·V complete
//              (O_t stable for the softmax warps' rare rescale). An item's
//              first P_t·V (which overwrites O_t) waits until the previous
//              item's epilogue has read O_t (o_empty).
//   warps 2-5  softmax of tile 0, warps 6-9 tile 1: one query row per thread,
//              128 scores in registers, P (bf16) over S in TMEM, final O / l.
// Causal: tile t of item i covers rows [512i + 256t, +256) and walks blocks
// 0..4i+2t+1; in the diagonal blocks the rows above the key range are masked.
// Measured alternatives (7B layer, causal): one pair per item without the
// overlap 138-140 us (1-CTA kernel 132.5); two softmax threads per row with a
// shared-memory max exchange (16 softmax warps, setmaxnreg) 154.8 us.
constexpr int kN2 = 128;                  // keys per block
constexpr int kKh = 64 * kHd * 2;         // per CTA per stage: 64 keys x hd 128 = 16 KB (2 SW128 atoms of 8 KB)
constexpr int kVh = (kHd / 2) * kN2 * 2;  // per CTA per stage: 64 Vᵀ rows x 128 keys = 16 KB (2 atoms)
constexpr int kStg2 = 3;
constexpr int kThreads2 = 320;
constexpr int kSmem2 = 2 * kQ + kStg2 * (kKh + kVh) + 256;

struct PairItem {
    int h, qi, nkv_t[2], nkv;
};
// Item `n` of cluster `c` (snake order: even rounds ascend, odd rounds
// descend over the clusters); items are numbered heaviest first.
__device__ __forceinline__ bool pair_item(const AttnParams& p, int c, int nc, int n, PairItem& it) {
    const int idx = n * nc + ((n & 1) ? nc - 1 - c : c);
    if (idx >= p.heads * p.nblk) return false;
    it.h = idx % p.heads;
    it.qi = p.nblk - 1 - idx / p.heads;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int row0 = it.qi * 512 + t * 256;
        it.nkv_t[t] = row0 >= p.seq ? 0 : p.causal ? (row0 + 256) / kN2 : p.seq / kN2;
    }
    it.nkv = max(it.nkv_t[0], it.nkv_t[1]);
    return true;
}

// Four K=16 pair MMAs from one elected lane: D (+)= A_k·B_k for k = 0..3,
// the smem descriptors advanced by 32 bytes (2 units) per k; A from smem (SS)
// or from TMEM (TS: 8 columns of packed bf16 per k). One elect per group
// instead of one per MMA: the issuer warp shares its sub-partition with two
// softmax warps, and the per-MMA elect / vote / uniform-register setup (~12
// issue slots each, ~470 per block) made those two the last to hand P over,
// ~400 clk after the others (TN_ATTN_DBG, profiles/r2d_attention_timeline.md).
__device__ __forceinline__ void mma4_ss_2sm(std::uint32_t d, std::uint64_t a, std::uint64_t b, std::uint32_t idesc,
                                            std::uint32_t acc0) {
    asm volatile(
        "{\n\t.reg .pred p, t, e;\n\t.reg .b32 r;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
        "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 t, %4, %4;\n\t"
        "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
        "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
        "elect.sync r|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %3, t;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %3, t;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %3, t;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc0)
        : "memory");
}
__device__ __forceinline__ void mma4_ts_2sm(std::uint32_t d, std::uint32_t a, std::uint64_t b, std::uint32_t idesc,
                                            std::uint32_t acc0) {
    asm volatile(
        "{\n\t.reg .pred p, t, e;\n\t.reg .b32 r, a1, a2, a3;\n\t.reg .b64 b1, b2, b3;\n\t"
        "setp.ne.b32 p, %4, 0;\n\tsetp.eq.b32 t, %4, %4;\n\t"
        "add.s32 a1, %1, 8;\n\tadd.s32 a2, %1, 16;\n\tadd.s32 a3, %1, 24;\n\t"
        "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
        "elect.sync r|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a1], b1, %3, t;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a2], b2, %3, t;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [a3], b3, %3, t;\n\t}" ::"r"(d),
        "r"(a), "l"(b), "r"(idesc), "r"(acc0)
        : "memory");
}

template <int EMU>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads2, 1)
    attention_kernel_2sm(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                         const __grid_constant__ CUtensorMap tv, const AttnParams p) {
    constexpr int CW = kN2;
    extern __shared__ std::uint8_t smem_raw[];
    const std::uint32_t base = smem_u32(smem_raw);
    if (base & 1023u) __trap();
    const std::uint32_t sQ = base, sK0 = base + 2 * kQ, sV0 = sK0 + kStg2 * kKh;
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem_raw + 2 * kQ + kStg2 * (kKh + kVh));
    const std::uint32_t b0 = smem_u32(bars);
    // q_full | k_full[3] | k_empty[3] | v_full[3] | v_empty[3] | s_full[2] | p_full[2][2] | o_full[2]
    // | o_empty[2] | q_empty
    const std::uint32_t q_full = b0, k_full = b0 + 8, k_empty = b0 + 32, v_full = b0 + 56, v_empty = b0 + 80,
                        s_full = b0 + 104, p_full = b0 + 120, o_full = b0 + 152, o_empty = b0 + 168,
                        q_empty = b0 + 184;
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 24);

    pdl_trigger();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const std::uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int cl = blockIdx.x / 2, ncl = gridDim.x / 2;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tq)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tk)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tv)) : "memory");
        for (int i = 0; i < 15; ++i) mbar_init(b0 + 8 * i, 1);  // q, k/v full/empty, s_full[2]
        for (int i = 0; i < 4; ++i) mbar_init(p_full + 8 * i, 8);  // 4 softmax warps x 2 CTAs
        mbar_init(o_full, 1);
        mbar_init(o_full + 8, 1);
        mbar_init(o_empty, 8);
        mbar_init(o_empty + 8, 8);
        mbar_init(q_empty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    pdl_wait();
    const std::uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int st = 0;
            std::uint32_t ph = 0;
            PairItem it;
            for (int n = 0; pair_item(p, cl, ncl, n, it); ++n) {
                const int ntiles = it.nkv_t[1] > 0 ? 2 : 1;
                if (n > 0) mbar_wait(q_empty, (n - 1) & 1);  // the previous item's S MMAs have read Q
                if (leader) mbar_expect_tx(q_full, 2 * kQ * ntiles);
                const std::uint32_t qf = mapa(q_full, 0);
                for (int t = 0; t < ntiles; ++t) {
                    const int qrow0 = it.qi * 512 + t * 256 + static_cast<int>(rank) * kB;
                    tma_load_3d_2sm(sQ + t * kQ, &tq, 0, qrow0, it.h, qf);
                    tma_load_3d_2sm(sQ + t * kQ + kQ / 2, &tq, 64, qrow0, it.h, qf);
                }
                for (int j = 0; j < it.nkv; ++j) {
                    mbar_wait(k_empty + 8 * st, ph ^ 1);
                    if (leader) mbar_expect_tx(k_full + 8 * st, 2 * kKh);
                    const std::uint32_t kf = mapa(k_full + 8 * st, 0), dk = sK0 + st * kKh;
                    const int key0 = j * kN2 + static_cast<int>(rank) * 64;
                    tma_load_3d_2sm(dk, &tk, 0, key0, it.h, kf);
                    tma_load_3d_2sm(dk + kKh / 2, &tk, 64, key0, it.h, kf);
                    mbar_wait(v_empty + 8 * st, ph ^ 1);
                    if (leader) mbar_expect_tx(v_full + 8 * st, 2 * kVh);
                    const std::uint32_t vf = mapa(v_full + 8 * st, 0), dv = sV0 + st * kVh;
                    const int vrow = static_cast<int>(rank) * (kHd / 2);
                    tma_load_3d_2sm(dv, &tv, j * kN2, vrow, it.h, vf);
                    tma_load_3d_2sm(dv + kVh / 2, &tv, j * kN2 + 64, vrow, it.h, vf);
                    if (++st == kStg2) {
                        st = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {  // whole warp: one elected lane issues
            const std::uint32_t idesc_s = make_idesc(1u, 2 * kB, kN2);
            const std::uint32_t idesc_o = make_idesc(1u, 2 * kB, kHd);
            auto issue_s = [&](int t, int st) {
                const std::uint64_t qa = sdesc(sQ + t * kQ), kb = sdesc(sK0 + st * kKh);
                mma4_ss_2sm(tmem + t * 128, qa, kb, idesc_s, 0);  // head dims [0, 64)
                mma4_ss_2sm(tmem + t * 128, qa + (kQ / 2 >> 4), kb + (kKh / 2 >> 4), idesc_s, 1);  // [64, 128)
                tc_commit_2sm(s_full + 8 * t);
            };
            int st = 0;
            std::uint32_t ph = 0;
            int bt[2] = {0, 0}, itc[2] = {0, 0};  // per tile: blocks and items processed before this item
            PairItem it;
            for (int n = 0; pair_item(p, cl, ncl, n, it); ++n) {
                mbar_wait(q_full, n & 1);
                mbar_wait(k_full + 8 * st, ph);
                tc_fence_after();
                issue_s(0, st);
                if (it.nkv_t[1] > 0) issue_s(1, st);
                tc_commit_2sm(k_empty + 8 * st);
                if (it.nkv == 1) tc_commit_2sm(q_empty);
                for (int j = 0; j < it.nkv; ++j) {
                    const int st1 = st + 1 == kStg2 ? 0 : st + 1;
                    const std::uint32_t ph1 = st1 == 0 ? ph ^ 1 : ph;
                    const bool knext = j + 1 < it.nkv;
                    bool kwaited = false;
                    mbar_wait(v_full + 8 * st, ph);
                    const std::uint32_t dv = sV0 + st * kVh;
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        if (j >= it.nkv_t[t]) continue;
                        const std::uint32_t tS = tmem + t * 128, tO = tmem + 256 + t * 128;
                        if (j == 0 && itc[t] > 0) mbar_wait(o_empty + 8 * t, (itc[t] - 1) & 1);
                        const std::uint32_t pph = static_cast<std::uint32_t>(bt[t] + j) & 1;
                        const bool dbgi = p.dbg && cl == 0 && n == 0 && j < 64;
                        if (dbgi) p.dbg[(t * 64 + j) * 4 + 0] = clock64();
                        mbar_wait(p_full + 16 * t, pph);
                        if (dbgi) p.dbg[(t * 64 + j) * 4 + 1] = clock64();
                        tc_fence_after();
                        const std::uint64_t vb = sdesc(dv);
                        mma4_ts_2sm(tO, tS, vb, idesc_o, j != 0);  // keys [0, 64)
                        mbar_wait(p_full + 16 * t + 8, pph);
                        if (dbgi) {
                            p.dbg[(t * 64 + j) * 4 + 2] = clock64();
                            long long gt;
                            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
                            p.dbg[(t * 64 + j) * 4 + 3] = gt;
                        }
                        tc_fence_after();
                        mma4_ts_2sm(tO, tS + 32, vb + (kVh / 2 >> 4), idesc_o, 1);  // keys [64, 128)
                        if (j + 1 == it.nkv_t[t]) tc_commit_2sm(o_full + 8 * t);
                        if (j + 1 < it.nkv_t[t]) {
                            if (!kwaited) {
                                mbar_wait(k_full + 8 * st1, ph1);
                                tc_fence_after();
                                kwaited = true;
                            }
                            issue_s(t, st1);
                        }
                    }
                    tc_commit_2sm(v_empty + 8 * st);
                    if (knext) tc_commit_2sm(k_empty + 8 * st1);
                    if (j + 2 == it.nkv) tc_commit_2sm(q_empty);  // the item's last S MMAs were just issued
                    st = st1;
                    ph = ph1;
                }
#pragma unroll
                for (int t = 0; t < 2; ++t)
                    if (it.nkv_t[t] > 0) {
                        bt[t] += it.nkv_t[t];
                        itc[t]++;
                    }
            }
        }
    } else {
        const int t = (warp - 2) / 4;
        const int lane_base = (warp % 4) * 32;
        const int r = lane_base + lane;
        const std::uint32_t trow = static_cast<std::uint32_t>(lane_base) << 16;
        const std::uint32_t tS = tmem + t * 128 + trow, tO = tmem + 256 + t * 128 + trow;
        const std::uint32_t pf0 = mapa(p_full + 16 * t, 0), pf1 = pf0 + 8;
        const std::uint32_t oe = mapa(o_empty + 8 * t, 0);
        const std::uint32_t sf = s_full + 8 * t;
        int bt = 0, itc = 0;
        PairItem it;
        for (int n = 0; pair_item(p, cl, ncl, n, it); ++n) {
            const int nk = t == 0 ? it.nkv_t[0] : it.nkv_t[1];
            if (nk == 0) continue;
            const int qrow = it.qi * 512 + t * 256 + static_cast<int>(rank) * kB + r;
            float m = -INFINITY, l = 0.f;
            constexpr int kW = 8;
            for (int j = 0; j < nk; ++j) {
                const bool dbgs = p.dbg && cl == 0 && n == 0 && j < 64 && rank == 0 && (warp == 2 || warp == 6) && lane == 0;
                long long* dp = dbgs ? p.dbg + 512 + (t * 64 + j) * 8 : nullptr;
                if (dbgs) dp[0] = clock64();
                mbar_wait(sf, (bt + j) & 1);
                if (dbgs) dp[1] = clock64();
                tc_fence_after();
                float s[CW];
#pragma unroll
                for (int c = 0; c < CW; c += 32) {
                    std::uint32_t u[32];
                    TN_LD32(tS + c, u);
#pragma unroll
                    for (int i = 0; i < 32; ++i) s[c + i] = __uint_as_float(u[i]);
                }
                tc_wait_ld();
                if (dbgs) dp[2] = clock64();
                const int lim = p.causal ? qrow - j * kN2 : CW;  // columns c <= lim are valid
                float pm[kW];
#pragma unroll
                for (int w = 0; w < kW; ++w) pm[w] = -INFINITY;
                if (lim < CW - 1) {
#pragma unroll
                    for (int c = 0; c < CW; ++c)
                        if (c > lim) s[c] = -INFINITY;
                }
#pragma unroll
                for (int c = 0; c < CW; c += 2) pm[(c / 2) % kW] = fmax3(pm[(c / 2) % kW], s[c], s[c + 1]);
#pragma unroll
                for (int w = kW / 2; w > 0; w /= 2)
#pragma unroll
                    for (int i = 0; i < w; ++i) pm[i] = fmaxf(pm[i], pm[i + w]);
                const float cand = fmaxf(m, pm[0] * p.scale_log2);  // a fully masked block keeps m
                const bool grew = cand > m + 8.0f;
                const float mx = grew ? cand : m;
                const float corr = ex2(m - mx);
                if (dbgs) dp[3] = clock64();
                float ps[kW];
#pragma unroll
                for (int w = 0; w < kW; ++w) ps[w] = 0.f;
#pragma unroll
                for (int c0 = 0; c0 < CW; c0 += 32) {
                    std::uint32_t pw[16];
#pragma unroll
                    for (int c = c0; c < c0 + 32; c += 2) {
                        fma2(s[c], s[c + 1], p.scale_log2, -mx);
                        if ((c % 8) < 2 * EMU) {
                            ex2_poly2(s[c], s[c + 1]);
                        } else {
                            s[c] = ex2(s[c]);
                            s[c + 1] = ex2(s[c + 1]);
                        }
                        add2(ps[c % kW], ps[c % kW + 1], s[c], s[c + 1]);
                        __nv_bfloat162 v2 = __floats2bfloat162_rn(s[c], s[c + 1]);
                        pw[(c - c0) / 2] = *reinterpret_cast<std::uint32_t*>(&v2);
                    }
                    TN_ST16(tS + c0 / 2, pw);  // P (bf16 pairs) over S
                    if (c0 == 32) {
                        // S_t,j complete => P_t,j-1·V complete: O_t is stable for the
                        // rare rescale, which must precede the first P_t,j·V MMA.
                        if (j > 0 && __any_sync(0xffffffffu, grew)) {
#pragma unroll 1
                            for (int c = 0; c < kHd; c += 32) {
                                std::uint32_t u[32];
                                TN_LD32(tO + c, u);
                                tc_wait_ld();
#pragma unroll
                                for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(__uint_as_float(u[i]) * corr);
                                TN_ST32(tO + c, u);
                            }
                        }
                        tc_wait_st();
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_remote(pf0);
                        if (dbgs) dp[4] = clock64();
                    }
                }
                tc_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(pf1);
                if (dbgs) dp[5] = clock64();
                if (p.dbg && cl == 0 && n == 0 && j < 64 && lane == 0) {  // every softmax warp: P_B hand-off
                    long long gt;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
                    const int w = (warp - 2) % 4, slot = (t * 64 + j) * 8 + static_cast<int>(rank) * 4 + w;
                    p.dbg[1536 + slot] = gt;                      // ns, comparable across the pair
                    if (rank == 0) p.dbg[2560 + (t * 64 + j) * 4 + w] = clock64();  // leader SM clock
                }
#pragma unroll
                for (int w = kW / 2; w > 0; w /= 2)
#pragma unroll
                    for (int i = 0; i < w; ++i) ps[i] += ps[i + w];
                l = l * corr + ps[0];
                m = mx;
            }
            bt += nk;
            mbar_wait(o_full + 8 * t, itc & 1);
            tc_fence_after();
            const float inv = 1.0f / l;
            if (p.lse) p.lse[static_cast<std::int64_t>(it.h) * p.seq + qrow] = (m + __log2f(l)) * 0.6931471805599453f;
            __nv_bfloat16* orow =
                p.O + static_cast<std::int64_t>(qrow) * p.ldo + static_cast<std::int64_t>(it.h) * kHd;
#pragma unroll 1
            for (int c = 0; c < kHd; c += 32) {
                std::uint32_t u[32];
                TN_LD32(tO + c, u);
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
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(oe);  // O_t read: the next item may overwrite it
            itc++;
        }
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512) : "memory");
}

// --- SIMT fallback (any seq / head dim): one warp per query row, fp32 online
// softmax over all keys in order. Slow; only for shapes the fused path rejects.
__global__ void attention_simt(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                               const __nv_bfloat16* __restrict__ vt, __nv_bfloat16* __restrict__ O, int heads, int seq,
                               int hd, std::int64_t ldo, float scale_log2, int causal, float* lse) {
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
    if (lse && lane == 0) lse[static_cast<std::int64_t>(h) * seq + i] = (m + log2f(l)) * 0.6931471805599453f;
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
                           kN) &&
             encode_tma_3d(&plan->tv, a.vt, 2, a.seq, a.hd, a.seq, a.heads, static_cast<std::int64_t>(a.seq) * a.hd, 64,
                           kHd);
    plan->path = ok ? 0 : 1;
    // CTA-pair kernel (persistent; 512-row items of two 256-row tiles; Vᵀ boxes
    // of 64 head-dim rows) whenever seq % 256 == 0: measured on the 7B layer
    // (32 heads, seq 4096) at 128.4-128.9 vs 133.2 us causal and 236.9 vs
    // 252.8 us non-causal against the 1-CTA kernel. TN_ATTN_PAIR=0 /
    // TN_ATTN_1CTA=1 force the 1-CTA kernel (A/B).
    static const char* pair_env = std::getenv("TN_ATTN_PAIR");
    static const bool force_1cta = std::getenv("TN_ATTN_1CTA") != nullptr;
    const bool want_pair = pair_env ? std::atoi(pair_env) != 0 : true;
    if (ok && a.seq % 256 == 0 && want_pair && !force_1cta)
        if (encode_tma_3d(&plan->tv2, a.vt, 2, a.seq, a.hd, a.seq, a.heads, static_cast<std::int64_t>(a.seq) * a.hd, 64,
                          kHd / 2))
            plan->path = 2;
    if (plan->path == 2) {  // persistent: one cluster (CTA pair) per TPC, at most one per item
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        plan->grid = 2 * std::min(a.heads * ((a.seq + 511) / 512), std::max(1, sms / 2));
    }
    if (ok) {
        static std::atomic<unsigned long long> attr_set{0};  // per CUDA device, any thread
        int dev = 0;
        cudaGetDevice(&dev);
        if (!((attr_set.load(std::memory_order_acquire) >> dev) & 1ULL)) {
            cudaFuncSetAttribute(attention_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
            cudaFuncSetAttribute(attention_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
            cudaFuncSetAttribute(attention_kernel_2sm<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2);
            cudaFuncSetAttribute(attention_kernel_2sm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2);
            attr_set.fetch_or(1ULL << dev, std::memory_order_release);
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
            sl2, a.causal, a.lse);
        return cudaGetLastError();
    }
    AttnParams p;
    p.O = static_cast<__nv_bfloat16*>(a.out);
    p.lse = a.lse;
    p.heads = a.heads;
    p.seq = a.seq;
    p.nblk = a.seq / kB;
    p.ldo = a.ldo;
    p.scale_log2 = sl2;
    p.causal = a.causal;
    p.dbg = nullptr;
    // TN_ATTN_DBG=<file>: per-block clock64 timeline of the pair kernel (cluster 0,
    // first item) appended to <file>; synchronises after the launch (diagnostics
    // only; tools/attn_timeline.py reads it)
    static const char* dbg_env = std::getenv("TN_ATTN_DBG");
    static long long* dbg_buf = nullptr;
    if (dbg_env && plan.path == 2) {
        if (!dbg_buf) cudaMalloc(&dbg_buf, 4096 * sizeof(long long));
        cudaMemsetAsync(dbg_buf, 0, 4096 * sizeof(long long), s);
        p.dbg = dbg_buf;
    }
    static const char* emu_env = std::getenv("TN_ATTN_EMU");  // A/B: "0" keeps every 2^x on MUFU
    const bool emu0 = emu_env && std::atoi(emu_env) == 0;
    if (plan.path == 2) {
        p.nblk = (a.seq + 511) / 512;
        const unsigned grid2 = static_cast<unsigned>(plan.grid);
        cudaError_t e = emu0 ? launch_pdl(attention_kernel_2sm<0>, dim3(grid2), dim3(kThreads2), kSmem2, s, plan.tq,
                                          plan.tk, plan.tv2, p)
                             : launch_pdl(attention_kernel_2sm<1>, dim3(grid2), dim3(kThreads2), kSmem2, s, plan.tq,
                                          plan.tk, plan.tv2, p);
        if (p.dbg && e == cudaSuccess) {
            static long long host[4096];
            cudaMemcpyAsync(host, p.dbg, sizeof(host), cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            if (FILE* f = std::fopen(dbg_env, "a")) {
                for (int i = 0; i < 4096; ++i) std::fprintf(f, "%lld%c", host[i], i == 4095 ? '\n' : ' ');
                std::fclose(f);
            }
        }
        return e;
    }
    const unsigned grid = p.heads * p.nblk;
    if (emu0)
        return launch_pdl(attention_kernel<0>, dim3(grid), dim3(kThreads), kSmem, s, plan.tq, plan.tk, plan.tv, p);
    return launch_pdl(attention_kernel<1>, dim3(grid), dim3(kThreads), kSmem, s, plan.tq, plan.tk, plan.tv, p);
}

double attention_flops(const AttnArgs& a) {
    double f = 4.0 * a.heads * static_cast<double>(a.seq) * a.seq * a.hd;
    return a.causal ? f * 0.5 * (1.0 + 1.0 / a.seq) : f;
}

}  // namespace tn::k
