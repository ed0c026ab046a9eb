// Fused attention backward (the LoRA step's attention gradient, SURVEY §8a
// config 4): from q, k, v, the forward output O with its per-row logsumexp,
// and dO, computes dQ, dK, dV without materialising the n² score /
// probability tiles — the backward counterpart of attention.cu, replacing the
// scores -> softmax -> dP -> softmax_bwd -> dQ/dK/dV GEMM chain (2 GB of fp32
// tiles per 7B layer at seq 4096).
//
//   P  = 2^(scale·log2e · Q Kᵀ − lse·log2e)        (recomputed, causal mask)
//   dP = dO Vᵀ,  dS = P ⊙ (dP − D),  D = rowsum(dO ⊙ O)     (D: attn_bwd_prep)
//   dV = Pᵀ dO,  dK = scale · dSᵀ Q,  dQ = scale · dS K
//
// One launch, two CTA roles (blockIdx even / odd); a CTA runs two items of
// its role and head, blocks b and nblk-1-b, so every CTA walks nblk+1 blocks
// (causal), and CTAs go head-major for L2 reuse:
//   role KV, per (head, 128-key block j): walks the query blocks i >= j with
//     Sᵀ = K_j Q_iᵀ and dPᵀ = V_j dO_iᵀ (M = keys), writes Pᵀ / dSᵀ (bf16) over
//     them in TMEM and accumulates dV += Pᵀ dO_i, dK += dSᵀ Q_i with the A
//     operand read from TMEM and B = the same Q_i / dO_i smem tiles read
//     MN-major (no transposed copies).
//   role Q, per (head, 128-query block i): walks the key blocks j <= i with
//     S = Q_i K_jᵀ, dP = dO_i V_jᵀ and accumulates dQ += dS K_j (dS from TMEM,
//     K_j read MN-major).
// dQ is computed by its own role instead of fp32 atomics, so the kernel is
// deterministic (fixed block order, per-row reductions) like the forward.
//
//   warp 0     TMA: the CTA's fixed tiles once, then a 2-stage ring of the
//              walked tiles (+ the 128 lse / D values of a query block)
//   warp 1     MMA issue (one elected lane)
//   warps 2-9  P, dS, epilogue: one TMEM lane (row) and 64 of its columns per thread
// TMEM (512 columns): S / P [0,128), dP / dS [128,256), dV or dQ [256,384),
// dK [384,512). smem: 2 fixed 32 KB tiles + 1 KB, 2 stages of 65 KB.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "kernels.hpp"
#include "tc_common.cuh"

namespace tn::k {
namespace {

constexpr int kT = 128;                   // rows per tile (keys or queries)
constexpr int kHdB = 128;                 // head dim
constexpr int kTile = kT * kHdB * 2;      // 32 KB: two SW128 atoms of [128 rows x 64]
constexpr int kAtomB = kTile / 2;         // 16 KB
constexpr int kVec = kT * 4;              // 512 B: the lse or D values of one query block
constexpr int kStage = 2 * kTile + 2 * kVec;  // 65 KB (a multiple of 1 KB)
constexpr int kThreadsB = 320;
constexpr int kSmemB = 3 * kStage + 256;  // fixed (2 tiles + vecs) + 2 stages + barriers

struct BwdParams {
    __nv_bfloat16 *dq, *dk, *dv;
    std::int64_t ldg;  // row pitch (elements) of dq / dk / dv
    const float* lse;  // [heads][seq], natural log
    const float* D;    // [heads][seq]
    const float* rope; // optional [seq][hd/2][cos, sin]: dq, dk leave inverse-rotated (pre-RoPE gradients)
    int heads, seq, nblk, causal;
    float scale, scale_log2;
};

// MN-major SW128 operand of a [128 rows (K) x 128 (N or M)] tile stored as two
// 16 KB atoms of 64 columns: LBO = 16 KB between the atoms, SBO = 1 KB between
// 8-row groups; the K16 step is +2 KB (16 rows of 128 B).
__device__ __forceinline__ std::uint64_t sdesc_mn16(std::uint32_t saddr) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((saddr & 0x3FFFF) >> 4);
    d |= static_cast<std::uint64_t>(kAtomB >> 4) << 16;
    d |= static_cast<std::uint64_t>(1024 >> 4) << 32;
    d |= static_cast<std::uint64_t>(1) << 46;
    d |= static_cast<std::uint64_t>(2) << 61;
    return d;
}
// K-major address of K16 step kk of a [128 rows x hd 128] tile.
__device__ __forceinline__ std::uint32_t kmaj(std::uint32_t tile, int kk) {
    return tile + (kk >> 2) * kAtomB + (kk & 3) * 32;
}
__device__ __forceinline__ void bulk_load(std::uint32_t dst, const void* src, std::uint32_t bytes, std::uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(reinterpret_cast<std::uint64_t>(src)), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ std::uint32_t pack2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<std::uint32_t*>(&v);
}
__device__ __forceinline__ float2 unpack2(std::uint32_t u) {
    __nv_bfloat162 v = *reinterpret_cast<__nv_bfloat162*>(&u);
    return __bfloat1622float2(v);
}
// The pre-RoPE gradient of one row (rotate-half RoPE, rotation by -theta):
// pairs i in [i0, i0+32) of the 128-column accumulator at taddr (lane = row),
// a = col i, b = col 64+i: dst[i] = (a cos + b sin) * mul, dst[64+i] = (b cos - a sin) * mul.
__device__ __forceinline__ void store_row_rope(std::uint32_t taddr, __nv_bfloat16* dst, float mul,
                                               const float* tab_row, int i0) {
    std::uint32_t ua[32], ub[32];
    TN_LD32(taddr + i0, ua);
    TN_LD32(taddr + 64 + i0, ub);
    tc_wait_ld();
    const float4* cs = reinterpret_cast<const float4*>(tab_row + 2 * i0);  // (cos, sin) pairs
    std::uint32_t ya[16], yb[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        const float4 t = __ldg(cs + q);  // pairs i0+2q, i0+2q+1
        const float a0 = __uint_as_float(ua[2 * q]), a1 = __uint_as_float(ua[2 * q + 1]);
        const float b0 = __uint_as_float(ub[2 * q]), b1 = __uint_as_float(ub[2 * q + 1]);
        ya[q] = pack2((a0 * t.x + b0 * t.y) * mul, (a1 * t.z + b1 * t.w) * mul);
        yb[q] = pack2((b0 * t.x - a0 * t.y) * mul, (b1 * t.z - a1 * t.w) * mul);
    }
    uint4* da = reinterpret_cast<uint4*>(dst + i0);
    uint4* db = reinterpret_cast<uint4*>(dst + 64 + i0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        da[q] = make_uint4(ya[4 * q], ya[4 * q + 1], ya[4 * q + 2], ya[4 * q + 3]);
        db[q] = make_uint4(yb[4 * q], yb[4 * q + 1], yb[4 * q + 2], yb[4 * q + 3]);
    }
}
// 64 fp32 TMEM columns of this thread's lane -> bf16 at dst, times mul.
__device__ __forceinline__ void store_row(std::uint32_t taddr, __nv_bfloat16* dst, float mul) {
#pragma unroll 1
    for (int c = 0; c < 64; c += 32) {
        std::uint32_t u[32];
        TN_LD32(taddr + c, u);
        tc_wait_ld();
        uint4* d4 = reinterpret_cast<uint4*>(dst + c);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint4 v;
            v.x = pack2(__uint_as_float(u[q * 8 + 0]) * mul, __uint_as_float(u[q * 8 + 1]) * mul);
            v.y = pack2(__uint_as_float(u[q * 8 + 2]) * mul, __uint_as_float(u[q * 8 + 3]) * mul);
            v.z = pack2(__uint_as_float(u[q * 8 + 4]) * mul, __uint_as_float(u[q * 8 + 5]) * mul);
            v.w = pack2(__uint_as_float(u[q * 8 + 6]) * mul, __uint_as_float(u[q * 8 + 7]) * mul);
            d4[q] = v;
        }
    }
}

// Work of one CTA: up to two items of its role and head, key (KV) or query
// (Q) blocks tb and nblk-1-tb, so every CTA walks nblk+1 blocks (causal).
struct Items {
    int n_items, tb0, tb1;
    __device__ __forceinline__ int tb(int k) const { return k == 0 ? tb0 : tb1; }
};
__device__ __forceinline__ Items cta_items(const BwdParams& p, int pr) {
    Items it;
    it.tb0 = pr;
    it.tb1 = p.nblk - 1 - pr;
    it.n_items = it.tb1 == it.tb0 ? 1 : 2;
    return it;
}
// (first block walked, blocks walked) of item tb
__device__ __forceinline__ void item_range(const BwdParams& p, bool role_q, int tb, int& first, int& n) {
    first = role_q ? 0 : (p.causal ? tb : 0);
    n = role_q ? (p.causal ? tb + 1 : p.nblk) : p.nblk - first;
}

__global__ void __launch_bounds__(kThreadsB, 1)
    attention_bwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                         const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                         const BwdParams p) {
    extern __shared__ std::uint8_t smem_raw[];
    const std::uint32_t base = smem_u32(smem_raw);
    if (base & 1023u) __trap();  // SW128 tiles need 1 KB alignment
    const std::uint32_t sFix0 = base, sFix1 = base + kTile, sFixV = base + 2 * kTile;
    const std::uint32_t sStg = base + kStage;
    const float* fixv = reinterpret_cast<const float*>(smem_raw + 2 * kTile);
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem_raw + 3 * kStage);
    const std::uint32_t b0 = smem_u32(bars);
    // fix_full | stg_full[2] | stg_empty[2] | s_full | p_full | ds_full | o_done | dp_full | fix_empty | acc_empty
    const std::uint32_t fix_full = b0, stg_full = b0 + 8, stg_empty = b0 + 24, s_full = b0 + 40, p_full = b0 + 48,
                        ds_full = b0 + 56, o_done = b0 + 64, dp_full = b0 + 72, fix_empty = b0 + 80,
                        acc_empty = b0 + 88;
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 12);

    pdl_trigger();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    // head-major order (all CTAs are equal work): the ~2 heads in flight keep
    // their q, k, v, dO tiles (5 MB per head) L2-resident while every CTA of
    // the head streams them
    const bool role_q = blockIdx.x & 1;
    const int idx = blockIdx.x >> 1, npairs = (p.nblk + 1) / 2;
    const int h = idx / npairs;
    const Items items = cta_items(p, idx % npairs);

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tq)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tk)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tv)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tdo)) : "memory");
        for (int i = 0; i < 6; ++i) mbar_init(b0 + 8 * i, 1);  // fix, stg full/empty, s_full
        mbar_init(p_full, 8);
        mbar_init(ds_full, 8);
        mbar_init(o_done, 1);
        mbar_init(dp_full, 1);
        mbar_init(fix_empty, 1);
        mbar_init(acc_empty, 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) tmem_alloc(smem_u32(tmem_slot), 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();  // D (attn_bwd_prep) and the forward's lse are complete
    const std::uint32_t tmem = *tmem_slot;
    const std::uint32_t tS = tmem, tdP = tmem + 128, tA0 = tmem + 256, tA1 = tmem + 384;

    if (warp == 0) {
        if (lane == 0) {
            const std::int64_t hs = static_cast<std::int64_t>(h) * p.seq;
            int g = 0;  // blocks walked by the previous items (stage ring position)
            for (int k = 0; k < items.n_items; ++k) {
                const int tb = items.tb(k);
                int first, n;
                item_range(p, role_q, tb, first, n);
                if (k > 0) mbar_wait(fix_empty, (k - 1) & 1);  // the previous item's last MMAs are done
                if (!role_q) {  // fixed K_j, V_j; walked Q_i, dO_i, lse_i, D_i
                    mbar_expect_tx(fix_full, 2 * kTile);
                    tma_load_3d(sFix0, &tk, 0, tb * kT, h, fix_full);
                    tma_load_3d(sFix0 + kAtomB, &tk, 64, tb * kT, h, fix_full);
                    tma_load_3d(sFix1, &tv, 0, tb * kT, h, fix_full);
                    tma_load_3d(sFix1 + kAtomB, &tv, 64, tb * kT, h, fix_full);
                } else {  // fixed Q_i, dO_i, lse_i, D_i; walked K_j, V_j
                    mbar_expect_tx(fix_full, 2 * kTile + 2 * kVec);
                    tma_load_3d(sFix0, &tq, 0, tb * kT, h, fix_full);
                    tma_load_3d(sFix0 + kAtomB, &tq, 64, tb * kT, h, fix_full);
                    tma_load_3d(sFix1, &tdo, 0, tb * kT, h, fix_full);
                    tma_load_3d(sFix1 + kAtomB, &tdo, 64, tb * kT, h, fix_full);
                    bulk_load(sFixV, p.lse + hs + tb * kT, kVec, fix_full);
                    bulk_load(sFixV + kVec, p.D + hs + tb * kT, kVec, fix_full);
                }
                for (int it = 0; it < n; ++it) {
                    const int gi = g + it, st = gi & 1, blk = first + it;
                    mbar_wait(stg_empty + 8 * st, ((gi >> 1) & 1) ^ 1);
                    const std::uint32_t sb = sStg + st * kStage, fb = stg_full + 8 * st;
                    if (!role_q) {
                        mbar_expect_tx(fb, kStage);
                        tma_load_3d(sb, &tq, 0, blk * kT, h, fb);
                        tma_load_3d(sb + kAtomB, &tq, 64, blk * kT, h, fb);
                        tma_load_3d(sb + kTile, &tdo, 0, blk * kT, h, fb);
                        tma_load_3d(sb + kTile + kAtomB, &tdo, 64, blk * kT, h, fb);
                        bulk_load(sb + 2 * kTile, p.lse + hs + blk * kT, kVec, fb);
                        bulk_load(sb + 2 * kTile + kVec, p.D + hs + blk * kT, kVec, fb);
                    } else {
                        mbar_expect_tx(fb, 2 * kTile);
                        tma_load_3d(sb, &tk, 0, blk * kT, h, fb);
                        tma_load_3d(sb + kAtomB, &tk, 64, blk * kT, h, fb);
                        tma_load_3d(sb + kTile, &tv, 0, blk * kT, h, fb);
                        tma_load_3d(sb + kTile + kAtomB, &tv, 64, blk * kT, h, fb);
                    }
                }
                g += n;
            }
        }
    } else if (warp == 1) {  // whole warp: one elected lane issues
        const std::uint32_t id_kk = make_idesc(1u, kT, kT);              // both operands K-major
        const std::uint32_t id_mn = make_idesc(1u, kT, kHdB) | (1u << 16);  // B MN-major
        // Issue order (KV role): S(0) dP(0) | dV(i) S(i+1) | dK(i) dP(i+1) | ...:
        // S(i+1) overwrites Pᵀ(i) only after dV(i) read it (in-order pipe) and
        // runs while the compute warps turn dP(i) into dS(i); dP(i+1) follows
        // dK(i), which reads dSᵀ(i) from the same columns. The Q role keeps P
        // in registers, so S(i+1) is issued once the warps consumed S(i).
        auto stage_of = [&](int gi) { return sStg + (gi & 1) * kStage; };
        auto wait_stage = [&](int gi) {
            mbar_wait(stg_full + 8 * (gi & 1), (gi >> 1) & 1);
            tc_fence_after();
        };
        auto issue_s = [&](int gi) {  // KV: Sᵀ = K_j Q_iᵀ; Q: S = Q_i K_jᵀ (fixed tile is A)
            const std::uint32_t sb = stage_of(gi);
#pragma unroll
            for (int kk = 0; kk < kHdB / 16; ++kk)
                tc_mma(tS, sdesc(kmaj(sFix0, kk)), sdesc(kmaj(sb, kk)), id_kk, kk != 0, false);
            tc_commit(s_full);
        };
        auto issue_dp = [&](int gi) {  // KV: dPᵀ = V_j dO_iᵀ; Q: dP = dO_i V_jᵀ
            const std::uint32_t sb = stage_of(gi);
#pragma unroll
            for (int kk = 0; kk < kHdB / 16; ++kk)
                tc_mma(tdP, sdesc(kmaj(sFix1, kk)), sdesc(kmaj(sb + kTile, kk)), id_kk, kk != 0, false);
            tc_commit(dp_full);
        };
        int g = 0;
        for (int k = 0; k < items.n_items; ++k) {
            int first, n;
            item_range(p, role_q, items.tb(k), first, n);
            mbar_wait(fix_full, k & 1);
            wait_stage(g);
            issue_s(g);
            issue_dp(g);
            for (int it = 0; it < n; ++it) {
                const int gi = g + it;
                const std::uint32_t sb = stage_of(gi);
                const bool more = it + 1 < n;
                mbar_wait(p_full, gi & 1);  // KV: Pᵀ(i) in TMEM; Q: S(i) consumed
                tc_fence_after();
                if (it == 0 && k > 0) {  // the previous item's accumulators were read out
                    mbar_wait(acc_empty, (k - 1) & 1);
                    tc_fence_after();
                }
                if (!role_q) {
                    // dV += Pᵀ dO_i (A = Pᵀ in TMEM, K = queries; B = dO_i MN-major)
#pragma unroll
                    for (int kk = 0; kk < kT / 16; ++kk)
                        tc_mma_ts(tA0, tS + (kk >> 2) * 64 + (kk & 3) * 8, sdesc_mn16(sb + kTile + kk * 2048),
                                  id_mn, (it | kk) != 0);
                }
                if (more) {
                    wait_stage(gi + 1);
                    issue_s(gi + 1);
                }
                mbar_wait(ds_full, gi & 1);
                tc_fence_after();
                if (!role_q) {
                    // dK += dSᵀ Q_i (A = dSᵀ in TMEM; B = Q_i MN-major)
#pragma unroll
                    for (int kk = 0; kk < kT / 16; ++kk)
                        tc_mma_ts(tA1, tdP + (kk >> 2) * 64 + (kk & 3) * 8, sdesc_mn16(sb + kk * 2048), id_mn,
                                  (it | kk) != 0);
                } else {
                    // dQ += dS K_j (A = dS in TMEM, K = keys; B = K_j MN-major)
#pragma unroll
                    for (int kk = 0; kk < kT / 16; ++kk)
                        tc_mma_ts(tA0, tdP + (kk >> 2) * 64 + (kk & 3) * 8, sdesc_mn16(sb + kk * 2048), id_mn,
                                  (it | kk) != 0);
                }
                tc_commit(stg_empty + 8 * (gi & 1));
                if (more) issue_dp(gi + 1);
            }
            tc_commit(fix_empty);
            tc_commit(o_done);
            g += n;
        }
    } else {
        // two warps per TMEM lane quadrant: warp w owns rows 32*(w%4).. and
        // the 64 columns [64*hf, +64) of them; its bf16 P / dS pairs go to the
        // first 32 of those columns (the MMA A operand reads columns
        // 64*(kk/4) + 8*(kk%4) for K16 step kk), never over a column another
        // warp has still to read
        const int lane_base = (warp % 4) * 32, hf = (warp - 2) / 4, c_lo = 64 * hf;
        const int r = lane_base + lane;  // this thread's TMEM lane = tile row
        const std::uint32_t trow = (static_cast<std::uint32_t>(lane_base) << 16) + static_cast<std::uint32_t>(c_lo);
        constexpr float kLog2e = 1.4426950408889634f;
        const float sl2 = p.scale_log2;
        std::uint32_t pk[32];
        int g = 0;
        for (int k = 0; k < items.n_items; ++k) {
            const int tb = items.tb(k);
            int first, n;
            item_range(p, role_q, tb, first, n);
            const std::int64_t row = static_cast<std::int64_t>(tb) * kT + r;
            const std::int64_t col = static_cast<std::int64_t>(h) * kHdB + c_lo;
            if (!role_q) {
                for (int it = 0; it < n; ++it) {
                    const int gi = g + it, i = first + it;
                    const float* lse =
                        reinterpret_cast<const float*>(smem_raw + kStage * (1 + (gi & 1)) + 2 * kTile) + c_lo;
                    const float* Dv = lse + kT;
                    const bool diag = p.causal && i == tb;  // key r > query c is masked
                    mbar_wait(s_full, gi & 1);
                    tc_fence_after();
#pragma unroll
                    for (int c0 = 0; c0 < 64; c0 += 32) {
                        std::uint32_t u[32];
                        TN_LD32(tS + trow + c0, u);
                        tc_wait_ld();
#pragma unroll
                        for (int cc = 0; cc < 32; cc += 2) {
                            const int c = c0 + cc;
                            float x0 = fmaf(__uint_as_float(u[cc]), sl2, -lse[c] * kLog2e);
                            float x1 = fmaf(__uint_as_float(u[cc + 1]), sl2, -lse[c + 1] * kLog2e);
                            float p0 = ex2(x0), p1 = ex2(x1);
                            if (diag) {
                                if (r > c_lo + c) p0 = 0.f;
                                if (r > c_lo + c + 1) p1 = 0.f;
                            }
                            pk[c / 2] = pack2(p0, p1);
                        }
                    }
                    TN_ST32(tS + trow, pk);  // Pᵀ (bf16 pairs) over Sᵀ
                    tc_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(p_full);
                    mbar_wait(dp_full, gi & 1);
                    tc_fence_after();
#pragma unroll
                    for (int c0 = 0; c0 < 64; c0 += 32) {
                        std::uint32_t u[32];
                        TN_LD32(tdP + trow + c0, u);
                        tc_wait_ld();
#pragma unroll
                        for (int cc = 0; cc < 32; cc += 2) {
                            const int c = c0 + cc;
                            const float2 pp = unpack2(pk[c / 2]);
                            pk[c / 2] = pack2(pp.x * (__uint_as_float(u[cc]) - Dv[c]),
                                              pp.y * (__uint_as_float(u[cc + 1]) - Dv[c + 1]));
                        }
                    }
                    TN_ST32(tdP + trow, pk);  // dSᵀ over dPᵀ
                    tc_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(ds_full);
                }
                mbar_wait(o_done, k & 1);
                tc_fence_after();
                store_row(tA0 + trow, p.dv + row * p.ldg + col, 1.0f);
                if (p.rope)  // warp half hf takes RoPE pairs [32 hf, +32) of the whole row
                    store_row_rope(tA1 + trow - c_lo, p.dk + row * p.ldg + static_cast<std::int64_t>(h) * kHdB,
                                   p.scale, p.rope + row * kHdB, 32 * hf);
                else
                    store_row(tA1 + trow, p.dk + row * p.ldg + col, p.scale);
            } else {
                mbar_wait(fix_full, k & 1);  // lse_i, D_i staged with Q_i
                const float lse2 = fixv[r] * kLog2e, Dr = fixv[kT + r];
                for (int it = 0; it < n; ++it) {
                    const int gi = g + it, j = first + it;
                    const bool diag = p.causal && j == tb;  // key c > query r is masked
                    mbar_wait(s_full, gi & 1);
                    tc_fence_after();
#pragma unroll
                    for (int c0 = 0; c0 < 64; c0 += 32) {
                        std::uint32_t us[32];
                        TN_LD32(tS + trow + c0, us);
                        tc_wait_ld();
#pragma unroll
                        for (int cc = 0; cc < 32; cc += 2) {
                            const int c = c0 + cc;
                            float p0 = ex2(fmaf(__uint_as_float(us[cc]), sl2, -lse2));
                            float p1 = ex2(fmaf(__uint_as_float(us[cc + 1]), sl2, -lse2));
                            if (diag) {
                                if (c_lo + c > r) p0 = 0.f;
                                if (c_lo + c + 1 > r) p1 = 0.f;
                            }
                            pk[c / 2] = pack2(p0, p1);  // the bf16 P the KV role multiplies
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(p_full);  // S(i) consumed: S(i+1) may overwrite it
                    mbar_wait(dp_full, gi & 1);
                    tc_fence_after();
#pragma unroll
                    for (int c0 = 0; c0 < 64; c0 += 32) {
                        std::uint32_t ud[32];
                        TN_LD32(tdP + trow + c0, ud);
                        tc_wait_ld();
#pragma unroll
                        for (int cc = 0; cc < 32; cc += 2) {
                            const int c = c0 + cc;
                            const float2 pp = unpack2(pk[c / 2]);
                            pk[c / 2] = pack2(pp.x * (__uint_as_float(ud[cc]) - Dr),
                                              pp.y * (__uint_as_float(ud[cc + 1]) - Dr));
                        }
                    }
                    TN_ST32(tdP + trow, pk);  // dS over dP
                    tc_wait_st();
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(ds_full);
                }
                mbar_wait(o_done, k & 1);
                tc_fence_after();
                if (p.rope)
                    store_row_rope(tA0 + trow - c_lo, p.dq + row * p.ldg + static_cast<std::int64_t>(h) * kHdB,
                                   p.scale, p.rope + row * kHdB, 32 * hf);
                else
                    store_row(tA0 + trow, p.dq + row * p.ldg + col, p.scale);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(acc_empty);  // accumulators read: the next item may overwrite
            g += n;
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_free(tmem, 512);
}

// D[h][i] = sum_c dO[i, h*hd + c] * O[i, h*hd + c] (fp32), one warp per (row, head).
__global__ void attn_bwd_prep(const __nv_bfloat16* __restrict__ o, std::int64_t ldo, const __nv_bfloat16* __restrict__ dout,
                              std::int64_t lddo, float* __restrict__ D, int heads, int seq, int hd) {
    const std::int64_t w = (static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (w >= static_cast<std::int64_t>(heads) * seq) return;
    const int i = static_cast<int>(w / heads), h = static_cast<int>(w % heads);
    const __nv_bfloat16* orow = o + i * ldo + static_cast<std::int64_t>(h) * hd;
    const __nv_bfloat16* drow = dout + i * lddo + static_cast<std::int64_t>(h) * hd;
    float acc = 0.f;
    for (int c = lane * 2; c < hd; c += 64) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(orow + c));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(drow + c));
        acc = fmaf(a.x, b.x, acc);
        acc = fmaf(a.y, b.y, acc);
    }
#pragma unroll
    for (int s = 16; s > 0; s /= 2) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if (lane == 0) D[static_cast<std::int64_t>(h) * seq + i] = acc;
}

}  // namespace

cudaError_t attention_bwd_prepare(const AttnBwdArgs& a, AttnBwdPlan* plan) {
    plan->args = a;
    auto al16 = [](const void* x) { return (reinterpret_cast<std::uintptr_t>(x) & 15) == 0; };
    const bool ok = a.hd == kHdB && a.seq % kT == 0 && a.seq >= kT && al16(a.q) && al16(a.k) && al16(a.v) &&
                    al16(a.dout) && al16(a.dq) && al16(a.dk) && al16(a.dv) && al16(a.lse) && al16(a.D) && al16(a.rope) &&
                    (a.ldv * 2) % 16 == 0 && (a.lddo * 2) % 16 == 0 && (a.ldg * 2) % 16 == 0 && a.o && a.lse;
    if (!ok) return cudaErrorInvalidValue;
    const std::int64_t shd = static_cast<std::int64_t>(a.seq) * a.hd;
    if (!encode_tma_3d(&plan->tq, a.q, 2, a.hd, a.seq, a.hd, a.heads, shd, 64, kT) ||
        !encode_tma_3d(&plan->tk, a.k, 2, a.hd, a.seq, a.hd, a.heads, shd, 64, kT) ||
        !encode_tma_3d(&plan->tv, a.v, 2, a.hd, a.seq, a.ldv, a.heads, a.hd, 64, kT) ||
        !encode_tma_3d(&plan->tdo, a.dout, 2, a.hd, a.seq, a.lddo, a.heads, a.hd, 64, kT))
        return cudaErrorInvalidValue;
    static std::atomic<unsigned long long> attr_set{0};  // per CUDA device, any thread
    int dev = 0;
    cudaGetDevice(&dev);
    if (!((attr_set.load(std::memory_order_acquire) >> dev) & 1ULL)) {
        cudaFuncSetAttribute(attention_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemB);
        attr_set.fetch_or(1ULL << dev, std::memory_order_release);
    }
    return cudaSuccess;
}

cudaError_t attention_bwd_launch(const AttnBwdPlan& plan, cudaStream_t s) {
    const AttnBwdArgs& a = plan.args;
    const std::int64_t rows = static_cast<std::int64_t>(a.heads) * a.seq;
    attn_bwd_prep<<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(a.o), a.ldo, static_cast<const __nv_bfloat16*>(a.dout), a.lddo, a.D, a.heads,
        a.seq, a.hd);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    BwdParams p;
    p.dq = static_cast<__nv_bfloat16*>(a.dq);
    p.dk = static_cast<__nv_bfloat16*>(a.dk);
    p.dv = static_cast<__nv_bfloat16*>(a.dv);
    p.ldg = a.ldg;
    p.lse = a.lse;
    p.D = a.D;
    p.rope = a.rope;
    p.heads = a.heads;
    p.seq = a.seq;
    p.nblk = a.seq / kT;
    p.causal = a.causal;
    p.scale = a.scale;
    p.scale_log2 = a.scale * 1.4426950408889634f;
    const unsigned grid = static_cast<unsigned>(2 * a.heads * ((p.nblk + 1) / 2));
    return launch_pdl(attention_bwd_kernel, dim3(grid), dim3(kThreadsB), kSmemB, s, plan.tq, plan.tk, plan.tv,
                      plan.tdo, p);
}

double attention_bwd_flops(const AttnBwdArgs& a) {
    // dV, dK, dQ and the recomputed S, dP: five [seq x seq x hd] products per head
    double f = 10.0 * a.heads * static_cast<double>(a.seq) * a.seq * a.hd;
    return a.causal ? f * 0.5 * (1.0 + 1.0 / a.seq) : f;
}

}  // namespace tn::k
