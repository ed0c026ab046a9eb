// Contraction tasks: C = alpha * A·Bᵀ (+ R), batched, on
// the 5th-gen tensor cores. Three persistent warp-specialised kernels:
//
//   gemm_kernel<BN>     1 CTA per SM, M=128 x N=BN tiles (small shapes):
//     warp 0 TMA producer (4-stage ring of 128-byte-swizzled K-major A/B
//     tiles, cp.async.bulk.tensor + mbarrier tx counts), warp 1 MMA issuer
//     (tcgen05.mma into a double-buffered TMEM accumulator, one elected lane
//     of a converged warp), warps 2-5 epilogue (tcgen05.ld -> registers).
//   gemm_kernel_2sm     CTA pairs (cta_group::2, cluster 2), 256x256 tiles:
//     the leader issues M=256 MMAs, each CTA stages half of A and half of B,
//     multicast commits; double-buffered 2x256-column accumulators.
//   gemm_kernel_2sm_w   CTA pairs, 512x256 "wide" tiles: each CTA owns two
//     128-row halves (all 512 TMEM columns), two drain warpgroups; 25 % fewer
//     operand bytes per FLOP, used for long K.
// Tails: the last partial wave of pair tiles is split into 2 or 4 N-slices
// (slice_brow); stream-K is available as tile "streamk". Epilogues: alpha,
// residual, SwiGLU, QKV+RoPE+Vᵀ, fused-RMSNorm producer/consumer; plain /
// residual / SwiGLU outputs of the pair kernels go through per-warp
// SWIZZLE_64B smem boxes and cp.async.bulk.tensor stores.
// bf16 inputs use kind::f16, fp32 inputs kind::tf32 (same byte geometry:
// a K block is always one 128-byte swizzle atom).
// Deterministic: each output element is accumulated by one CTA in K order
// (stream-K partials are summed in ascending pair order).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "kernels.hpp"
#include "tc_common.cuh"

namespace tn::k {
namespace {

constexpr int kBM = 128;
constexpr int kStages = 4;
constexpr int kAtom = 128;  // bytes of one K block row (SWIZZLE_128B span)
constexpr int kThreads = 32 * 6;

struct Params {
    void* C;
    const void* R;
    int M, N, K, batch;
    int tiles_m, tiles_n;
    std::int64_t ldc, sc;
    float alpha;
    int out_dtype;
    int causal;
    int in_bytes;
    int a_batched, b_batched;
    int epi;  // 0 plain, 1 swiglu (out[:, 128b + j] = silu(C[:, 256b + j]) * C[:, 256b + 128 + j]), 2 qkv_rope
    const float* rope;  // qkv_rope: [seq, 64, 2] (cos, sin)
    int heads;          // qkv_rope: heads per q/k/v section (hd = 128)
    // Stream-K tail (CTA-pair kernel): tiles [0, dp_tiles) go round-robin to
    // the pairs; the K blocks of the remaining tiles are split evenly across
    // all pairs (sk_total = sk_tiles * sk_nk blocks). Partial accumulators go
    // to ws (one 256x256 fp32 slot per pair) and are summed by the pair that
    // owns a tile's first K block, in ascending pair order (deterministic).
    int dp_tiles, sk_nk;
    long long sk_total;
    // Sliced tail (CTA-pair kernels, default): the tiles of the last, partial
    // wave of pairs are each split into `tail_split` (2 or 4) N-slices of
    // 256/tail_split accumulator columns (N=128/64 MMAs), so the tail costs
    // 1/tail_split of a tile-time when the slices fit in one wave. Tiles
    // [dp_tiles, dp_tiles + tail_units / tail_split).
    int tail_split, tail_units;
    int tma_c;  // 1: plain/SwiGLU epilogues store through smem staging + TMA (tensor map `tc`)
    int split;  // 3xTF32 (1-CTA kernel, SPLIT = true)
    // Fused RMSNorm (consumer side): row m of the product is scaled by
    // rsqrt(sum_c rs_P[(rs_row0 + m)*rs_ld + c] / dim + eps), c in [0, rs_chunks),
    // summed in c order — the per-32-column sums of squares its producer wrote.
    const float* rs_P;
    int rs_ld, rs_row0, rs_chunks;
    float rs_inv_dim, rs_eps;
    // Fused RMSNorm (producer side, plain epilogue + residual, bf16, TMA
    // path): x = bf16(alpha*acc + R) goes to C (box batch 0), h = bf16(x * g)
    // to the rows after it (box batch 1), and per 32-column chunk c the sum of
    // x^2 (in column order) to no_P[row*(N/32) + c].
    const __nv_bfloat16* no_g;
    float* no_P;
    float* ws;
    unsigned* flags;  // per CTA of each pair: epoch of its last published partial
    unsigned epoch;
    // Split-K (1-CTA kernel, plain epilogue): each tile's K blocks are split
    // into `ksplit` ranges (work unit = tile x split); every unit writes its
    // fp32 partial to ws, and the unit that completes a tile's count sums the
    // partials in split order 0..ksplit-1 (the order never depends on which
    // unit arrives last), then runs the epilogue. The counter only elects the
    // reducer and is reset by it.
    int ksplit;
    // MN-major operands (bf16): A stored [K, M] (M contiguous, row pitch lda),
    // B stored [K, N]; staged as 64x64 boxes (64 M/N elements x 64 K rows, 8 KB,
    // SWIZZLE_128B) read by MN-major UMMA descriptors (LBO = 8 KB between
    // 64-element chunks, SBO = 1 KB between 8-row K groups, +2 KB per K = 16).
    int a_mn, b_mn;
};

__device__ __forceinline__ std::uint64_t sdesc_mn(std::uint32_t saddr) {
    std::uint64_t d = 0;
    d |= static_cast<std::uint64_t>((saddr & 0x3FFFF) >> 4);
    d |= static_cast<std::uint64_t>(8192 >> 4) << 16;
    d |= static_cast<std::uint64_t>(1024 >> 4) << 32;
    d |= static_cast<std::uint64_t>(1) << 46;
    d |= static_cast<std::uint64_t>(2) << 61;
    return d;
}
// Operand descriptor and its per-K16 increment (descriptor units of 16 B).
__device__ __forceinline__ std::uint64_t op_desc(std::uint32_t saddr, int mn) { return mn ? sdesc_mn(saddr) : sdesc(saddr); }
__device__ __forceinline__ int op_kstep(int mn) { return mn ? 2048 >> 4 : 32 >> 4; }
// Stages `rows` rows (M or N) x one 64-element K block of an operand at
// smem `dst`: K-major = one box {64 K, rows}; MN-major = rows/64 boxes {64, 64 K}.
__device__ __forceinline__ void load_operand(std::uint32_t dst, const CUtensorMap* map, int k0, int row0, int rows,
                                             int batch, std::uint32_t bar, int mn) {
    if (!mn) {
        tma_load_3d(dst, map, k0, row0, batch, bar);
        return;
    }
    for (int i = 0; i < rows / 64; ++i) tma_load_3d(dst + i * 8192, map, row0 + i * 64, k0, batch, bar);
}
// Same for the CTA-pair kernels (.cta_group::2 loads signalling the leader's barrier).
__device__ __forceinline__ void load_operand_2sm(std::uint32_t dst, const CUtensorMap* map, int k0, int row0,
                                                 int rows, int batch, std::uint32_t leader_bar, int mn) {
    if (!mn) {
        tma_load_3d_2sm(dst, map, k0, row0, batch, leader_bar);
        return;
    }
    for (int i = 0; i < rows / 64; ++i) tma_load_3d_2sm(dst + i * 8192, map, row0 + i * 64, k0, batch, leader_bar);
}

__device__ __forceinline__ float row_alpha(const Params& p, int row, bool row_ok) {
    if (!p.rs_P || !row_ok) return p.alpha;
    const float* P = p.rs_P + static_cast<std::int64_t>(p.rs_row0 + row) * p.rs_ld;  // row-major [rows, chunks]
    float ss = 0.f;
    if ((p.rs_chunks & 3) == 0 && (reinterpret_cast<std::uintptr_t>(P) & 15) == 0) {
        const float4* P4 = reinterpret_cast<const float4*>(P);
#pragma unroll 8
        for (int c = 0; c < p.rs_chunks / 4; ++c) {
            const float4 x = __ldg(P4 + c);
            ss += x.x;
            ss += x.y;
            ss += x.z;
            ss += x.w;
        }
    } else {
        for (int c = 0; c < p.rs_chunks; ++c) ss += __ldg(P + c);
    }
    return p.alpha * rsqrtf(ss * p.rs_inv_dim + p.rs_eps);
}

__device__ __forceinline__ bool tile_skipped(const Params& p, int mb, int nb, int bn) {
    return p.causal == 1 && nb * bn > mb * kBM + kBM - 1;
}

// Grouped rasterisation: within a group of up to 16 M-tiles the M index runs
// fastest, so the ~74-148 tiles in flight share a few B column panels and a
// group's A rows stay L2-resident (B is streamed from DRAM about once instead
// of once per M-tile row).
__device__ __forceinline__ void decode(const Params& p, int t, int& b, int& mb, int& nb) {
    constexpr int G = 16;
    const int per = p.tiles_m * p.tiles_n;
    b = t / per;
    const int r = t - b * per;
    const int group = r / (G * p.tiles_n);
    const int m0 = group * G;
    const int gsz = min(G, p.tiles_m - m0);
    const int local = r - group * G * p.tiles_n;
    mb = m0 + local % gsz;
    nb = local / gsz;
}

__device__ __forceinline__ int kblocks(const Params& p, int mb, int bk) {
    int kb = (p.K + bk - 1) / bk;
    if (p.causal == 2) kb = min(kb, ((mb + 1) * kBM + bk - 1) / bk);
    return kb;
}

// Work unit u of the 1-CTA kernel -> (tile, split, K-block range).
__device__ __forceinline__ void unit_range(const Params& p, int u, int nk, int& t, int& k, int& kb0, int& kb1) {
    const int ks = p.ksplit;
    t = u / ks;
    k = u - t * ks;
    kb0 = static_cast<int>(static_cast<long long>(nk) * k / ks);
    kb1 = static_cast<int>(static_cast<long long>(nk) * (k + 1) / ks);
}

__device__ __forceinline__ std::uint32_t pack_bf16(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<std::uint32_t*>(&v);
}

// Stores one 32-column chunk of an accumulator row (alpha, residual, dtype).
__device__ __forceinline__ void store_chunk(const Params& p, const std::uint32_t* r, std::int64_t off, int n0,
                                            bool row_ok, bool vec_ok, float alpha) {
    if (!row_ok || n0 >= p.N) return;
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * alpha;
    if (vec_ok) {
        if (p.out_dtype == BF16) {
            __nv_bfloat16* c = static_cast<__nv_bfloat16*>(p.C) + off + n0;
            if (p.R) {
                const uint4* rr = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.R) + off + n0);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint4 x = rr[q];
                    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&x);
#pragma unroll
                    for (int j = 0; j < 8; ++j) v[q * 8 + j] += __bfloat162float(h[j]);
                }
            }
            uint4* dst = reinterpret_cast<uint4*>(c);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                dst[q] = make_uint4(pack_bf16(v[q * 8 + 0], v[q * 8 + 1]), pack_bf16(v[q * 8 + 2], v[q * 8 + 3]),
                                    pack_bf16(v[q * 8 + 4], v[q * 8 + 5]), pack_bf16(v[q * 8 + 6], v[q * 8 + 7]));
        } else {
            float* c = static_cast<float*>(p.C) + off + n0;
            if (p.R) {
                const float4* rr = reinterpret_cast<const float4*>(static_cast<const float*>(p.R) + off + n0);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    float4 x = rr[q];
                    v[q * 4 + 0] += x.x;
                    v[q * 4 + 1] += x.y;
                    v[q * 4 + 2] += x.z;
                    v[q * 4 + 3] += x.w;
                }
            }
            float4* dst = reinterpret_cast<float4*>(c);
#pragma unroll
            for (int q = 0; q < 8; ++q) dst[q] = make_float4(v[q * 4], v[q * 4 + 1], v[q * 4 + 2], v[q * 4 + 3]);
        }
    } else {
        for (int j = 0; j < 32 && n0 + j < p.N; ++j) {
            float x = v[j];
            if (p.out_dtype == BF16) {
                __nv_bfloat16* c = static_cast<__nv_bfloat16*>(p.C) + off + n0 + j;
                if (p.R) x += __bfloat162float(static_cast<const __nv_bfloat16*>(p.R)[off + n0 + j]);
                *c = __float2bfloat16_rn(x);
            } else {
                float* c = static_cast<float*>(p.C) + off + n0 + j;
                if (p.R) x += static_cast<const float*>(p.R)[off + n0 + j];
                *c = x;
            }
        }
    }
}

// --- TMA-store epilogue ------------------------------------------------------
// Each epilogue warp owns two 2 KB staging buffers, each one {64 B x 32 rows}
// TMA box in the SWIZZLE_64B layout (16-byte chunk q of row r at
// r*64 + ((q ^ ((r >> 1) & 3)) << 4): a warp's 16-byte stores hit 8 distinct
// bank groups, i.e. the ideal 4 wavefronts per 512 B). A 32-column chunk of
// accumulator rows (one row per lane) is packed into a buffer and one lane
// issues cp.async.bulk.tensor: full-line global writes, asynchronous, so the
// warp (and the TMEM columns it drained) is free as soon as the smem writes
// are fenced. Replaces 32 scattered rows per store instruction.
constexpr int kStgBuf = 2048;
constexpr int kStgWarp = 2 * kStgBuf;

__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, std::uint32_t src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<std::uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void st_shared_v4(std::uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

struct Stager {
    std::uint32_t base;  // this warp's two buffers
    int n;               // boxes issued so far (buffer = n & 1)
};

// Alpha and residual of one 32-column chunk of this lane's row (vector path).
__device__ __forceinline__ void chunk_values(const Params& p, const std::uint32_t* r, std::int64_t off, int n0,
                                             bool row_ok, float* v, float alpha) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * alpha;
    if (!p.R || !row_ok || n0 >= p.N) return;
    if (p.out_dtype == BF16) {
        const uint4* rr = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(p.R) + off + n0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint4 x = rr[q];
            const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&x);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[q * 8 + j] += __bfloat162float(h[j]);
        }
    } else {
        const float4* rr = reinterpret_cast<const float4*>(static_cast<const float*>(p.R) + off + n0);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            float4 x = rr[q];
            v[q * 4 + 0] += x.x;
            v[q * 4 + 1] += x.y;
            v[q * 4 + 2] += x.z;
            v[q * 4 + 3] += x.w;
        }
    }
}

// Stages a 32-column chunk (values for rows row0 + lane, columns n0..n0+31 of
// batch b) and stores it with TMA; out-of-range rows/columns are clipped by
// the tensor map. bf16: one box; fp32: two 16-column boxes.
__device__ __forceinline__ void stage_chunk(const Params& p, const CUtensorMap* tc, Stager& st, const float* v,
                                            int row0, int n0, int b) {
    const int lane = threadIdx.x % 32;
    const std::uint32_t sw = static_cast<std::uint32_t>((lane >> 1) & 3);
    const int nbox = p.out_dtype == BF16 ? 1 : 2;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (h >= nbox) break;
        const std::uint32_t buf = st.base + static_cast<std::uint32_t>(st.n & 1) * kStgBuf;
        if (lane == 0) bulk_wait_read1();  // the box issued from this buffer two boxes ago has been read
        __syncwarp();
        uint4 w[4];
        if (p.out_dtype == BF16) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                w[q] = make_uint4(pack_bf16(v[q * 8 + 0], v[q * 8 + 1]), pack_bf16(v[q * 8 + 2], v[q * 8 + 3]),
                                  pack_bf16(v[q * 8 + 4], v[q * 8 + 5]), pack_bf16(v[q * 8 + 6], v[q * 8 + 7]));
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
                w[q] = make_uint4(__float_as_uint(v[h * 16 + q * 4 + 0]), __float_as_uint(v[h * 16 + q * 4 + 1]),
                                  __float_as_uint(v[h * 16 + q * 4 + 2]), __float_as_uint(v[h * 16 + q * 4 + 3]));
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) st_shared_v4(buf + lane * 64 + ((static_cast<std::uint32_t>(q) ^ sw) << 4), w[q]);
        fence_async_smem();
        __syncwarp();
        if (lane == 0) {
            tma_store_3d(tc, buf, n0 + h * 16, row0, b);
            bulk_commit();
        }
        ++st.n;
    }
}

// Residual epilogues read R in 64-byte pieces of each lane's row, one
// 32-column chunk at a time: 32 rows x 64 B per warp load, each piece in a
// different DRAM page, each row's page reopened once per chunk. Pulling the
// lane's whole row segment (w columns, contiguous) into L2 before the tile's
// accumulator is ready turns that into one burst per row and overlaps it
// with the tile's MMAs (C = U·Bᵀ + base at K = 64, 4096 x 22016: 136 -> 111 us
// with the prefetch at the start of the epilogue; no residual 53 us).
__device__ __forceinline__ void prefetch_residual(const Params& p, std::int64_t off, int n0, int w, bool row_ok) {
    // Only short-K GEMMs, whose tiles are epilogue-bound: with a long K the
    // residual read overlaps the next tile's main loop anyway, and the early
    // lines crowd A/B out of L2 (ncu DRAM per launch: ffn_out 333 -> 365 MB,
    // attn_out 146 -> 167 MB with the prefetch on every residual GEMM).
    if (!p.R || p.epi != 0 || !row_ok || n0 >= p.N || p.K > 1024) return;
    const int es = p.out_dtype == BF16 ? 2 : 4;
    const char* rb = static_cast<const char*>(p.R) + (off + n0) * es;
    const int nb = min(w, p.N - n0) * es;
    for (int b = 0; b < nb; b += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(rb + b));
}

// Plain epilogue through the stager: 128-row x width accumulator slab.
__device__ __forceinline__ void epilogue_plain_tma(const Params& p, const CUtensorMap* tc, Stager& st,
                                                   std::uint32_t tbase, std::int64_t off, int row0, int n0, int width,
                                                   int b, bool row_ok, float alpha) {
#pragma unroll 1
    for (int c0 = 0; c0 < width; c0 += 32) {
        std::uint32_t r[32];
        TN_LD32(tbase + c0, r);
        tc_wait_ld();
        float v[32];
        chunk_values(p, r, off, n0 + c0, row_ok, v, alpha);
        if (p.no_P) {  // fused RMSNorm producer: x, h = x * g, per-chunk sum of x^2
            float ss = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                v[j] = __bfloat162float(__float2bfloat16_rn(v[j]));  // x as stored
                ss = fmaf(v[j], v[j], ss);
            }
            stage_chunk(p, tc, st, v, row0, n0 + c0, 0);
            if (row_ok) p.no_P[static_cast<std::int64_t>(row0 + threadIdx.x % 32) * (p.N / 32) + (n0 + c0) / 32] = ss;
            const uint4* gv = reinterpret_cast<const uint4*>(p.no_g + n0 + c0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                float g[8];
                const uint4 u = __ldg(gv + q);
                const __nv_bfloat16* hb = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
                for (int j = 0; j < 8; ++j) g[j] = __bfloat162float(hb[j]);
#pragma unroll
                for (int j = 0; j < 8; ++j) v[q * 8 + j] *= g[j];
            }
            stage_chunk(p, tc, st, v, row0, n0 + c0, 1);
        } else {
            stage_chunk(p, tc, st, v, row0, n0 + c0, b);
        }
    }
}

// SwiGLU epilogue: the N tile holds 128-column gate/up block pairs (the
// weight rows are interleaved that way), so each output column needs two
// TMEM columns of the same row: out = silu(alpha*g) * (alpha*u).
__device__ __forceinline__ void epilogue_swiglu(const Params& p, std::uint32_t tbase, std::int64_t off, int H,
                                                int out0, bool row_ok, float alpha) {
    Params q = p;
    q.N = p.N / 2;
    q.alpha = 1.0f;
    q.R = nullptr;
    const int ob = p.out_dtype == BF16 ? 2 : 4;
    const bool vec_ok = (q.N % 32 == 0) && ((q.ldc * ob) % 16 == 0) && ((reinterpret_cast<std::uintptr_t>(q.C) & 15) == 0);
#pragma unroll 1
    for (int c0 = 0; c0 < H; c0 += 32) {
        std::uint32_t g[32], u[32];
        TN_LD32(tbase + c0, g);
        TN_LD32(tbase + H + c0, u);
        tc_wait_ld();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const float x = __uint_as_float(g[j]) * alpha, y = __uint_as_float(u[j]) * alpha;
            g[j] = __float_as_uint(x / (1.0f + __expf(-x)) * y);
        }
        store_chunk(q, g, off, out0 + c0, row_ok, vec_ok, 1.0f);
    }
}

// H: gate (= up) columns in the accumulator ([gate | up]); out0: first output column.
__device__ __forceinline__ void epilogue_swiglu_tma(const Params& p, const CUtensorMap* tc, Stager& st,
                                                    std::uint32_t tbase, int row0, int H, int out0, int b, float alpha) {
#pragma unroll 1
    for (int c0 = 0; c0 < H; c0 += 32) {
        std::uint32_t g[32], u[32];
        TN_LD32(tbase + c0, g);
        TN_LD32(tbase + H + c0, u);
        tc_wait_ld();
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const float x = __uint_as_float(g[j]) * alpha, y = __uint_as_float(u[j]) * alpha;
            v[j] = x / (1.0f + __expf(-x)) * y;
        }
        stage_chunk(p, tc, st, v, row0, out0 + c0, b);
    }
}

// QKV epilogue (hd = 128, BN = 256 = two heads per N tile): rotate-half
// RoPE for the q and k sections written head-major [H, seq, 128], and the v
// section written transposed [H, 128, seq] (lanes hold consecutive tokens, so
// the transposed stores coalesce across the warp). Output = packed
// [q | k | vᵀ], each H*seq*128 elements.
__device__ __forceinline__ void epilogue_qkv_rope(const Params& p, std::uint32_t tbase, int row, int n0, int width,
                                                  bool row_ok, float alpha) {
    constexpr int HD = 128;
    const std::int64_t sec = static_cast<std::int64_t>(p.heads) * p.M * HD;
    __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.C);
#pragma unroll 1
    for (int hb = 0; hb < width; hb += HD) {
        const int col = n0 + hb;  // first column of this head in [0, 3*H*HD)
        const int which = col / (p.heads * HD), h = (col % (p.heads * HD)) / HD;
        if (which < 2) {
            __nv_bfloat16* dst = out + which * sec + (static_cast<std::int64_t>(h) * p.M + row) * HD;
#pragma unroll 1
            for (int c0 = 0; c0 < HD / 2; c0 += 32) {
                std::uint32_t lo[32], hi[32];
                TN_LD32(tbase + hb + c0, lo);
                TN_LD32(tbase + hb + HD / 2 + c0, hi);
                tc_wait_ld();
                if (!row_ok) continue;
                const float4* cs = reinterpret_cast<const float4*>(p.rope + (static_cast<std::int64_t>(row) * (HD / 2) + c0) * 2);
                float a[32], b[32];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const float4 q = cs[j];  // (cos_2j, sin_2j, cos_2j+1, sin_2j+1)
                    const float x0 = __uint_as_float(lo[2 * j]) * alpha, y0 = __uint_as_float(hi[2 * j]) * alpha;
                    const float x1 = __uint_as_float(lo[2 * j + 1]) * alpha, y1 = __uint_as_float(hi[2 * j + 1]) * alpha;
                    a[2 * j] = x0 * q.x - y0 * q.y;
                    b[2 * j] = y0 * q.x + x0 * q.y;
                    a[2 * j + 1] = x1 * q.z - y1 * q.w;
                    b[2 * j + 1] = y1 * q.z + x1 * q.w;
                }
                uint4* d0 = reinterpret_cast<uint4*>(dst + c0);
                uint4* d1 = reinterpret_cast<uint4*>(dst + HD / 2 + c0);
#pragma unroll
                for (int qd = 0; qd < 4; ++qd) {
                    d0[qd] = make_uint4(pack_bf16(a[qd * 8], a[qd * 8 + 1]), pack_bf16(a[qd * 8 + 2], a[qd * 8 + 3]),
                                        pack_bf16(a[qd * 8 + 4], a[qd * 8 + 5]), pack_bf16(a[qd * 8 + 6], a[qd * 8 + 7]));
                    d1[qd] = make_uint4(pack_bf16(b[qd * 8], b[qd * 8 + 1]), pack_bf16(b[qd * 8 + 2], b[qd * 8 + 3]),
                                        pack_bf16(b[qd * 8 + 4], b[qd * 8 + 5]), pack_bf16(b[qd * 8 + 6], b[qd * 8 + 7]));
                }
            }
        } else {
            __nv_bfloat16* dst = out + 2 * sec + static_cast<std::int64_t>(h) * HD * p.M + row;
#pragma unroll 1
            for (int c0 = 0; c0 < HD; c0 += 32) {
                std::uint32_t v[32];
                TN_LD32(tbase + hb + c0, v);
                tc_wait_ld();
                if (!row_ok) continue;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    dst[static_cast<std::int64_t>(c0 + j) * p.M] = __float2bfloat16_rn(__uint_as_float(v[j]) * alpha);
            }
        }
    }
}

// 3xTF32 operand split (SPLIT kernels): x = hi + lo with hi = tf32(x)
// (round to nearest, low 13 mantissa bits zero) and lo = tf32(x - hi); the
// subtraction is exact, so hi·hi + hi·lo + lo·hi misses only lo·lo
// (|lo| <= 2^-11 |x|) and fp32-input products come out fp32-accurate.
__device__ __forceinline__ float tf32_rna(float x) {
    std::uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
// Splits `bytes` of fp32 operands in place (hi) and into `lo` (same offsets,
// so the same 128-byte swizzle applies to both buffers).
__device__ __forceinline__ void split_operands(std::uint8_t* hi, std::uint8_t* lo, int bytes, int tid, int nthr) {
#pragma unroll 4
    for (int off = tid * 16; off < bytes; off += nthr * 16) {
        float4 x = *reinterpret_cast<const float4*>(hi + off);
        float4 h, l;
        h.x = tf32_rna(x.x), l.x = tf32_rna(x.x - h.x);
        h.y = tf32_rna(x.y), l.y = tf32_rna(x.y - h.y);
        h.z = tf32_rna(x.z), l.z = tf32_rna(x.z - h.z);
        h.w = tf32_rna(x.w), l.w = tf32_rna(x.w - h.w);
        *reinterpret_cast<float4*>(hi + off) = h;
        *reinterpret_cast<float4*>(lo + off) = l;
    }
}

// SPLIT kernels also accumulate K in chunks of kChunkKB blocks: each chunk
// goes into a fresh TMEM accumulator and the epilogue adds the chunks in
// fp32 registers (round to nearest). The tensor core's own accumulation
// truncates, so its error grows with the number of MMAs summed into one
// accumulator (measured 7e-6 normwise at K = 1024 unchunked); chunking bounds
// that to one chunk.
constexpr int kChunkKB = 4;

template <int BN, bool SPLIT>
constexpr int stages_1cta() {
    return SPLIT ? (BN >= 128 ? 3 : 4) : kStages;
}
template <int BN, bool SPLIT>
constexpr int threads_1cta() {
    return SPLIT ? kThreads + 128 : kThreads;  // + 4 splitter warps (6-9)
}

template <int BN, bool SPLIT>
__global__ void __launch_bounds__(threads_1cta<BN, SPLIT>(), 1)
    gemm_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, const Params p) {
    constexpr int A_BYTES = kBM * kAtom;
    constexpr int B_BYTES = BN * kAtom;
    constexpr int LOADED = A_BYTES + B_BYTES;               // TMA bytes per stage
    constexpr int STAGE = SPLIT ? 2 * LOADED : LOADED;       // SPLIT: [A_hi | B_hi | A_lo | B_lo]
    constexpr int kStages = stages_1cta<BN, SPLIT>();
    constexpr std::uint32_t TMEM_COLS = 2 * BN;

    extern __shared__ std::uint8_t smem_raw[];
    const std::uint32_t raw = smem_u32(smem_raw);
    const std::uint32_t pad = ((raw + 1023) & ~1023u) - raw;
    std::uint8_t* smem = smem_raw + pad;
    const std::uint32_t sbase = raw + pad;
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + kStages * STAGE);
    const std::uint32_t full = smem_u32(bars), empty = full + 8 * kStages;
    const std::uint32_t tfull = empty + 8 * kStages, tempty = tfull + 16;
    const std::uint32_t splitb = tempty + 16;  // SPLIT: stage s operands split (4 splitter warps)
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + (SPLIT ? 3 : 2) * kStages + 4);

    pdl_trigger();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int bk = kAtom / p.in_bytes;
    const bool tf32 = p.in_bytes == 4;
    const int tiles = p.batch * p.tiles_m * p.tiles_n;
    const int units = tiles * p.ksplit;  // ksplit == 1 unless split-K (never with SPLIT)

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&ta)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tb)) : "memory");
        for (int s = 0; s < kStages; ++s) {
            mbar_init(full + 8 * s, 1);
            mbar_init(empty + 8 * s, 1);
            if (SPLIT) mbar_init(splitb + 8 * s, 4);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + 8 * a, 1);
            mbar_init(tempty + 8 * a, 4);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    pdl_wait();  // previous kernel complete: its outputs are visible, its inputs may be overwritten
    const std::uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            std::uint32_t phase = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int t, ks, kb0, kb1, b, mb, nb;
                unit_range(p, u, 0, t, ks, kb0, kb1);
                decode(p, t, b, mb, nb);
                if (tile_skipped(p, mb, nb, BN)) continue;
                unit_range(p, u, kblocks(p, mb, bk), t, ks, kb0, kb1);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(empty + 8 * stage, phase ^ 1);
                    const std::uint32_t fb = full + 8 * stage;
                    mbar_expect_tx(fb, LOADED);
                    const std::uint32_t sa = sbase + stage * STAGE;
                    load_operand(sa, &ta, kb * bk, mb * kBM, kBM, p.a_batched ? b : 0, fb, p.a_mn);
                    load_operand(sa + A_BYTES, &tb, kb * bk, nb * BN, BN, p.b_batched ? b : 0, fb, p.b_mn);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        {  // whole warp: one elected lane issues (tc_mma)
            const std::uint32_t fmt = tf32 ? 2u : 1u;
            const std::uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) |
                                        (static_cast<std::uint32_t>(p.a_mn) << 15) |
                                        (static_cast<std::uint32_t>(p.b_mn) << 16) |
                                        (static_cast<std::uint32_t>(BN >> 3) << 17) |
                                        (static_cast<std::uint32_t>(kBM >> 4) << 24);
            const int as = op_kstep(p.a_mn), bs = op_kstep(p.b_mn);
            int stage = 0, acc = 0;
            std::uint32_t phase = 0, acc_phase = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                int t, ks, ulo, nk, b, mb, nb;
                unit_range(p, u, 0, t, ks, ulo, nk);
                decode(p, t, b, mb, nb);
                if (tile_skipped(p, mb, nb, BN)) continue;
                unit_range(p, u, kblocks(p, mb, bk), t, ks, ulo, nk);  // K blocks [ulo, nk)
                const int chunk = SPLIT ? kChunkKB : nk - ulo;
                for (int kb0 = ulo; kb0 < nk; kb0 += chunk) {
                mbar_wait(tempty + 8 * acc, acc_phase ^ 1);
                tc_fence_after();
                const std::uint32_t d = tmem + acc * BN;
                for (int kb = kb0; kb < nk && kb < kb0 + chunk; ++kb) {
                    mbar_wait((SPLIT ? splitb : full) + 8 * stage, phase);
                    tc_fence_after();
                    const std::uint32_t sa = sbase + stage * STAGE;
                    const std::uint64_t ad = op_desc(sa, p.a_mn), bd = op_desc(sa + A_BYTES, p.b_mn);
                    if (SPLIT) {
                        const std::uint64_t al = sdesc(sa + LOADED), bl = sdesc(sa + LOADED + A_BYTES);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {  // small terms first, then hi·hi
                            tc_mma(d, al + 2 * k, bd + 2 * k, idesc, (kb != kb0) | (k != 0), true);
                            tc_mma(d, ad + 2 * k, bl + 2 * k, idesc, 1u, true);
                            tc_mma(d, ad + 2 * k, bd + 2 * k, idesc, 1u, true);
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < 4; ++k)  // 4 x K16 per 64-element K block
                            tc_mma(d, ad + as * k, bd + bs * k, idesc, (kb != kb0) | (k != 0), tf32);
                    }
                    tc_commit(empty + 8 * stage);
                    if (++stage == kStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit(tfull + 8 * acc);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
                }
            }
        }
    } else if (SPLIT && warp >= 6) {
        // Splitter warps: per stage, fp32 operands -> (hi in place, lo beside),
        // then a generic->async proxy fence so the MMAs see the new bytes.
        const int tid = threadIdx.x - 6 * 32;
        int stage = 0;
        std::uint32_t phase = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            int b, mb, nb;
            decode(p, t, b, mb, nb);
            if (tile_skipped(p, mb, nb, BN)) continue;
            const int nk = kblocks(p, mb, bk);
            for (int kb = 0; kb < nk; ++kb) {
                mbar_wait(full + 8 * stage, phase);
                std::uint8_t* st = smem + stage * STAGE;
                split_operands(st, st + LOADED, LOADED, tid, 128);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(splitb + 8 * stage);
                if (++stage == kStages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else {
        // Epilogue: warp w reads TMEM lanes 32*(w%4) .. +31 (its subpartition).
        const int lane_base = (warp % 4) * 32;
        int acc = 0;
        std::uint32_t acc_phase = 0;
        const int ob = p.out_dtype == BF16 ? 2 : 4;
        const bool vec_ok = (p.N % 32 == 0) && ((p.ldc * ob) % 16 == 0) && ((p.sc * ob) % 16 == 0) &&
                            ((reinterpret_cast<std::uintptr_t>(p.C) & 15) == 0) &&
                            ((reinterpret_cast<std::uintptr_t>(p.R) & 15) == 0);
        __shared__ int s_reducer;
        for (int u = blockIdx.x; u < units; u += gridDim.x) {
            int t, ks, kb0, kb1, b, mb, nb;
            unit_range(p, u, 0, t, ks, kb0, kb1);
            decode(p, t, b, mb, nb);
            if (tile_skipped(p, mb, nb, BN)) continue;
            const int row = mb * kBM + lane_base + lane;
            const bool row_ok = row < p.M;
            const float alpha = row_alpha(p, row, row_ok);  // before the wait: overlaps this tile's MMAs
            mbar_wait(tfull + 8 * acc, acc_phase);
            tc_fence_after();
            const std::int64_t off = static_cast<std::int64_t>(b) * p.sc + static_cast<std::int64_t>(row) * p.ldc;
            if (SPLIT) {  // sum the tile's K chunks in registers, then store
                float sum[BN];
#pragma unroll
                for (int c = 0; c < BN; ++c) sum[c] = 0.f;
                const int nk = kblocks(p, mb, bk);
                for (int kb0 = 0; kb0 < nk; kb0 += kChunkKB) {
                    if (kb0) mbar_wait(tfull + 8 * acc, acc_phase);
                    tc_fence_after();
                    const std::uint32_t tb = tmem + (static_cast<std::uint32_t>(lane_base) << 16) + acc * BN;
#pragma unroll
                    for (int c0 = 0; c0 < BN; c0 += 32) {
                        std::uint32_t r[32];
                        TN_LD32(tb + c0, r);
                        tc_wait_ld();
#pragma unroll
                        for (int j = 0; j < 32; ++j) sum[c0 + j] += __uint_as_float(r[j]);
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(tempty + 8 * acc);
                    if (++acc == 2) {
                        acc = 0;
                        acc_phase ^= 1;
                    }
                }
#pragma unroll
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    std::uint32_t r[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(sum[c0 + j]);
                    store_chunk(p, r, off, nb * BN + c0, row_ok, vec_ok, alpha);
                }
                continue;
            }
            const std::uint32_t tbase = tmem + (static_cast<std::uint32_t>(lane_base) << 16) + acc * BN;
            if (!SPLIT && p.ksplit > 1) {
                // publish this split's partial, free the accumulator, elect the reducer
                const int r_local = lane_base + lane;
                float* slot = p.ws + (static_cast<std::int64_t>(t) * p.ksplit + ks) * (kBM * BN) +
                              static_cast<std::int64_t>(r_local) * BN;
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    std::uint32_t r[32];
                    TN_LD32(tbase + c0, r);
                    tc_wait_ld();
                    float4* dst = reinterpret_cast<float4*>(slot + c0);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        __stcg(dst + q, make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                                    __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty + 8 * acc);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
                __threadfence();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (threadIdx.x == 64) s_reducer = atomicAdd(p.flags + t, 1u) == static_cast<unsigned>(p.ksplit - 1);
                asm volatile("bar.sync 1, 128;" ::: "memory");
                if (s_reducer) {
                    __threadfence();
                    const float* base = p.ws + static_cast<std::int64_t>(t) * p.ksplit * (kBM * BN) +
                                        static_cast<std::int64_t>(r_local) * BN;
#pragma unroll 1
                    for (int c0 = 0; c0 < BN; c0 += 32) {
                        float a[32];
#pragma unroll
                        for (int q = 0; q < 8; ++q) {
                            const float4 x = __ldcg(reinterpret_cast<const float4*>(base + c0) + q);
                            a[4 * q] = x.x, a[4 * q + 1] = x.y, a[4 * q + 2] = x.z, a[4 * q + 3] = x.w;
                        }
                        for (int sp = 1; sp < p.ksplit; ++sp) {  // split order: deterministic
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const float4 x =
                                    __ldcg(reinterpret_cast<const float4*>(base + sp * (kBM * BN) + c0) + q);
                                a[4 * q] += x.x, a[4 * q + 1] += x.y, a[4 * q + 2] += x.z, a[4 * q + 3] += x.w;
                            }
                        }
                        std::uint32_t r[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(a[j]);
                        store_chunk(p, r, off, nb * BN + c0, row_ok, vec_ok, alpha);
                    }
                    if (threadIdx.x == 64) p.flags[t] = 0u;  // ready for the next launch
                }
                continue;
            }
            if (p.epi == 1) {
                epilogue_swiglu(p, tbase, off, BN / 2, nb * (BN / 2), row_ok, alpha);
            } else if (p.epi == 2) {
                epilogue_qkv_rope(p, tbase, row, nb * BN, BN, row_ok, alpha);
            } else {
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    std::uint32_t r[32];
                    TN_LD32(tbase + c0, r);
                    tc_wait_ld();
                    store_chunk(p, r, off, nb * BN + c0, row_ok, vec_ok, alpha);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty + 8 * acc);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
}


// ---------------------------------------------------------------------------
// 2-CTA variant (cta_group::2): a cluster of two CTAs on a TPC computes a
// 256x256 output tile with M=256 MMAs issued by the leader. Each CTA stages
// half of A (its 128 rows) and half of B (128 rows) per 128-byte K block, so
// per-SM L2->SMEM traffic per FLOP drops by 1.5x vs the 1-CTA 128x256 tile
// (which is L2-bandwidth bound: ~96 B/clk/SM at full MMA rate).
//   full[s]   leader only: expect_tx(64 KB) by the leader, complete_tx from
//             both CTAs' TMA (.cta_group::2 loads signal the leader barrier)
//   empty[s]  per CTA: multicast tcgen05.commit from the leader MMA
//   tfull[a]  per CTA: multicast commit after the last K block of a tile
//   tempty[a] leader only: 8 arrivals (4 epilogue warps x 2 CTAs)
constexpr int kStages2 = 6;

__device__ __forceinline__ long long sk_begin(const Params& p, int q, int npairs) {
    return p.sk_total * q / npairs;
}
// Pair owning stream-K block `it`: largest q with sk_begin(q) <= it.
__device__ __forceinline__ int sk_owner(const Params& p, long long it, int npairs) {
    int q = static_cast<int>(it * npairs / max(1LL, p.sk_total));
    while (q + 1 < npairs && sk_begin(p, q + 1, npairs) <= it) ++q;
    while (q > 0 && sk_begin(p, q, npairs) > it) --q;
    return q;
}
// B rows staged by CTA `rank` for slice k of s of N tile nb (256 accumulator
// columns; each CTA of the pair stages half of the slice's B rows). A plain
// tile's slice is GEMM columns [nb*256 + k*256/s, +256/s). A SwiGLU tile
// (128 gate rows then the matching 128 up rows) keeps the pairing: rank 0
// stages the slice's gate rows and rank 1 the matching up rows, so the
// accumulator holds [gate | up] halves of 128/s columns each.
__device__ __forceinline__ int slice_brow(const Params& p, int nb, int k, int s, int rank) {
    const int w = 256 / s;
    return p.epi == 1 ? nb * 256 + rank * 128 + k * (w / 2) : nb * 256 + k * w + rank * (w / 2);
}

// Visits this pair's work as (tile, N-slice, K-block range) segments: its
// round-robin data-parallel tiles, then its share of the sliced tail, then
// its contiguous slice of the stream-K blocks. f(b, mb, nb, k, s, kb0, kb1, nk, it0).
template <class F>
__device__ __forceinline__ void for_each_segment(const Params& p, int pair, int npairs, int bk, F&& f) {
    constexpr int BN = 256, BM2 = 256;
    for (int t = pair; t < p.dp_tiles; t += npairs) {
        int b, mb, nb;
        decode(p, t, b, mb, nb);
        if (p.causal == 1 && nb * BN > mb * BM2 + BM2 - 1) continue;
        int nk = (p.K + bk - 1) / bk;
        if (p.causal == 2) nk = min(nk, ((mb + 1) * BM2 + bk - 1) / bk);
        f(b, mb, nb, 0, 1, 0, nk, nk, 0LL);
    }
    for (int u = pair; u < p.tail_units; u += npairs) {  // causal == 0 only
        int b, mb, nb;
        decode(p, p.dp_tiles + u / p.tail_split, b, mb, nb);
        const int nk = (p.K + bk - 1) / bk;
        f(b, mb, nb, u % p.tail_split, p.tail_split, 0, nk, nk, 0LL);
    }
    if (p.sk_total <= 0) return;
    const long long end = sk_begin(p, pair + 1, npairs);
    for (long long it = sk_begin(p, pair, npairs); it < end;) {
        const int tt = p.dp_tiles + static_cast<int>(it / p.sk_nk);
        const int kb0 = static_cast<int>(it % p.sk_nk);
        const int kb1 = static_cast<int>(min(static_cast<long long>(p.sk_nk), kb0 + (end - it)));
        int b, mb, nb;
        decode(p, tt, b, mb, nb);
        f(b, mb, nb, 0, 1, kb0, kb1, p.sk_nk, it - kb0);
        it += kb1 - kb0;
    }
}
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_kernel_2sm(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                    const __grid_constant__ CUtensorMap tbh, const __grid_constant__ CUtensorMap tbq,
                    const __grid_constant__ CUtensorMap tc, const Params p) {
    constexpr int HALF = 128;                  // rows of A and of B staged per CTA
    constexpr int A_BYTES = HALF * kAtom;      // 16 KB
    constexpr int STAGE = 2 * A_BYTES;         // 32 KB per CTA
    constexpr int BN = 256, BM2 = 256;
    constexpr std::uint32_t TMEM_COLS = 512;   // 2 x 256 fp32 accumulators

    extern __shared__ std::uint8_t smem_raw[];
    const std::uint32_t raw = smem_u32(smem_raw);
    const std::uint32_t pad = ((raw + 1023) & ~1023u) - raw;
    std::uint8_t* smem = smem_raw + pad;
    const std::uint32_t sbase = raw + pad;
    const std::uint32_t stg = sbase + kStages2 * STAGE;  // 4 epilogue warps x kStgWarp
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + kStages2 * STAGE + 4 * kStgWarp);
    const std::uint32_t full = smem_u32(bars), empty = full + 8 * kStages2;
    const std::uint32_t tfull = empty + 8 * kStages2, tempty = tfull + 16;
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 2 * kStages2 + 4);

    pdl_trigger();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const std::uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int bk = kAtom / p.in_bytes;
    const bool tf32 = p.in_bytes == 4;
    const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&ta)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tb)) : "memory");
        if (p.tail_units > 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(p.tail_split == 2 ? &tbh : &tbq))
                         : "memory");
        }
        for (int s = 0; s < kStages2; ++s) {
            mbar_init(full + 8 * s, 1);
            mbar_init(empty + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull + 8 * a, 1);
            mbar_init(tempty + 8 * a, 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    pdl_wait();  // previous kernel complete: its outputs are visible, its inputs may be overwritten
    const std::uint32_t tmem = *tmem_slot;
    const std::uint32_t full_leader0 = mapa(full, 0);
    const std::uint32_t tempty_leader0 = mapa(tempty, 0);

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            std::uint32_t phase = 0;
            for_each_segment(p, pair, npairs, bk, [&](int b, int mb, int nb, int k, int sl, int kb0, int kb1, int, long long) {
                const int brows = BN / 2 / sl;  // B rows staged per CTA
                const CUtensorMap* mb_map = sl == 1 ? &tb : sl == 2 ? &tbh : &tbq;
                const int brow = slice_brow(p, nb, k, sl, static_cast<int>(rank));
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(empty + 8 * stage, phase ^ 1);
                    const std::uint32_t fb = full_leader0 + 8 * stage;
                    if (leader) mbar_expect_tx(full + 8 * stage, 2 * (A_BYTES + brows * kAtom));
                    const std::uint32_t sa = sbase + stage * STAGE;
                    load_operand_2sm(sa, &ta, kb * bk, mb * BM2 + rank * HALF, HALF, p.a_batched ? b : 0, fb, p.a_mn);
                    load_operand_2sm(sa + A_BYTES, mb_map, kb * bk, brow, brows, p.b_batched ? b : 0, fb, p.b_mn);
                    if (++stage == kStages2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            });
        }
    } else if (warp == 1) {
        if (leader) {  // whole warp: one elected lane issues (tc_mma_2sm)
            const std::uint32_t fmt = tf32 ? 2u : 1u;
            int stage = 0, acc = 0;
            std::uint32_t phase = 0, acc_phase = 0;
            for_each_segment(p, pair, npairs, bk, [&](int, int, int, int, int sl, int kb0, int kb1, int, long long) {
                const std::uint32_t idesc = make_idesc(fmt, BM2, BN / sl) | (static_cast<std::uint32_t>(p.a_mn) << 15) |
                                            (static_cast<std::uint32_t>(p.b_mn) << 16);
                const int as = op_kstep(p.a_mn), bs = op_kstep(p.b_mn);
                mbar_wait(tempty + 8 * acc, acc_phase ^ 1);
                tc_fence_after();
                const std::uint32_t d = tmem + acc * BN;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(full + 8 * stage, phase);
                    tc_fence_after();
                    const std::uint32_t sa = sbase + stage * STAGE;
                    const std::uint64_t ad = op_desc(sa, p.a_mn), bd = op_desc(sa + A_BYTES, p.b_mn);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        tc_mma_2sm(d, ad + as * k, bd + bs * k, idesc, (kb != kb0) | (k != 0), tf32);
                    tc_commit_2sm(empty + 8 * stage);
                    if (++stage == kStages2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit_2sm(tfull + 8 * acc);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            });
        }
    } else {
        const int lane_base = (warp % 4) * 32;
        int acc = 0;
        std::uint32_t acc_phase = 0;
        const int ob = p.out_dtype == BF16 ? 2 : 4;
        const bool vec_ok = (p.N % 32 == 0) && ((p.ldc * ob) % 16 == 0) && ((p.sc * ob) % 16 == 0) &&
                            ((reinterpret_cast<std::uintptr_t>(p.C) & 15) == 0) &&
                            ((reinterpret_cast<std::uintptr_t>(p.R) & 15) == 0);
        const int r_local = lane_base + lane;
        Stager st{stg + static_cast<std::uint32_t>(warp - 2) * kStgWarp, 0};
        for_each_segment(p, pair, npairs, bk, [&](int b, int mb, int nb, int k, int sl, int kb0, int kb1, int nk, long long tile_it0) {
            const int w = BN / sl;      // accumulator columns of this segment
            const int n0 = nb * BN + k * w;  // first GEMM column (plain / qkv)
            const int row0 = mb * BM2 + static_cast<int>(rank) * HALF + lane_base;
            const int row = row0 + lane;
            const bool row_ok = row < p.M;
            const float alpha = row_alpha(p, row, row_ok);  // before the wait: overlaps this tile's MMAs
            const std::int64_t off = static_cast<std::int64_t>(b) * p.sc + static_cast<std::int64_t>(row) * p.ldc;
            if (kb0 == 0) prefetch_residual(p, off, n0, w, row_ok);
            mbar_wait(tfull + 8 * acc, acc_phase);
            tc_fence_after();
            const std::uint32_t tbase = tmem + (static_cast<std::uint32_t>(lane_base) << 16) + acc * BN;
            if (kb0 > 0) {
                // Stream-K contributor (the first segment of this pair's
                // slice, a tile's later K blocks): publish the partial.
                float* slot = p.ws + ((static_cast<std::int64_t>(pair) * 2 + rank) * HALF + r_local) * BN;
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    std::uint32_t r[32];
                    TN_LD32(tbase + c0, r);
                    tc_wait_ld();
                    float4* dst = reinterpret_cast<float4*>(slot + c0);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        __stcg(dst + q, make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                                    __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3])));
                }
                __threadfence();
                epi_bar();
                if (threadIdx.x == 64) {
                    __threadfence();
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.flags + pair * 2 + rank), "r"(p.epoch)
                                 : "memory");
                }
            } else if (kb1 < nk) {
                // Stream-K finisher: owns the tile's first K blocks, which
                // are the last segment of its slice, so the later pairs'
                // partials (their first segments) are published by now.
                const int q1 = sk_owner(p, tile_it0 + nk - 1, npairs);
                if (threadIdx.x == 64) {
                    for (int q = pair + 1; q <= q1; ++q) {
                        if (sk_begin(p, q, npairs) == sk_begin(p, q + 1, npairs)) continue;
                        const unsigned* f = p.flags + q * 2 + rank;
                        unsigned v;
                        do {
                            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
                        } while (v != p.epoch);
                    }
                }
                epi_bar();
#pragma unroll 1
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    std::uint32_t r[32];
                    TN_LD32(tbase + c0, r);
                    tc_wait_ld();
                    for (int q = pair + 1; q <= q1; ++q) {
                        if (sk_begin(p, q, npairs) == sk_begin(p, q + 1, npairs)) continue;
                        const float4* src = reinterpret_cast<const float4*>(
                            p.ws + ((static_cast<std::int64_t>(q) * 2 + rank) * HALF + r_local) * BN + c0);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const float4 x = __ldcg(src + j);
                            r[4 * j] = __float_as_uint(__uint_as_float(r[4 * j]) + x.x);
                            r[4 * j + 1] = __float_as_uint(__uint_as_float(r[4 * j + 1]) + x.y);
                            r[4 * j + 2] = __float_as_uint(__uint_as_float(r[4 * j + 2]) + x.z);
                            r[4 * j + 3] = __float_as_uint(__uint_as_float(r[4 * j + 3]) + x.w);
                        }
                    }
                    if (p.epi == 0) store_chunk(p, r, off, nb * BN + c0, row_ok, vec_ok, alpha);
                    else TN_ST32(tbase + c0, r);  // summed tile back to TMEM for the fused epilogue
                }
                if (p.epi != 0) {
                    tc_wait_st();
                    if (p.epi == 1) epilogue_swiglu(p, tbase, off, BN / 2, nb * (BN / 2), row_ok, alpha);
                    else epilogue_qkv_rope(p, tbase, row, n0, BN, row_ok, alpha);
                }
            } else if (p.epi == 1) {  // [gate | up] halves of w/2 columns -> output columns nb*128 + k*w/2
                if (p.tma_c) epilogue_swiglu_tma(p, &tc, st, tbase, row0, w / 2, nb * (BN / 2) + k * (w / 2), b, alpha);
                else epilogue_swiglu(p, tbase, off, w / 2, nb * (BN / 2) + k * (w / 2), row_ok, alpha);
            } else if (p.epi == 2) {
                epilogue_qkv_rope(p, tbase, row, n0, w, row_ok, alpha);
            } else if (p.tma_c) {
                epilogue_plain_tma(p, &tc, st, tbase, off, row0, n0, w, b, row_ok, alpha);
            } else {
#pragma unroll 1
                for (int c0 = 0; c0 < w; c0 += 32) {
                    std::uint32_t r[32];
                    TN_LD32(tbase + c0, r);
                    tc_wait_ld();
                    store_chunk(p, r, off, n0 + c0, row_ok, vec_ok, alpha);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader0 + 8 * acc);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        });
        if (lane == 0) bulk_wait_all();  // staged TMA stores complete before the CTA exits
    }

    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
}

// ---------------------------------------------------------------------------
// Wide CTA-pair variant: a 512x256 output tile per pair (each CTA owns 256
// rows = two 128-row M-halves, one M=256 MMA per half per K step, both
// accumulators filling the 512 TMEM columns). Per 64-element K block a CTA
// receives 48 KB for 2x256x256x64 MACs — 25% fewer bytes per FLOP than the
// 256x256 pair tile, whose L2->SM operand stream (64 B/clk/SM) caps the
// tensor pipe near 2/3 busy. With no spare TMEM for a second accumulator,
// the next tile's half-0 MMAs start as soon as the epilogue has drained half
// 0, and half-1 MMAs are deferred (holding their stages) until half 1 drains.
// Two epilogue warpgroups (warps 2-5: half 0, warps 6-9: half 1) drain the
// halves concurrently, so the accumulator is free again after one half's
// drain time rather than two.
constexpr int kStagesW = 4;
constexpr int kThreadsW = 32 * 10;

// Plain epilogue of one 128-row x BN accumulator slab: two 32-column TMEM
// loads in flight per wait.
__device__ __forceinline__ void epilogue_plain(const Params& p, std::uint32_t tbase, std::int64_t off, int n0, int width,
                                               bool row_ok, bool vec_ok, float alpha) {
#pragma unroll 1
    for (int c0 = 0; c0 < width; c0 += 64) {
        std::uint32_t r0[32], r1[32];
        TN_LD32(tbase + c0, r0);
        TN_LD32(tbase + c0 + 32, r1);
        tc_wait_ld();
        store_chunk(p, r0, off, n0 + c0, row_ok, vec_ok, alpha);
        store_chunk(p, r1, off, n0 + c0 + 32, row_ok, vec_ok, alpha);
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreadsW, 1)
    gemm_kernel_2sm_w(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                      const __grid_constant__ CUtensorMap tbh, const __grid_constant__ CUtensorMap tbq,
                      const __grid_constant__ CUtensorMap tc, const Params p) {
    constexpr int HALF = 128;
    constexpr int A_SUB = HALF * kAtom;        // 16 KB: one 128-row A sub-tile
    constexpr int STAGE = 3 * A_SUB;           // A half 0, A half 1, B (48 KB per CTA)
    constexpr int BN = 256, BMW = 512;
    constexpr std::uint32_t TMEM_COLS = 512;   // half h accumulates in columns [256h, 256h+256)

    extern __shared__ std::uint8_t smem_raw[];
    const std::uint32_t raw = smem_u32(smem_raw);
    const std::uint32_t pad = ((raw + 1023) & ~1023u) - raw;
    std::uint8_t* smem = smem_raw + pad;
    const std::uint32_t sbase = raw + pad;
    const std::uint32_t stg = sbase + kStagesW * STAGE;  // 8 epilogue warps x kStgWarp
    std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(smem + kStagesW * STAGE + 8 * kStgWarp);
    const std::uint32_t full = smem_u32(bars), empty = full + 8 * kStagesW;
    const std::uint32_t tfull = empty + 8 * kStagesW, tempty = tfull + 8;  // tempty[2]
    std::uint32_t* tmem_slot = reinterpret_cast<std::uint32_t*>(bars + 2 * kStagesW + 3);

    pdl_trigger();
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const std::uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int bk = kAtom / p.in_bytes;
    const bool tf32 = p.in_bytes == 4;
    const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
    auto tile_nk = [&](int mb) {
        int nk = (p.K + bk - 1) / bk;
        if (p.causal == 2) nk = min(nk, ((mb + 1) * BMW + bk - 1) / bk);
        return nk;
    };
    auto skipped = [&](int mb, int nb) { return p.causal == 1 && nb * BN > mb * BMW + BMW - 1; };
    // This pair's work: round-robin full tiles, then its share of the sliced
    // tail (slice k of sl of tile nb, see slice_brow). f(b, mb, nb, k, sl).
    auto for_each_tile = [&](auto&& f) {
        for (int t = pair; t < p.dp_tiles; t += npairs) {
            int b, mb, nb;
            decode(p, t, b, mb, nb);
            if (!skipped(mb, nb)) f(b, mb, nb, 0, 1);
        }
        for (int u = pair; u < p.tail_units; u += npairs) {
            int b, mb, nb;
            decode(p, p.dp_tiles + u / p.tail_split, b, mb, nb);
            f(b, mb, nb, u % p.tail_split, p.tail_split);
        }
    };

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&ta)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(&tb)) : "memory");
        if (p.tail_units > 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<std::uint64_t>(p.tail_split == 2 ? &tbh : &tbq))
                         : "memory");
        }
        for (int s = 0; s < kStagesW; ++s) {
            mbar_init(full + 8 * s, 1);
            mbar_init(empty + 8 * s, 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 8);
        mbar_init(tempty + 8, 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    pdl_wait();  // previous kernel complete: its outputs are visible, its inputs may be overwritten
    const std::uint32_t tmem = *tmem_slot;
    const std::uint32_t full_leader0 = mapa(full, 0);
    const std::uint32_t tempty_leader0 = mapa(tempty, 0);

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            std::uint32_t phase = 0;
            for_each_tile([&](int b, int mb, int nb, int k, int sl) {
                const int nk = tile_nk(mb);
                const CUtensorMap* bmap = sl == 1 ? &tb : sl == 2 ? &tbh : &tbq;
                const int brow = slice_brow(p, nb, k, sl, static_cast<int>(rank));
                const int brows = BN / 2 / sl;  // B rows staged per CTA
                const std::uint32_t tx = 2 * (2 * A_SUB + brows * kAtom);
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(empty + 8 * stage, phase ^ 1);
                    const std::uint32_t fb = full_leader0 + 8 * stage;
                    if (leader) mbar_expect_tx(full + 8 * stage, tx);
                    const std::uint32_t sa = sbase + stage * STAGE;
                    const int ab = p.a_batched ? b : 0;
                    load_operand_2sm(sa, &ta, kb * bk, mb * BMW + rank * HALF, HALF, ab, fb, p.a_mn);
                    load_operand_2sm(sa + A_SUB, &ta, kb * bk, mb * BMW + 256 + rank * HALF, HALF, ab, fb, p.a_mn);
                    load_operand_2sm(sa + 2 * A_SUB, bmap, kb * bk, brow, brows, p.b_batched ? b : 0, fb, p.b_mn);
                    if (++stage == kStagesW) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            });
        }
    } else if (warp == 1) {
        if (leader) {  // whole warp: one elected lane issues (tc_mma_2sm)
            const std::uint32_t fmt = tf32 ? 2u : 1u;
            int stage = 0;
            std::uint32_t phase = 0, tphase = 0;
            int defer_stage[kStagesW];
            for_each_tile([&](int, int mb, int, int, int sl) {
                const int nk = tile_nk(mb);
                const std::uint32_t idesc = make_idesc(fmt, 256, BN / sl) | (static_cast<std::uint32_t>(p.a_mn) << 15) |
                                            (static_cast<std::uint32_t>(p.b_mn) << 16);
                const int as = op_kstep(p.a_mn), bs = op_kstep(p.b_mn);
                mbar_wait(tempty, tphase ^ 1);  // half 0 drained by the previous tile's epilogue
                tc_fence_after();
                bool h1_ready = false;
                int ndefer = 0, h1_done = 0;  // half-1 K blocks issued so far
                auto issue_h1 = [&](int st) {
                    const std::uint32_t sa = sbase + st * STAGE;
                    const std::uint64_t ad = op_desc(sa + A_SUB, p.a_mn), bd = op_desc(sa + 2 * A_SUB, p.b_mn);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        tc_mma_2sm(tmem + 256, ad + as * k, bd + bs * k, idesc, (h1_done | k) != 0, tf32);
                    tc_commit_2sm(empty + 8 * st);
                    ++h1_done;
                };
                for (int kb = 0; kb < nk; ++kb) {
                    mbar_wait(full + 8 * stage, phase);
                    tc_fence_after();
                    const std::uint32_t sa = sbase + stage * STAGE;
                    const std::uint64_t ad = op_desc(sa, p.a_mn), bd = op_desc(sa + 2 * A_SUB, p.b_mn);
#pragma unroll
                    for (int k = 0; k < 4; ++k) tc_mma_2sm(tmem, ad + as * k, bd + bs * k, idesc, (kb | k) != 0, tf32);
                    if (!h1_ready) {
                        defer_stage[ndefer++] = stage;
                        const bool drained = __shfl_sync(0xffffffffu, mbar_test(tempty + 8, tphase ^ 1), 0);
                        if (ndefer == kStagesW || kb == nk - 1 || drained) {
                            mbar_wait(tempty + 8, tphase ^ 1);
                            tc_fence_after();
                            h1_ready = true;
                            for (int i = 0; i < ndefer; ++i) issue_h1(defer_stage[i]);
                        }
                    } else {
                        issue_h1(stage);
                    }
                    if (++stage == kStagesW) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit_2sm(tfull);
                tphase ^= 1;
            });
        }
    } else {
        const int lane_base = (warp % 4) * 32;
        const int h = (warp - 2) / 4;  // the accumulator half this warpgroup drains
        Stager st{stg + static_cast<std::uint32_t>(warp - 2) * kStgWarp, 0};
        std::uint32_t tphase = 0;
        const int ob = p.out_dtype == BF16 ? 2 : 4;
        const bool vec_ok = (p.N % 32 == 0) && ((p.ldc * ob) % 16 == 0) && ((p.sc * ob) % 16 == 0) &&
                            ((reinterpret_cast<std::uintptr_t>(p.C) & 15) == 0) &&
                            ((reinterpret_cast<std::uintptr_t>(p.R) & 15) == 0);
        for_each_tile([&](int b, int mb, int nb, int k, int sl) {
            const int w = BN / sl;
            const int row = mb * BMW + h * 256 + static_cast<int>(rank) * HALF + lane_base + lane;
            const bool row_ok = row < p.M;
            const float alpha = row_alpha(p, row, row_ok);  // before the wait: overlaps this tile's MMAs
            const std::int64_t off = static_cast<std::int64_t>(b) * p.sc + static_cast<std::int64_t>(row) * p.ldc;
            prefetch_residual(p, off, nb * BN + k * w, w, row_ok);
            mbar_wait(tfull, tphase);
            tc_fence_after();
            const std::uint32_t tbase = tmem + (static_cast<std::uint32_t>(lane_base) << 16) + h * 256;
            const int row0 = row - lane;
            if (p.epi == 1) {
                if (p.tma_c) epilogue_swiglu_tma(p, &tc, st, tbase, row0, w / 2, nb * (BN / 2) + k * (w / 2), b, alpha);
                else epilogue_swiglu(p, tbase, off, w / 2, nb * (BN / 2) + k * (w / 2), row_ok, alpha);
            } else if (p.epi == 2) {
                epilogue_qkv_rope(p, tbase, row, nb * BN + k * w, w, row_ok, alpha);
            } else if (p.tma_c) {
                epilogue_plain_tma(p, &tc, st, tbase, off, row0, nb * BN + k * w, w, b, row_ok, alpha);
            } else {
                epilogue_plain(p, tbase, off, nb * BN + k * w, w, row_ok, vec_ok, alpha);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty_leader0 + 8 * h);
            tphase ^= 1;
        });
        if (lane == 0) bulk_wait_all();
    }

    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS) : "memory");
}

// --- SIMT fallback: one warp per output element, fp32 accumulate in K order.
// Used for tiny M (GEMV-like last-token heads) or shapes TMA cannot describe.
__global__ void gemm_simt_kernel(GemmArgs a) {
    pdl_trigger();
    pdl_wait();
    const std::int64_t gw = (static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    const int Nout = a.epi == 1 ? a.N / 2 : a.N;
    const std::int64_t total = static_cast<std::int64_t>(a.batch) * a.M * Nout;
    if (gw >= total) return;
    const int nout = static_cast<int>(gw % Nout);
    const int m = static_cast<int>((gw / Nout) % a.M);
    const int b = static_cast<int>(gw / (static_cast<std::int64_t>(Nout) * a.M));
    // swiglu: gate column 256*(j/128) + j%128, up column + 128
    const int n = a.epi == 1 ? 256 * (nout / 128) + nout % 128 : nout;
    if (a.causal == 1 && n > m) return;
    int kend = a.K;
    if (a.causal == 2) kend = min(kend, m + 1);
    float alpha = a.alpha;
    if (a.rs_P) {
        float ss = 0.f;
        for (int c = 0; c < a.rs_chunks; ++c) ss += a.rs_P[static_cast<std::int64_t>(a.rs_row0 + m) * a.rs_ld + c];
        alpha *= rsqrtf(ss * a.rs_inv_dim + a.rs_eps);
    }
    auto dot = [&](int col) {
        float acc = 0.f;
        if (a.a_mn || a.b_mn) {  // MN-major operand(s): element (m|n, k) at k * ld + m|n
            const std::int64_t as = a.a_mn ? a.lda : 1, am = a.a_mn ? 1 : a.lda;
            const std::int64_t bs = a.b_mn ? a.ldb : 1, bn = a.b_mn ? 1 : a.ldb;
            const std::int64_t a0 = b * a.sa + static_cast<std::int64_t>(m) * am, b0 = b * a.sb + static_cast<std::int64_t>(col) * bn;
            if (a.in_dtype == BF16) {
                const __nv_bfloat16* A = static_cast<const __nv_bfloat16*>(a.A);
                const __nv_bfloat16* B = static_cast<const __nv_bfloat16*>(a.B);
                for (int k = lane; k < kend; k += 32) acc += __bfloat162float(A[a0 + k * as]) * __bfloat162float(B[b0 + k * bs]);
            } else {
                const float* A = static_cast<const float*>(a.A);
                const float* B = static_cast<const float*>(a.B);
                for (int k = lane; k < kend; k += 32) acc += A[a0 + k * as] * B[b0 + k * bs];
            }
        } else if (a.in_dtype == BF16) {
            const __nv_bfloat16* A = static_cast<const __nv_bfloat16*>(a.A) + b * a.sa + static_cast<std::int64_t>(m) * a.lda;
            const __nv_bfloat16* B = static_cast<const __nv_bfloat16*>(a.B) + b * a.sb + static_cast<std::int64_t>(col) * a.ldb;
            const bool vec = ((reinterpret_cast<std::uintptr_t>(A) | reinterpret_cast<std::uintptr_t>(B)) & 15) == 0;
            int k0 = 0;
            if (vec) {  // 16-byte loads: lane covers 8 consecutive k per 256-wide step (GEMV heads are HBM-bound)
                const int kv = kend / 256 * 256;
                for (int k = lane * 8; k < kv; k += 256) {
                    const uint4 x = __ldg(reinterpret_cast<const uint4*>(A + k));
                    const uint4 y = __ldcs(reinterpret_cast<const uint4*>(B + k));  // streamed once
                    const __nv_bfloat162* xh = reinterpret_cast<const __nv_bfloat162*>(&x);
                    const __nv_bfloat162* yh = reinterpret_cast<const __nv_bfloat162*>(&y);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float2 xf = __bfloat1622float2(xh[i]), yf = __bfloat1622float2(yh[i]);
                        acc = fmaf(xf.x, yf.x, acc);
                        acc = fmaf(xf.y, yf.y, acc);
                    }
                }
                k0 = kv;
            }
            for (int k = k0 + lane; k < kend; k += 32) acc += __bfloat162float(A[k]) * __bfloat162float(B[k]);
        } else {
            const float* A = static_cast<const float*>(a.A) + b * a.sa + static_cast<std::int64_t>(m) * a.lda;
            const float* B = static_cast<const float*>(a.B) + b * a.sb + static_cast<std::int64_t>(col) * a.ldb;
            for (int k = lane; k < kend; k += 32) acc += A[k] * B[k];
        }
#pragma unroll
        for (int o = 16; o > 0; o /= 2) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        return acc * alpha;
    };
    float acc = dot(n);
    if (a.epi == 1) {
        const float up = dot(n + 128);
        acc = acc / (1.0f + __expf(-acc)) * up;
    }
    if (lane != 0) return;
    const std::int64_t off = b * a.sc + static_cast<std::int64_t>(m) * a.ldc + nout;
    if (a.out_dtype == BF16) {
        if (a.R) acc += __bfloat162float(static_cast<const __nv_bfloat16*>(a.R)[off]);
        static_cast<__nv_bfloat16*>(a.C)[off] = __float2bfloat16_rn(acc);
    } else {
        if (a.R) acc += static_cast<const float*>(a.R)[off];
        static_cast<float*>(a.C)[off] = acc;
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

bool encode(CUtensorMap* map, const void* base, int esize, std::int64_t K, std::int64_t rows, std::int64_t ld,
            int batch, std::int64_t bstride, int box_rows) {
    return encode_tma_3d(map, base, esize, K, rows, ld, batch, bstride, kAtom / esize, box_rows);
}

}  // namespace

bool encode_tma_3d(CUtensorMap* map, const void* base, int esize, std::int64_t inner, std::int64_t rows,
                   std::int64_t ld, int batch, std::int64_t bstride, int box_inner, int box_rows) {
    return encode_tma_3d_swz(map, base, esize, inner, rows, ld, batch, bstride, box_inner, box_rows,
                             CU_TENSOR_MAP_SWIZZLE_128B);
}

bool encode_tma_3d_swz(CUtensorMap* map, const void* base, int esize, std::int64_t inner, std::int64_t rows,
                       std::int64_t ld, int batch, std::int64_t bstride, int box_inner, int box_rows,
                       CUtensorMapSwizzle swz) {
    EncodeFn fn = get_encode();
    if (!fn) return false;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(batch)};
    std::int64_t bs = batch > 1 ? bstride : rows * ld;
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld * esize), static_cast<cuuint64_t>(bs * esize)};
    cuuint32_t box[3] = {static_cast<cuuint32_t>(box_inner), static_cast<cuuint32_t>(box_rows), 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, esize == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                    const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

namespace {

template <int BN, bool SPLIT = false>
int smem_bytes() {
    return stages_1cta<BN, SPLIT>() * (SPLIT ? 2 : 1) * (kBM + BN) * kAtom + 256 + 1024;
}
int smem_bytes_2sm() { return kStages2 * 2 * 128 * kAtom + 4 * kStgWarp + 256 + 1024; }
int smem_bytes_2sm_w() { return kStagesW * 3 * 128 * kAtom + 8 * kStgWarp + 256 + 1024; }

}  // namespace

double gemm_flops(const GemmArgs& a) {
    double mnk = 2.0 * a.M * static_cast<double>(a.N) * a.K * a.batch;
    if (a.causal) mnk *= 0.5 * (1.0 + 1.0 / std::max(1, a.M));  // lower triangle incl. diagonal
    return mnk;
}

cudaError_t gemm_prepare(const GemmArgs& a, GemmPlan* plan, int num_sms) {
    plan->args = a;
    const int es = dtype_size(a.in_dtype);
    auto al16 = [](const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15) == 0; };
    const bool split = a.split && a.in_dtype == F32;
    // 3xTF32 runs on the 1-CTA kernel (the split doubles the staged bytes; the
    // chunked epilogue keeps a BN-float row sum in registers), 128-column tiles when they still fill every SM (shared-memory traffic
    // per FLOP drops by a third: 4096^3 137.5 vs 93 TF/s), else 64 (1024^3: 54.9 vs 43.5)
    const long long tiles128 = static_cast<long long>(a.batch) * ((a.M + kBM - 1) / kBM) * ((a.N + 127) / 128);
    const int bn = split ? (a.N >= 128 && tiles128 >= num_sms ? 128 : 64) : a.N >= 256 ? 256 : a.N >= 128 ? 128 : 64;
    const bool two_sm = !split && a.M >= 256 && a.N >= 256;
    if (a.split && a.in_dtype != F32) return cudaErrorInvalidValue;
    const bool mn = a.a_mn || a.b_mn;
    bool ok = (!mn || (a.in_dtype == BF16 && !split && a.epi == 0 && !a.no_P)) &&
              (!split || (a.epi == 0 && !a.no_P && !a.rs_P)) &&
              (a.epi == 0 || (a.N % 256 == 0 && bn == 256 && a.R == nullptr)) &&
              (a.epi != 2 || (a.batch == 1 && (reinterpret_cast<std::uintptr_t>(a.rope) & 15) == 0)) && a.M >= kBM && a.N >= bn && a.K * es >= kAtom && al16(a.A) && al16(a.B) && (a.lda * es) % 16 == 0 &&
              (a.ldb * es) % 16 == 0 && (a.batch == 1 || ((a.sa * es) % 16 == 0 && (a.sb * es) % 16 == 0)) &&
              (a.in_dtype == BF16 || a.in_dtype == F32);
    if (ok) {
        const bool ab = a.batch > 1 && a.sa != 0, bb = a.batch > 1 && a.sb != 0;
        // MN-major operands: [K rows, M|N contiguous] maps with 64x64 boxes (load_operand)
        ok = (a.a_mn ? encode_tma_3d(&plan->ta, a.A, es, a.M, a.K, a.lda, ab ? a.batch : 1, a.sa, 64, 64)
                     : encode(&plan->ta, a.A, es, a.K, a.M, a.lda, ab ? a.batch : 1, a.sa, kBM)) &&
             (a.b_mn ? encode_tma_3d(&plan->tb, a.B, es, a.N, a.K, a.ldb, bb ? a.batch : 1, a.sb, 64, 64)
                     : encode(&plan->tb, a.B, es, a.K, a.N, a.ldb, bb ? a.batch : 1, a.sb, two_sm ? 128 : bn));
        plan->tbh_ok = ok && two_sm && !a.b_mn && encode(&plan->tbh, a.B, es, a.K, a.N, a.ldb, bb ? a.batch : 1, a.sb, 64) &&
                       encode(&plan->tbq, a.B, es, a.K, a.N, a.ldb, bb ? a.batch : 1, a.sb, 32);
        // C for the TMA-store epilogue: {64 B x 32 rows} boxes, SWIZZLE_64B
        const int oes = dtype_size(a.out_dtype);
        const int n_out = a.epi == 1 ? a.N / 2 : a.N;
        const bool cb = a.batch > 1;
        // (fused-norm producers: batch index 1 of the map is the h block after C)
        const bool no = a.no_P != nullptr;
        plan->tc_ok = ok && two_sm && (a.epi == 0 || a.epi == 1) && (a.out_dtype == BF16 || a.out_dtype == F32) &&
                      al16(a.C) && (a.ldc * oes) % 16 == 0 && (!cb || (a.sc * oes) % 16 == 0) &&
                      (a.R == nullptr || al16(a.R)) && n_out % 32 == 0 &&
                      encode_tma_3d_swz(&plan->tc, a.C, oes, n_out, a.M, a.ldc, no ? 2 : cb ? a.batch : 1,
                                        no ? static_cast<std::int64_t>(a.M) * a.ldc : a.sc, 64 / oes, 32,
                                        CU_TENSOR_MAP_SWIZZLE_64B);
    }
    plan->path = ok ? (two_sm ? 2 : 0) : 1;
    plan->bn = bn;
    int tile = a.tile;
    if (tile == 0) {  // TN_GEMM_TILE=narrow|wide overrides the automatic choice (tuning experiments)
        static const char* env = std::getenv("TN_GEMM_TILE");
        if (env && std::strcmp(env, "narrow") == 0) tile = 1;
        if (env && std::strcmp(env, "wide") == 0) tile = 2;
    }
    if (plan->path == 2 && tile == 2) plan->path = 3;
    if (a.no_P) {  // fused-norm producer: only the TMA-store epilogue of the CTA-pair kernels writes x | h | P
        if (!(plan->path == 2 || plan->path == 3) || !plan->tc_ok || a.epi != 0 || a.R == nullptr ||
            a.out_dtype != BF16 || a.batch != 1 || a.causal != 0 || a.N % 32 != 0 || !al16(a.no_g) || tile == 3)
            return cudaErrorNotSupported;
    }
    // Tail of the last, partial wave of pairs: its tiles are split into
    // sl in {1, 2, 4} N-slices (slice_brow) so that the tail costs
    // ceil(rem * sl / P) / sl tile-times. SwiGLU slices keep gate/up pairs;
    // the QKV+RoPE epilogue needs whole heads (sl <= 2).
    const int P = std::max(1, num_sms / 2);
    // Wide tiles slice at most 2 ways: a 512x64 slice still stages both
    // 256-row A halves, so it is operand-bound at ~3/4 of a full tile-time.
    auto tail_plan = [&](long long T, int* split, bool wide) {
        const long long rem = T >= P ? T % P : T;
        double best = rem == 0 ? 0.0 : 1.0;
        *split = 1;
        if (rem > 0 && a.causal == 0 && plan->tbh_ok) {
            for (int sl = 2; sl <= (a.epi == 2 || wide ? 2 : 4); sl *= 2) {
                const double t = static_cast<double>((rem * sl + P - 1) / P) / sl;
                if (t < best - 1e-9) {
                    best = t;
                    *split = sl;
                }
            }
        }
        return static_cast<double>(T / P) + best;  // whole waves + the tail, in tile-times
    };
    if (plan->path == 2 && a.M > 256 && tile == 0) {
        // Wide 512x256 pair tiles stage 25% fewer operand bytes per FLOP
        // (lower power, so higher clocks under the power cap) but have no
        // second accumulator: each tile boundary exposes the drain of its
        // two halves (short with the TMA-store epilogue). Measured in the
        // 7B step (power-capped, per GEMM class): wide wins ~6.5% at
        // K = 11008 despite worse wave quantisation (4 vs 3.5 narrow
        // tile-times); the QKV+RoPE epilogue does not stage through TMA, so
        // it stays narrow. Hence: compare wave quantisation (a wide tile =
        // two narrow tile-times) with a bias of 1.2 in favour of wide tiles
        // (with PDL on, wide attn_out / gate_up tiles at K = 4096 too: 7B
        // step 49.60-49.65 vs 49.91-50.07 ms, alternating runs).
        const long long tn = (a.N + 255) / 256;
        const long long narrow = a.batch * ((a.M + 255) / 256) * tn, wide = a.batch * ((a.M + 511) / 512) * tn;
        int s1, s2;
        const double t_narrow = tail_plan(narrow, &s1, false), t_wide = 2.0 * tail_plan(wide, &s2, true);
        static const char* wenv = std::getenv("TN_GEMM_WIDE_BIAS");  // tuning override
        const double bias = wenv ? std::atof(wenv) : 1.2;
        // fused-norm producers stage two outputs per chunk: their drain would
        // double the wide tiles' exposed accumulator hand-off, so they stay narrow
        if (a.epi != 2 && !a.no_P && t_wide <= t_narrow * bias + 1e-9 && (a.M % 512 == 0 || a.M > 2048)) plan->path = 3;
    }
    const int bm = plan->path == 2 ? 256 : plan->path == 3 ? 512 : kBM;
    const int tm = (a.M + bm - 1) / bm, tn = (a.N + bn - 1) / bn;
    plan->tiles = a.batch * tm * tn;
    plan->grid = std::min(plan->tiles, std::max(1, num_sms));
    plan->ksplit = 1;
    if (plan->path == 0 && !split && a.epi == 0 && a.causal == 0 && !a.no_P && a.ksplit >= 0) {
        // Split-K for tiles that fill few SMs with a long K (the LoRA adapter
        // GEMMs M 4096 x N 64 x K 4096-22016 = 32 tiles; config 5's P·V):
        // ksplit units per tile, fp32 partials in the workspace, reduced in
        // split order. Automatic (ksplit 0) when the tiles fill <= 1/4 of the
        // SMs and K has >= 32 blocks; n > 1 forces n.
        const int nk = static_cast<int>((a.K * es + kAtom - 1) / kAtom);
        int ks = a.ksplit;
        if (ks == 0 && 4 * plan->tiles <= num_sms && nk >= 32)
            ks = std::min({num_sms / std::max(1, plan->tiles), nk / 8, 8});
        ks = std::min(ks, nk);
        if (ks >= 2) {
            plan->ksplit = ks;
            plan->grid = std::min(plan->tiles * ks, std::max(1, num_sms));
            plan->ws_bytes = static_cast<std::size_t>(plan->tiles) * ks * kBM * bn * 4;
        }
    }
    if (plan->path == 2 || plan->path == 3) {
        plan->grid = std::max(2, std::min(2 * plan->tiles, num_sms) / 2 * 2);
        const int npairs = plan->grid / 2, T = plan->tiles;
        const int nk = static_cast<int>((a.K * es + kAtom - 1) / kAtom);
        // TN_GEMM_SK=1 (or tile "streamk") selects a stream-K tail instead
        // (narrow tiles; last partial wave + one full wave split by K
        // blocks). Measured on B200 it never beat the sliced tail (fix-up
        // traffic + serialised finishers), so it is off by default.
        static const char* sk_env = std::getenv("TN_GEMM_SK");
        const bool sk_on = plan->path == 2 && !a.no_P && !mn && (tile == 3 || (sk_env && std::strcmp(sk_env, "1") == 0));
        if (sk_on) {
            if (a.causal == 0 && T >= npairs && T % npairs != 0) {
                const int sk = T / npairs >= 2 ? T % npairs + npairs : T;
                if (static_cast<long long>(sk) * nk >= 4LL * npairs) {
                    plan->sk_tiles = sk;
                    plan->sk_nk = nk;
                    plan->ws_bytes = static_cast<std::size_t>(npairs) * 2 * 128 * 256 * 4 + static_cast<std::size_t>(npairs) * 2 * 4;
                }
            }
        } else {
            int sl = 1;
            tail_plan(T, &sl, plan->path == 3);
            if (sl > 1) {
                const int rem = T >= P ? T % P : T;
                plan->tail_split = sl;
                plan->tail_units = rem * sl;
                plan->grid = 2 * std::min(P, T >= P ? P : rem * sl);
            }
        }
    }
    if (ok) {
        // Kernel attributes once per CUDA device (any thread; setting them twice is harmless).
        static std::atomic<unsigned long long> attr_set{0};
        int dev = 0;
        cudaGetDevice(&dev);
        if (!((attr_set.load(std::memory_order_acquire) >> dev) & 1ULL)) {
            cudaFuncSetAttribute(gemm_kernel<64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<64>());
            cudaFuncSetAttribute(gemm_kernel<128, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<128>());
            cudaFuncSetAttribute(gemm_kernel<256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<256>());
            cudaFuncSetAttribute(gemm_kernel<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<64, true>());
            cudaFuncSetAttribute(gemm_kernel<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem_bytes<128, true>());
            cudaFuncSetAttribute(gemm_kernel_2sm, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes_2sm());
            cudaFuncSetAttribute(gemm_kernel_2sm_w, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes_2sm_w());
            attr_set.fetch_or(1ULL << dev, std::memory_order_release);
        }
    }
    return cudaSuccess;
}

cudaError_t gemm_launch(const GemmPlan& plan, cudaStream_t s, GemmWorkspace* ws) {
    const GemmArgs& a = plan.args;
    if (plan.path == 1 && a.epi == 2) return cudaErrorNotSupported;  // rejected at prepare time
    if (plan.path == 1) {
        const std::int64_t warps = static_cast<std::int64_t>(a.batch) * a.M * (a.epi == 1 ? a.N / 2 : a.N);
        const int threads = 256;
        const std::int64_t blocks = (warps * 32 + threads - 1) / threads;
        return launch_pdl(gemm_simt_kernel, dim3(static_cast<unsigned>(blocks)), dim3(threads), 0, s, a);
    }
    Params p;
    p.C = a.C;
    p.R = a.R;
    p.M = a.M;
    p.N = a.N;
    p.K = a.K;
    p.batch = a.batch;
    const int bm = plan.path == 3 ? 512 : plan.path == 2 ? 256 : kBM;
    p.tiles_m = (a.M + bm - 1) / bm;
    p.tiles_n = (a.N + plan.bn - 1) / plan.bn;
    p.ldc = a.ldc;
    p.sc = a.sc;
    p.alpha = a.alpha;
    p.out_dtype = a.out_dtype;
    p.causal = a.causal;
    p.in_bytes = dtype_size(a.in_dtype);
    p.a_batched = a.batch > 1 && a.sa != 0;
    p.b_batched = a.batch > 1 && a.sb != 0;
    p.epi = a.epi;
    p.rope = static_cast<const float*>(a.rope);
    p.heads = a.heads;
    p.tail_split = std::max(1, plan.tail_split);
    p.tail_units = plan.tail_units;
    p.dp_tiles = plan.tiles - plan.tail_units / p.tail_split;
    p.tma_c = plan.tc_ok && (plan.path == 2 || plan.path == 3) && (a.epi == 0 || a.epi == 1) ? 1 : 0;
    p.split = a.split && a.in_dtype == F32 && plan.path == 0 ? 1 : 0;
    p.a_mn = a.a_mn ? 1 : 0;
    p.b_mn = a.b_mn ? 1 : 0;
    p.rs_P = a.rs_P;
    p.rs_ld = a.rs_ld;
    p.rs_row0 = a.rs_row0;
    p.rs_chunks = a.rs_chunks;
    p.rs_inv_dim = a.rs_inv_dim;
    p.rs_eps = a.rs_eps;
    p.no_g = static_cast<const __nv_bfloat16*>(a.no_g);
    p.no_P = a.no_P;
    p.sk_nk = 0;
    p.sk_total = 0;
    p.ws = nullptr;
    p.flags = nullptr;
    p.epoch = 0;
    if (plan.path == 2 && plan.sk_tiles > 0 && ws && ws->p && ws->bytes >= plan.ws_bytes) {
        const int npairs = plan.grid / 2;
        p.dp_tiles = plan.tiles - plan.sk_tiles;
        p.sk_nk = plan.sk_nk;
        p.sk_total = static_cast<long long>(plan.sk_tiles) * plan.sk_nk;
        p.ws = static_cast<float*>(ws->p);
        p.flags = reinterpret_cast<unsigned*>(static_cast<char*>(ws->p) + static_cast<std::size_t>(npairs) * 2 * 128 * 256 * 4);
        if (++ws->epoch == 0) ws->epoch = 1;  // 0 = never published
        p.epoch = ws->epoch;
    }
    p.ksplit = 1;
    unsigned grid = static_cast<unsigned>(plan.grid);
    if (plan.path == 0 && plan.ksplit > 1) {
        if (ws && ws->p && ws->bytes >= plan.ws_bytes && ws->counters &&
            ws->counter_count >= static_cast<std::size_t>(plan.tiles)) {
            p.ksplit = plan.ksplit;
            p.ws = static_cast<float*>(ws->p);
            p.flags = ws->counters;
        } else {
            grid = static_cast<unsigned>(std::min(plan.tiles, plan.grid));  // no workspace: unsplit
        }
    }
    if (plan.path == 3)
        return launch_pdl(gemm_kernel_2sm_w, dim3(plan.grid), dim3(kThreadsW), smem_bytes_2sm_w(), s, plan.ta, plan.tb,
                          plan.tbh, plan.tbq, plan.tc, p);
    if (plan.path == 2)
        return launch_pdl(gemm_kernel_2sm, dim3(plan.grid), dim3(kThreads), smem_bytes_2sm(), s, plan.ta, plan.tb,
                          plan.tbh, plan.tbq, plan.tc, p);
    if (p.split)
        return plan.bn == 128 ? launch_pdl(gemm_kernel<128, true>, dim3(grid), dim3(threads_1cta<128, true>()),
                                           smem_bytes<128, true>(), s, plan.ta, plan.tb, p)
                              : launch_pdl(gemm_kernel<64, true>, dim3(grid), dim3(threads_1cta<64, true>()),
                                           smem_bytes<64, true>(), s, plan.ta, plan.tb, p);
    if (plan.bn == 128)
        return launch_pdl(gemm_kernel<128, false>, dim3(grid), dim3(kThreads), smem_bytes<128>(), s, plan.ta,
                          plan.tb, p);
    if (plan.bn == 64)
        return launch_pdl(gemm_kernel<64, false>, dim3(grid), dim3(kThreads), smem_bytes<64>(), s, plan.ta,
                          plan.tb, p);
    return launch_pdl(gemm_kernel<256, false>, dim3(grid), dim3(kThreads), smem_bytes<256>(), s, plan.ta, plan.tb,
                      p);
}

}  // namespace tn::k
