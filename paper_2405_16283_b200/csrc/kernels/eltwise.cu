// Elementwise / layout tasks: RoPE, per-head V
// transpose, SiLU·mul, fixed-order sum of partials, embedding gather, casts.
// HBM-bound: 128-bit coalesced loads/stores, grid-stride loops sized to the
// SM count, fp32 math with one round-to-nearest-even per output.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"
#include "tc_common.cuh"

namespace tn::k {

namespace {
thread_local bool g_pdl = false;
}
void set_pdl(bool on) { g_pdl = on; }
bool pdl_enabled() { return g_pdl; }

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float2 x = __bfloat1622float2(h[i]);
        f[2 * i] = x.x;
        f[2 * i + 1] = x.y;
    }
}
__device__ __forceinline__ uint4 pack8(const float* f) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    return u;
}

unsigned grid_for(std::int64_t work, int per_block = kThreads) {
    std::int64_t b = (work + per_block - 1) / per_block;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return static_cast<unsigned>(b);
}

// One thread = 8 consecutive rotation pairs (i, i + hd/2) of one (t, h).
__global__ void rope_vec(const __nv_bfloat16* __restrict__ src, const float* __restrict__ table,
                         __nv_bfloat16* __restrict__ out, int seq, std::int64_t ld, std::int64_t col_off, int heads,
                         int hd, float sgn, int tokens_out) {
    const int half = hd / 2, groups = half / 8;
    const std::int64_t total = static_cast<std::int64_t>(seq) * heads * groups;
    for (std::int64_t w = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; w < total;
         w += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(w % groups);
        const int h = static_cast<int>((w / groups) % heads);
        const int t = static_cast<int>(w / (static_cast<std::int64_t>(groups) * heads));
        const __nv_bfloat16* x = src + t * ld + col_off + static_cast<std::int64_t>(h) * hd;
        float a[8], b[8];
        unpack8(*reinterpret_cast<const uint4*>(x + g * 8), a);
        unpack8(*reinterpret_cast<const uint4*>(x + half + g * 8), b);
        const float4* cs = reinterpret_cast<const float4*>(table + (static_cast<std::int64_t>(t) * half + g * 8) * 2);
        float lo[8], hi[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float4 q = cs[j];  // (cos_j0, sin_j0, cos_j1, sin_j1); sgn = -1 rotates back
            q.y *= sgn;
            q.w *= sgn;
            lo[2 * j] = a[2 * j] * q.x - b[2 * j] * q.y;
            hi[2 * j] = b[2 * j] * q.x + a[2 * j] * q.y;
            lo[2 * j + 1] = a[2 * j + 1] * q.z - b[2 * j + 1] * q.w;
            hi[2 * j + 1] = b[2 * j + 1] * q.z + a[2 * j + 1] * q.w;
        }
        __nv_bfloat16* o = tokens_out ? out + static_cast<std::int64_t>(t) * heads * hd + static_cast<std::int64_t>(h) * hd
                                      : out + (static_cast<std::int64_t>(h) * seq + t) * hd;
        *reinterpret_cast<uint4*>(o + g * 8) = pack8(lo);
        *reinterpret_cast<uint4*>(o + half + g * 8) = pack8(hi);
    }
}

__global__ void rope_scalar(const __nv_bfloat16* __restrict__ src, const float* __restrict__ table,
                            __nv_bfloat16* __restrict__ out, int seq, std::int64_t ld, std::int64_t col_off, int heads,
                            int hd, float sgn, int tokens_out) {
    const int half = hd / 2;
    const std::int64_t total = static_cast<std::int64_t>(seq) * heads * half;
    for (std::int64_t w = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; w < total;
         w += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(w % half);
        const int h = static_cast<int>((w / half) % heads);
        const int t = static_cast<int>(w / (static_cast<std::int64_t>(half) * heads));
        const __nv_bfloat16* x = src + t * ld + col_off + static_cast<std::int64_t>(h) * hd;
        const float a = __bfloat162float(x[i]), b = __bfloat162float(x[i + half]);
        const float c = table[(static_cast<std::int64_t>(t) * half + i) * 2];
        const float s = sgn * table[(static_cast<std::int64_t>(t) * half + i) * 2 + 1];
        __nv_bfloat16* o = tokens_out ? out + static_cast<std::int64_t>(t) * heads * hd + static_cast<std::int64_t>(h) * hd
                                      : out + (static_cast<std::int64_t>(h) * seq + t) * hd;
        o[i] = __float2bfloat16_rn(a * c - b * s);
        o[i + half] = __float2bfloat16_rn(b * c + a * s);
    }
}

// 32x32 smem tile transpose per head: src[t][col_off + h*hd + d] -> out[h][d][t].
__global__ void transpose_heads_kernel(const __nv_bfloat16* __restrict__ src, __nv_bfloat16* __restrict__ out, int seq,
                                       std::int64_t ld, std::int64_t col_off, int heads, int hd) {
    __shared__ __nv_bfloat16 tile[32][33];
    const int h = blockIdx.z;
    const int t0 = blockIdx.x * 32, d0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        int t = t0 + r, d = d0 + threadIdx.x;
        if (t < seq && d < hd) tile[r][threadIdx.x] = src[t * ld + col_off + static_cast<std::int64_t>(h) * hd + d];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        int d = d0 + r, t = t0 + threadIdx.x;
        if (t < seq && d < hd) out[(static_cast<std::int64_t>(h) * hd + d) * seq + t] = tile[threadIdx.x][r];
    }
}

// 64x64 tile per CTA (256 threads) with 16-byte accesses on both sides:
// src[t][col_off + h*hd + d] -> out[h][d][t]. Loads: a thread reads 8
// consecutive d of one t; stores: 8 consecutive t of one d (gathered from the
// padded smem tile). Needs hd % 8 == 0, seq % 8 == 0, 16-byte alignment.
__global__ void __launch_bounds__(256) transpose_heads_vec(const __nv_bfloat16* __restrict__ src,
                                                           __nv_bfloat16* __restrict__ out, int seq, std::int64_t ld,
                                                           std::int64_t col_off, int heads, int hd) {
    __shared__ __nv_bfloat16 tile[64][64 + 8];
    const int h = blockIdx.z;
    const int t0 = blockIdx.x * 64, d0 = blockIdx.y * 64;
    const __nv_bfloat16* base = src + col_off + static_cast<std::int64_t>(h) * hd;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int idx = threadIdx.x + k * 256;  // 512 vectors: 64 rows (t) x 8 vectors (d)
        const int r = idx / 8, c = (idx % 8) * 8;
        const int t = t0 + r, d = d0 + c;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (t < seq && d < hd) v = *reinterpret_cast<const uint4*>(base + static_cast<std::int64_t>(t) * ld + d);
        *reinterpret_cast<uint4*>(&tile[r][c]) = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        // 64 rows (d) x 8 vectors (t); lanes of a warp take consecutive d so the
        // smem column reads tile[c + j][r] hit consecutive banks
        const int idx = threadIdx.x + k * 256;
        const int r = idx % 64, c = (idx / 64) * 8;
        const int d = d0 + r, t = t0 + c;
        if (d >= hd || t >= seq) continue;
        uint4 v;
        __nv_bfloat16* e = reinterpret_cast<__nv_bfloat16*>(&v);
#pragma unroll
        for (int j = 0; j < 8; ++j) e[j] = tile[c + j][r];
        *reinterpret_cast<uint4*>(out + (static_cast<std::int64_t>(h) * hd + d) * seq + t) = v;
    }
}

__global__ void silu_mul_vec(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ out, int rows,
                             int cols) {
    const int nv = cols / 8;
    const std::int64_t total = static_cast<std::int64_t>(rows) * nv;
    const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
    // two independent vectors in flight per thread (loads issued before any math)
    for (std::int64_t w = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; w < total; w += 2 * stride) {
        const std::int64_t w2 = w + stride;
        const std::int64_t r = w / nv, c = w % nv, r2 = w2 / nv, c2 = w2 % nv;
        const uint4* row = reinterpret_cast<const uint4*>(gu + r * 2 * cols);
        const uint4 gv = __ldcs(row + c), uv = __ldcs(row + nv + c);
        uint4 gv2 = make_uint4(0, 0, 0, 0), uv2 = gv2;
        if (w2 < total) {
            const uint4* row2 = reinterpret_cast<const uint4*>(gu + r2 * 2 * cols);
            gv2 = __ldcs(row2 + c2);
            uv2 = __ldcs(row2 + nv + c2);
        }
        float g[8], u[8];
        unpack8(gv, g);
        unpack8(uv, u);
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = g[j] / (1.0f + __expf(-g[j])) * u[j];
        reinterpret_cast<uint4*>(out + r * cols)[c] = pack8(g);
        if (w2 < total) {
            unpack8(gv2, g);
            unpack8(uv2, u);
#pragma unroll
            for (int j = 0; j < 8; ++j) g[j] = g[j] / (1.0f + __expf(-g[j])) * u[j];
            reinterpret_cast<uint4*>(out + r2 * cols)[c2] = pack8(g);
        }
    }
}

__global__ void silu_mul_scalar(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ out, int rows,
                                int cols) {
    const std::int64_t total = static_cast<std::int64_t>(rows) * cols;
    for (std::int64_t w = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; w < total;
         w += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t r = w / cols, c = w % cols;
        float g = __bfloat162float(gu[r * 2 * cols + c]), u = __bfloat162float(gu[r * 2 * cols + cols + c]);
        out[w] = __float2bfloat16_rn(g / (1.0f + __expf(-g)) * u);
    }
}

constexpr int kMaxSum = 16;
struct SumArgs {
    const void* in[kMaxSum];
    int n;
};

constexpr int kMaxParts = 64;
struct CatArgs {
    const void* in[kMaxParts];
    int n;
};

// out = in[0] ++ in[1] ++ ... (equal-sized parts, bytes), 16-byte vectors.
__global__ void concat_kernel(CatArgs a, uint4* __restrict__ out, std::int64_t part_vec) {
    const std::int64_t total = part_vec * a.n;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int p = static_cast<int>(i / part_vec);
        out[i] = static_cast<const uint4*>(a.in[p])[i - p * part_vec];
    }
}
__global__ void concat_bytes_kernel(CatArgs a, std::uint8_t* __restrict__ out, std::int64_t part_bytes) {
    const std::int64_t total = part_bytes * a.n;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const int p = static_cast<int>(i / part_bytes);
        out[i] = static_cast<const std::uint8_t*>(a.in[p])[i - p * part_bytes];
    }
}

__device__ __forceinline__ float ld_as_float(const void* p, std::int64_t i, int dt) {
    return dt == BF16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]) : static_cast<const float*>(p)[i];
}

__global__ void sum_kernel(SumArgs a, int in_dt, void* __restrict__ out, int out_dt, std::int64_t count) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        float acc = ld_as_float(a.in[0], i, in_dt);
        for (int k = 1; k < a.n; ++k) acc += ld_as_float(a.in[k], i, in_dt);
        if (out_dt == BF16) static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(acc);
        else static_cast<float*>(out)[i] = acc;
    }
}

// bf16 (or fp32) inputs, 8 elements per thread with 16-byte loads; each
// element is still summed over the arguments in argument order.
__global__ void sum_vec8(SumArgs a, int in_dt, void* __restrict__ out, int out_dt, std::int64_t count8) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < count8;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        float acc[8], x[8];
        auto load8 = [&](const void* p, float* f) {
            if (in_dt == BF16) {
                unpack8(static_cast<const uint4*>(p)[i], f);
            } else {
                const float4 lo = static_cast<const float4*>(p)[2 * i], hi = static_cast<const float4*>(p)[2 * i + 1];
                f[0] = lo.x; f[1] = lo.y; f[2] = lo.z; f[3] = lo.w; f[4] = hi.x; f[5] = hi.y; f[6] = hi.z; f[7] = hi.w;
            }
        };
        load8(a.in[0], acc);
        for (int k = 1; k < a.n; ++k) {
            load8(a.in[k], x);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += x[j];
        }
        if (out_dt == BF16) {
            static_cast<uint4*>(out)[i] = pack8(acc);
        } else {
            float4* o = static_cast<float4*>(out);
            o[2 * i] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            o[2 * i + 1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        }
    }
}

// fp32 partial tiles, 4 elements per thread (the fp32 matmul-chain combine).
__global__ void sum_f32_vec(SumArgs a, float* __restrict__ out, std::int64_t count4) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < count4;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        float4 acc = static_cast<const float4*>(a.in[0])[i];
        for (int k = 1; k < a.n; ++k) {
            float4 x = static_cast<const float4*>(a.in[k])[i];
            acc.x += x.x;
            acc.y += x.y;
            acc.z += x.z;
            acc.w += x.w;
        }
        reinterpret_cast<float4*>(out)[i] = acc;
    }
}

__global__ void embedding_kernel(const int* __restrict__ tok, const __nv_bfloat16* __restrict__ table,
                                 __nv_bfloat16* __restrict__ out, int dim, int vocab, int vec) {
    pdl_trigger();
    pdl_wait();
    const int t = blockIdx.x;
    int id = tok[t];
    id = id < 0 ? 0 : (id >= vocab ? vocab - 1 : id);
    const __nv_bfloat16* src = table + static_cast<std::int64_t>(id) * dim;
    __nv_bfloat16* dst = out + static_cast<std::int64_t>(t) * dim;
    if (vec) {
        for (int c = threadIdx.x; c < dim / 8; c += blockDim.x)
            reinterpret_cast<uint4*>(dst)[c] = reinterpret_cast<const uint4*>(src)[c];
    } else {
        for (int c = threadIdx.x; c < dim; c += blockDim.x) dst[c] = src[c];
    }
}

// Embedding gather fused with the first RMSNorm's producer side: x = table
// row, h = bf16(x * g) in the seq*dim elements after x, and per 32-column
// chunk c the sum of x^2 (column order) to P[t * dim/32 + c]. One thread per
// chunk (dim % 32 == 0, 16-byte aligned).
__global__ void embedding_norm_kernel(const int* __restrict__ tok, const __nv_bfloat16* __restrict__ table,
                                      const __nv_bfloat16* __restrict__ g, __nv_bfloat16* __restrict__ out, int seq,
                                      int dim, int vocab) {
    const int t = blockIdx.x;
    int id = tok[t];
    id = id < 0 ? 0 : (id >= vocab ? vocab - 1 : id);
    const uint4* src = reinterpret_cast<const uint4*>(table + static_cast<std::int64_t>(id) * dim);
    uint4* x = reinterpret_cast<uint4*>(out + static_cast<std::int64_t>(t) * dim);
    uint4* h = reinterpret_cast<uint4*>(out + static_cast<std::int64_t>(seq) * dim + static_cast<std::int64_t>(t) * dim);
    float* P = reinterpret_cast<float*>(out + 2 * static_cast<std::int64_t>(seq) * dim);
    const uint4* gv = reinterpret_cast<const uint4*>(g);
    for (int c = threadIdx.x; c < dim / 32; c += blockDim.x) {
        float ss = 0.f;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint4 u = src[4 * c + q];
            float f[8], w[8];
            unpack8(u, f);
            unpack8(gv[4 * c + q], w);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                ss = fmaf(f[j], f[j], ss);
                w[j] *= f[j];
            }
            x[4 * c + q] = u;
            h[4 * c + q] = pack8(w);
        }
        P[static_cast<std::int64_t>(t) * (dim / 32) + c] = ss;
    }
}

__global__ void cast_kernel(const void* __restrict__ in, int in_dt, void* __restrict__ out, int out_dt,
                            std::int64_t count) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        float x = ld_as_float(in, i, in_dt);
        if (out_dt == BF16) static_cast<__nv_bfloat16*>(out)[i] = __float2bfloat16_rn(x);
        else static_cast<float*>(out)[i] = x;
    }
}

// f32 -> bf16, 8 elements per thread (two 16-byte loads, one 16-byte store).
__global__ void cast_f32_bf16_vec(const float4* __restrict__ in, uint4* __restrict__ out, std::int64_t count8) {
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < count8;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const float4 lo = __ldcs(in + 2 * i), hi = __ldcs(in + 2 * i + 1);
        const float f[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
        out[i] = pack8(f);
    }
}

bool al16(const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15) == 0; }

}  // namespace

cudaError_t rope(const void* src, const void* table, void* out, int seq, std::int64_t ld, std::int64_t col_off,
                 int heads, int hd, cudaStream_t s, int inverse, int tokens_out) {
    const float sgn = inverse ? -1.0f : 1.0f;
    auto S = static_cast<const __nv_bfloat16*>(src);
    auto T = static_cast<const float*>(table);
    auto O = static_cast<__nv_bfloat16*>(out);
    if (hd % 16 == 0 && ld % 8 == 0 && col_off % 8 == 0 && al16(src) && al16(table) && al16(out)) {
        std::int64_t work = static_cast<std::int64_t>(seq) * heads * (hd / 16);
        rope_vec<<<grid_for(work), kThreads, 0, s>>>(S, T, O, seq, ld, col_off, heads, hd, sgn, tokens_out);
    } else {
        std::int64_t work = static_cast<std::int64_t>(seq) * heads * (hd / 2);
        rope_scalar<<<grid_for(work), kThreads, 0, s>>>(S, T, O, seq, ld, col_off, heads, hd, sgn, tokens_out);
    }
    return cudaGetLastError();
}

cudaError_t transpose_heads(const void* src, void* out, int seq, std::int64_t ld, std::int64_t col_off, int heads,
                            int hd, cudaStream_t s) {
    if (hd % 8 == 0 && seq % 8 == 0 && ld % 8 == 0 && col_off % 8 == 0 && al16(src) && al16(out)) {
        dim3 grid((seq + 63) / 64, (hd + 63) / 64, heads);
        transpose_heads_vec<<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(src),
                                                 static_cast<__nv_bfloat16*>(out), seq, ld, col_off, heads, hd);
        return cudaGetLastError();
    }
    dim3 grid((seq + 31) / 32, (hd + 31) / 32, heads), block(32, 8);
    transpose_heads_kernel<<<grid, block, 0, s>>>(static_cast<const __nv_bfloat16*>(src),
                                                  static_cast<__nv_bfloat16*>(out), seq, ld, col_off, heads, hd);
    return cudaGetLastError();
}

cudaError_t silu_mul(const void* gu, void* out, int rows, int cols, cudaStream_t s) {
    auto G = static_cast<const __nv_bfloat16*>(gu);
    auto O = static_cast<__nv_bfloat16*>(out);
    if (cols % 8 == 0 && al16(gu) && al16(out))
        silu_mul_vec<<<grid_for(static_cast<std::int64_t>(rows) * cols / 8), kThreads, 0, s>>>(G, O, rows, cols);
    else
        silu_mul_scalar<<<grid_for(static_cast<std::int64_t>(rows) * cols), kThreads, 0, s>>>(G, O, rows, cols);
    return cudaGetLastError();
}

cudaError_t sum_n(const void* const* ins, int n, int in_dtype, void* out, int out_dtype, std::int64_t count,
                  cudaStream_t s) {
    if (n < 1 || n > kMaxSum) return cudaErrorInvalidValue;
    SumArgs a{};
    a.n = n;
    bool aligned = al16(out);
    for (int i = 0; i < n; ++i) {
        a.in[i] = ins[i];
        aligned = aligned && al16(ins[i]);
    }
    if (in_dtype == F32 && out_dtype == F32 && count % 4 == 0 && aligned)
        sum_f32_vec<<<grid_for(count / 4), kThreads, 0, s>>>(a, static_cast<float*>(out), count / 4);
    else if (count % 8 == 0 && aligned)
        sum_vec8<<<grid_for(count / 8), kThreads, 0, s>>>(a, in_dtype, out, out_dtype, count / 8);
    else
        sum_kernel<<<grid_for(count), kThreads, 0, s>>>(a, in_dtype, out, out_dtype, count);
    return cudaGetLastError();
}

cudaError_t concat(const void* const* parts, int n, std::int64_t part_bytes, void* out, cudaStream_t s) {
    if (n < 1 || n > kMaxParts) return cudaErrorInvalidValue;
    CatArgs a{};
    a.n = n;
    bool aligned = al16(out) && part_bytes % 16 == 0;
    for (int i = 0; i < n; ++i) {
        a.in[i] = parts[i];
        aligned = aligned && al16(parts[i]);
    }
    if (aligned)
        concat_kernel<<<grid_for(part_bytes / 16 * n), kThreads, 0, s>>>(a, static_cast<uint4*>(out), part_bytes / 16);
    else
        concat_bytes_kernel<<<grid_for(part_bytes * n), kThreads, 0, s>>>(a, static_cast<std::uint8_t*>(out), part_bytes);
    return cudaGetLastError();
}

cudaError_t embedding_norm(const void* tokens, const void* table, const void* g, void* out, int seq, int dim, int vocab,
                           cudaStream_t s) {
    if (dim % 32 != 0 || !al16(table) || !al16(out) || !al16(g)) return cudaErrorNotSupported;
    embedding_norm_kernel<<<seq, 128, 0, s>>>(static_cast<const int*>(tokens), static_cast<const __nv_bfloat16*>(table),
                                              static_cast<const __nv_bfloat16*>(g), static_cast<__nv_bfloat16*>(out), seq,
                                              dim, vocab);
    return cudaGetLastError();
}

cudaError_t embedding(const void* tokens, const void* table, void* out, int seq, int dim, int vocab, cudaStream_t s) {
    int vec = dim % 8 == 0 && al16(table) && al16(out);
    return launch_pdl(embedding_kernel, dim3(seq), dim3(128), 0, s, static_cast<const int*>(tokens),
                      static_cast<const __nv_bfloat16*>(table), static_cast<__nv_bfloat16*>(out), dim, vocab, vec);
    return cudaGetLastError();
}

cudaError_t cast(const void* in, int in_dtype, void* out, int out_dtype, std::int64_t count, cudaStream_t s) {
    if (in_dtype == F32 && out_dtype == BF16 && count % 8 == 0 && al16(in) && al16(out)) {
        cast_f32_bf16_vec<<<grid_for(count / 8), kThreads, 0, s>>>(static_cast<const float4*>(in),
                                                                   static_cast<uint4*>(out), count / 8);
        return cudaGetLastError();
    }
    cast_kernel<<<grid_for(count), kThreads, 0, s>>>(in, in_dtype, out, out_dtype, count);
    return cudaGetLastError();
}

}  // namespace tn::k
