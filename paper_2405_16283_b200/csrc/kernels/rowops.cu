// Row-reduction tasks: RMSNorm and (causal) softmax.
// One CTA per row; 128-bit coalesced loads, the row is kept in registers,
// warp-shuffle + shared-memory reductions in a fixed tree order (the result
// is independent of the schedule and of other rows).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "kernels.hpp"
#include "tc_common.cuh"

namespace tn::k {
namespace {

constexpr int kRowThreads = 256;

template <bool kMax>
__device__ __forceinline__ float block_reduce(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o /= 2) {
        float w = __shfl_xor_sync(0xffffffffu, v, o);
        v = kMax ? fmaxf(v, w) : v + w;
    }
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    __syncthreads();  // red[] reuse across calls
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float r = red[0];
    for (int i = 1; i < kRowThreads / 32; ++i) r = kMax ? fmaxf(r, red[i]) : r + red[i];
    return r;
}

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

// cols % 8 == 0, <= kRowThreads * 8 * kMaxVec
template <int kMaxVec>
__global__ void __launch_bounds__(kRowThreads) rmsnorm_vec(const __nv_bfloat16* __restrict__ x,
                                                           const __nv_bfloat16* __restrict__ w,
                                                           __nv_bfloat16* __restrict__ y, int cols, float eps) {
    __shared__ float red[kRowThreads / 32];
    const std::int64_t row = blockIdx.x;
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
    const int nv = cols / 8;
    float v[kMaxVec][8];
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
        int c = threadIdx.x + i * kRowThreads;
        if (c < nv) {
            unpack8(xr[c], v[i]);
#pragma unroll
            for (int j = 0; j < 8; ++j) ss += v[i][j] * v[i][j];
        }
    }
    ss = block_reduce<false>(ss, red);
    const float inv = rsqrtf(ss / static_cast<float>(cols) + eps);
    const uint4* wr = reinterpret_cast<const uint4*>(w);
    uint4* yr = reinterpret_cast<uint4*>(y + row * cols);
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
        int c = threadIdx.x + i * kRowThreads;
        if (c < nv) {
            float g[8];
            unpack8(wr[c], g);
#pragma unroll
            for (int j = 0; j < 8; ++j) v[i][j] = v[i][j] * inv * g[j];
            yr[c] = pack8(v[i]);
        }
    }
}

// Persistent variant: grid = a few CTAs per SM, each CTA walks rows with a
// stride and loads row i+1 into registers before reducing row i, so HBM/L2
// latency overlaps the reduction and there is no tail wave.
template <int kMaxVec>
__global__ void __launch_bounds__(kRowThreads) rmsnorm_persist(const __nv_bfloat16* __restrict__ x,
                                                               const __nv_bfloat16* __restrict__ w,
                                                               __nv_bfloat16* __restrict__ y, int rows, int cols,
                                                               float eps) {
    __shared__ float red[kRowThreads / 32];
    const int nv = cols / 8;
    uint4 cur[kMaxVec], nxt[kMaxVec];
    auto load = [&](std::int64_t row, uint4* dst) {
        const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
#pragma unroll
        for (int i = 0; i < kMaxVec; ++i) {
            const int c = threadIdx.x + i * kRowThreads;
            dst[i] = c < nv ? xr[c] : make_uint4(0, 0, 0, 0);
        }
    };
    pdl_trigger();
    pdl_wait();
    std::int64_t row = blockIdx.x;
    if (row >= rows) return;
    load(row, cur);
    const uint4* wr = reinterpret_cast<const uint4*>(w);
    for (; row < rows; row += gridDim.x) {
        const std::int64_t next = row + gridDim.x;
        if (next < rows) load(next, nxt);
        float ss = 0.f;
#pragma unroll
        for (int i = 0; i < kMaxVec; ++i) {
            float v[8];
            unpack8(cur[i], v);
#pragma unroll
            for (int j = 0; j < 8; ++j) ss += v[j] * v[j];
        }
        ss = block_reduce<false>(ss, red);
        const float inv = rsqrtf(ss / static_cast<float>(cols) + eps);
        uint4* yr = reinterpret_cast<uint4*>(y + row * cols);
#pragma unroll
        for (int i = 0; i < kMaxVec; ++i) {
            const int c = threadIdx.x + i * kRowThreads;
            if (c < nv) {
                float v[8], g[8];
                unpack8(cur[i], v);
                unpack8(wr[c], g);
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = v[j] * inv * g[j];
                yr[c] = pack8(v);
            }
        }
#pragma unroll
        for (int i = 0; i < kMaxVec; ++i) cur[i] = nxt[i];
    }
}

__global__ void __launch_bounds__(kRowThreads) rmsnorm_scalar(const __nv_bfloat16* __restrict__ x,
                                                              const __nv_bfloat16* __restrict__ w,
                                                              __nv_bfloat16* __restrict__ y, int cols, float eps) {
    __shared__ float red[kRowThreads / 32];
    const std::int64_t row = blockIdx.x;
    float ss = 0.f;
    for (int c = threadIdx.x; c < cols; c += kRowThreads) {
        float a = __bfloat162float(x[row * cols + c]);
        ss += a * a;
    }
    ss = block_reduce<false>(ss, red);
    const float inv = rsqrtf(ss / static_cast<float>(cols) + eps);
    for (int c = threadIdx.x; c < cols; c += kRowThreads)
        y[row * cols + c] = __float2bfloat16_rn(__bfloat162float(x[row * cols + c]) * inv * __bfloat162float(w[c]));
}

// Causal/full softmax of fp32 scores into bf16 probabilities, row in
// registers (cols % 4 == 0, cols <= kRowThreads * 4 * kMaxVec).
template <int kMaxVec>
__global__ void __launch_bounds__(kRowThreads) softmax_vec(const float* __restrict__ S, __nv_bfloat16* __restrict__ P,
                                                           int rows, int cols, float scale_log2, int causal) {
    __shared__ float red[kRowThreads / 32];
    const std::int64_t r = blockIdx.x;  // over batch*rows
    const int i = static_cast<int>(r % rows);
    const int valid = causal ? min(cols, i + 1) : cols;
    const float4* sr = reinterpret_cast<const float4*>(S + r * cols);
    const int nv = cols / 4;
    float v[kMaxVec][4];
    float mx = -INFINITY;
#pragma unroll
    for (int q = 0; q < kMaxVec; ++q) {
        int c = threadIdx.x + q * kRowThreads;
        if (c < nv && c * 4 < valid) {
            float4 a = sr[c];
            v[q][0] = a.x * scale_log2;
            v[q][1] = a.y * scale_log2;
            v[q][2] = a.z * scale_log2;
            v[q][3] = a.w * scale_log2;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (c * 4 + j < valid) mx = fmaxf(mx, v[q][j]);
        }
    }
    mx = block_reduce<true>(mx, red);
    float sum = 0.f;
#pragma unroll
    for (int q = 0; q < kMaxVec; ++q) {
        int c = threadIdx.x + q * kRowThreads;
        if (c < nv) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                float e = (c * 4 + j < valid) ? exp2f(v[q][j] - mx) : 0.f;
                v[q][j] = e;
                sum += e;
            }
        }
    }
    sum = block_reduce<false>(sum, red);
    const float inv = 1.0f / sum;
    uint2* pr = reinterpret_cast<uint2*>(P + r * cols);
#pragma unroll
    for (int q = 0; q < kMaxVec; ++q) {
        int c = threadIdx.x + q * kRowThreads;
        if (c < nv) {
            uint2 u;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
            h[0] = __floats2bfloat162_rn(v[q][0] * inv, v[q][1] * inv);
            h[1] = __floats2bfloat162_rn(v[q][2] * inv, v[q][3] * inv);
            pr[c] = u;
        }
    }
}

__global__ void __launch_bounds__(kRowThreads) softmax_scalar(const float* __restrict__ S, __nv_bfloat16* __restrict__ P,
                                                              int rows, int cols, float scale_log2, int causal) {
    __shared__ float red[kRowThreads / 32];
    const std::int64_t r = blockIdx.x;
    const int i = static_cast<int>(r % rows);
    const int valid = causal ? min(cols, i + 1) : cols;
    const float* s = S + r * cols;
    float mx = -INFINITY;
    for (int c = threadIdx.x; c < valid; c += kRowThreads) mx = fmaxf(mx, s[c] * scale_log2);
    mx = block_reduce<true>(mx, red);
    float sum = 0.f;
    for (int c = threadIdx.x; c < valid; c += kRowThreads) sum += exp2f(s[c] * scale_log2 - mx);
    sum = block_reduce<false>(sum, red);
    const float inv = 1.0f / sum;
    for (int c = threadIdx.x; c < cols; c += kRowThreads)
        P[r * cols + c] = __float2bfloat16_rn(c < valid ? exp2f(s[c] * scale_log2 - mx) * inv : 0.f);
}


// ---------------------------------------------------------------------------
// Two-pass blockwise softmax over materialised score tiles (config 5: the
// n^2 intermediates live in memgraph vertices the planner may offload).
// Statistics are (m, l) per row in natural-log units: m = max_j s_j,
// l = sum_j exp(s_j - m). `causal` marks a diagonal tile: column j of row i
// is valid iff j <= i.

// st[r] = (m, l) of one bf16 score-tile row.
__global__ void __launch_bounds__(kRowThreads) rowstats_kernel(const __nv_bfloat16* __restrict__ S,
                                                               float2* __restrict__ st, int cols, int causal) {
    __shared__ float red[kRowThreads / 32];
    const std::int64_t r = blockIdx.x;
    const int valid = causal ? min(cols, static_cast<int>(r) + 1) : cols;
    const __nv_bfloat16* s = S + r * cols;
    constexpr float L2E = 1.4426950408889634f;
    float mx = -INFINITY;
    const bool vec = (cols % 8 == 0) && ((reinterpret_cast<std::uintptr_t>(S) & 15) == 0);
    if (vec) {
        for (int c = threadIdx.x * 8; c < valid; c += kRowThreads * 8) {
            float f[8];
            unpack8(*reinterpret_cast<const uint4*>(s + c), f);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (c + j < valid) mx = fmaxf(mx, f[j]);
        }
    } else {
        for (int c = threadIdx.x; c < valid; c += kRowThreads) mx = fmaxf(mx, __bfloat162float(s[c]));
    }
    mx = block_reduce<true>(mx, red);
    float sum = 0.f;
    if (vec) {
        for (int c = threadIdx.x * 8; c < valid; c += kRowThreads * 8) {
            float f[8];
            unpack8(*reinterpret_cast<const uint4*>(s + c), f);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (c + j < valid) sum += exp2f((f[j] - mx) * L2E);
        }
    } else {
        for (int c = threadIdx.x; c < valid; c += kRowThreads) sum += exp2f((__bfloat162float(s[c]) - mx) * L2E);
    }
    sum = block_reduce<false>(sum, red);
    if (threadIdx.x == 0) st[r] = make_float2(mx, sum);
}

// Single pass: the row segment stays in registers between the max and the
// sum (cols % 8 == 0, 16-byte aligned, cols <= kRowThreads * 8 * kMaxVec).
template <int kMaxVec>
__global__ void __launch_bounds__(kRowThreads) rowstats_vec(const __nv_bfloat16* __restrict__ S,
                                                            float2* __restrict__ st, int cols, int causal) {
    __shared__ float red[kRowThreads / 32];
    const std::int64_t r = blockIdx.x;
    const int valid = causal ? min(cols, static_cast<int>(r) + 1) : cols;
    const uint4* s = reinterpret_cast<const uint4*>(S + r * cols);
    constexpr float L2E = 1.4426950408889634f;
    float v[kMaxVec][8];
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
        const int c = (threadIdx.x + i * kRowThreads) * 8;
        if (c < valid) {
            unpack8(__ldcs(s + c / 8), v[i]);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (c + j < valid) mx = fmaxf(mx, v[i][j]);
        }
    }
    mx = block_reduce<true>(mx, red);
    float sum = 0.f;
#pragma unroll
    for (int i = 0; i < kMaxVec; ++i) {
        const int c = (threadIdx.x + i * kRowThreads) * 8;
        if (c < valid) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (c + j < valid) sum += exp2f((v[i][j] - mx) * L2E);
        }
    }
    sum = block_reduce<false>(sum, red);
    if (threadIdx.x == 0) st[r] = make_float2(mx, sum);
}

// Warp-per-row variants for long bf16 rows (cols % 256 == 0, 16-byte
// aligned): 8 rows per 256-thread CTA, no block barriers; lane l reads the
// 16-byte chunks l, l+32, ... (coalesced), four in flight per lane per pass.
// rowstats: pass 1 the row max (warp shuffles), pass 2 re-reads the row (an
// L2 hit: 8 KB per row was just read) for sum exp(s - m). Each lane sums its
// columns in chunk order, then a fixed xor-shuffle tree: deterministic.
constexpr int kWarpRows = kRowThreads / 32;
__global__ void __launch_bounds__(kRowThreads) rowstats_warp(const __nv_bfloat16* __restrict__ S,
                                                             float2* __restrict__ st, int rows, int cols,
                                                             int causal) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const std::int64_t r = static_cast<std::int64_t>(blockIdx.x) * kWarpRows + warp;
    if (r >= rows) return;
    const int valid = causal ? min(cols, static_cast<int>(r) + 1) : cols;
    const uint4* s = reinterpret_cast<const uint4*>(S + r * cols);
    const int nch = cols / 8;  // 16-byte chunks per row
    constexpr float L2E = 1.4426950408889634f;
    float mx = -INFINITY;
    for (int c0 = lane; c0 < nch; c0 += 32 * 4) {
        uint4 u[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (c0 + 32 * i < nch) u[i] = __ldg(s + c0 + 32 * i);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = (c0 + 32 * i) * 8;
            if (c0 + 32 * i >= nch || c >= valid) continue;
            float f[8];
            unpack8(u[i], f);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (c + j < valid) mx = fmaxf(mx, f[j]);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o /= 2) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float moff = mx * L2E;
    float sum = 0.f;
    for (int c0 = lane; c0 < nch; c0 += 32 * 4) {
        uint4 u[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (c0 + 32 * i < nch) u[i] = __ldcs(s + c0 + 32 * i);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = (c0 + 32 * i) * 8;
            if (c0 + 32 * i >= nch || c >= valid) continue;
            float f[8];
            unpack8(u[i], f);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (c + j < valid) sum += exp2f(fmaf(f[j], L2E, -moff));
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o /= 2) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) st[r] = make_float2(mx, sum);
}

// P = exp(S - m) / l, warp per row (same layout as rowstats_warp).
__global__ void __launch_bounds__(kRowThreads) softmax_apply_warp(const __nv_bfloat16* __restrict__ S,
                                                                  const float2* __restrict__ st,
                                                                  __nv_bfloat16* __restrict__ P, int rows, int cols,
                                                                  int causal) {
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const std::int64_t r = static_cast<std::int64_t>(blockIdx.x) * kWarpRows + warp;
    if (r >= rows) return;
    const int valid = causal ? min(cols, static_cast<int>(r) + 1) : cols;
    constexpr float L2E = 1.4426950408889634f;
    const float2 ml = st[r];
    const float inv = 1.0f / ml.y, moff = ml.x * L2E;
    const uint4* s = reinterpret_cast<const uint4*>(S + r * cols);
    uint4* p = reinterpret_cast<uint4*>(P + r * cols);
    const int nch = cols / 8;
    for (int c0 = lane; c0 < nch; c0 += 32 * 4) {
        uint4 u[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
            if (c0 + 32 * i < nch) u[i] = __ldcs(s + c0 + 32 * i);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (c0 + 32 * i >= nch) continue;
            const int c = (c0 + 32 * i) * 8;
            float f[8];
            unpack8(u[i], f);
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = (c + j < valid) ? exp2f(fmaf(f[j], L2E, -moff)) * inv : 0.f;
            __stcs(p + c0 + 32 * i, pack8(f));
        }
    }
}

constexpr int kMaxParts = 64;
struct Parts {
    const float2* p[kMaxParts];
    int n;
};

// (m, l) of the union of k column ranges, folded in argument order.
__global__ void stats_combine_kernel(Parts a, float2* __restrict__ out, int rows) {
    constexpr float L2E = 1.4426950408889634f;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
        float2 acc = a.p[0][r];
        for (int k = 1; k < a.n; ++k) {
            const float2 x = a.p[k][r];
            const float m = fmaxf(acc.x, x.x);
            acc.y = acc.y * exp2f((acc.x - m) * L2E) + x.y * exp2f((x.x - m) * L2E);
            acc.x = m;
        }
        out[r] = acc;
    }
}

// P = exp(S - m) / l (bf16), masked (diagonal tile) entries exactly zero.
__global__ void __launch_bounds__(kRowThreads) softmax_apply_kernel(const __nv_bfloat16* __restrict__ S,
                                                                    const float2* __restrict__ st,
                                                                    __nv_bfloat16* __restrict__ P, int cols,
                                                                    int causal) {
    const std::int64_t r = blockIdx.x;
    const int valid = causal ? min(cols, static_cast<int>(r) + 1) : cols;
    constexpr float L2E = 1.4426950408889634f;
    const float2 ml = st[r];
    const float inv = 1.0f / ml.y, moff = ml.x * L2E;
    const __nv_bfloat16* s = S + r * cols;
    __nv_bfloat16* p = P + r * cols;
    const bool vec = (cols % 8 == 0) && ((reinterpret_cast<std::uintptr_t>(S) & 15) == 0) &&
                     ((reinterpret_cast<std::uintptr_t>(P) & 15) == 0);
    if (vec) {
        for (int c = threadIdx.x * 8; c < cols; c += kRowThreads * 8) {
            float f[8];
            unpack8(*reinterpret_cast<const uint4*>(s + c), f);
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = (c + j < valid) ? exp2f(f[j] * L2E - moff) * inv : 0.f;
            *reinterpret_cast<uint4*>(p + c) = pack8(f);
        }
    } else {
        for (int c = threadIdx.x; c < cols; c += kRowThreads)
            p[c] = __float2bfloat16_rn(c < valid ? exp2f(__bfloat162float(s[c]) * L2E - moff) * inv : 0.f);
    }
}

bool al16(const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15) == 0; }

}  // namespace

cudaError_t rmsnorm(const void* x, const void* w, void* y, int rows, int cols, float eps, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    auto X = static_cast<const __nv_bfloat16*>(x);
    auto W = static_cast<const __nv_bfloat16*>(w);
    auto Y = static_cast<__nv_bfloat16*>(y);
    static const char* env = std::getenv("TN_RMSNORM");  // A/B: "vec" = one CTA per row
    const bool persist = !(env && std::strcmp(env, "vec") == 0);
    if (persist && cols % 8 == 0 && al16(x) && al16(w) && al16(y) && cols <= kRowThreads * 8 * 4) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        static const char* cps_env = std::getenv("TN_RMSNORM_CPS");  // tuning: CTAs per SM
        const int cps = cps_env ? std::atoi(cps_env) : 4;
        const int grid = std::min(rows, sms * cps);
        if (cols <= kRowThreads * 8 * 2) return launch_pdl(rmsnorm_persist<2>, dim3(grid), dim3(kRowThreads), 0, s, X, W, Y, rows, cols, eps);
        return launch_pdl(rmsnorm_persist<4>, dim3(grid), dim3(kRowThreads), 0, s, X, W, Y, rows, cols, eps);
    } else if (cols % 8 == 0 && al16(x) && al16(w) && al16(y) && cols <= kRowThreads * 8 * 8) {
        if (cols <= kRowThreads * 8 * 2) rmsnorm_vec<2><<<rows, kRowThreads, 0, s>>>(X, W, Y, cols, eps);
        else if (cols <= kRowThreads * 8 * 4) rmsnorm_vec<4><<<rows, kRowThreads, 0, s>>>(X, W, Y, cols, eps);
        else rmsnorm_vec<8><<<rows, kRowThreads, 0, s>>>(X, W, Y, cols, eps);
    } else {
        rmsnorm_scalar<<<rows, kRowThreads, 0, s>>>(X, W, Y, cols, eps);
    }
    return cudaGetLastError();
}

cudaError_t softmax(const void* S, void* P, int batch, int rows, int cols, float scale, int causal, cudaStream_t s) {
    const std::int64_t n = static_cast<std::int64_t>(batch) * rows;
    if (n <= 0) return cudaSuccess;
    const float sl2 = scale * 1.4426950408889634f;
    auto Sp = static_cast<const float*>(S);
    auto Pp = static_cast<__nv_bfloat16*>(P);
    if (cols % 4 == 0 && al16(S) && (reinterpret_cast<std::uintptr_t>(P) & 7) == 0 && cols <= kRowThreads * 4 * 16) {
        if (cols <= kRowThreads * 4 * 4) softmax_vec<4><<<static_cast<unsigned>(n), kRowThreads, 0, s>>>(Sp, Pp, rows, cols, sl2, causal);
        else if (cols <= kRowThreads * 4 * 8) softmax_vec<8><<<static_cast<unsigned>(n), kRowThreads, 0, s>>>(Sp, Pp, rows, cols, sl2, causal);
        else softmax_vec<16><<<static_cast<unsigned>(n), kRowThreads, 0, s>>>(Sp, Pp, rows, cols, sl2, causal);
    } else {
        softmax_scalar<<<static_cast<unsigned>(n), kRowThreads, 0, s>>>(Sp, Pp, rows, cols, sl2, causal);
    }
    return cudaGetLastError();
}

cudaError_t rowstats(const void* S, void* st, int rows, int cols, int causal, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    auto Sp = static_cast<const __nv_bfloat16*>(S);
    auto Tp = static_cast<float2*>(st);
    static const char* env = std::getenv("TN_ROWOPS");  // A/B: "block" = one CTA per row
    const bool warp_rows = !(env && std::strcmp(env, "block") == 0);
    if (warp_rows && cols % 256 == 0 && al16(S)) {
        rowstats_warp<<<(rows + kWarpRows - 1) / kWarpRows, kRowThreads, 0, s>>>(Sp, Tp, rows, cols, causal);
        return cudaGetLastError();
    }
    if (cols % 8 == 0 && al16(S) && cols <= kRowThreads * 8 * 4) {
        if (cols <= kRowThreads * 8 * 2) rowstats_vec<2><<<rows, kRowThreads, 0, s>>>(Sp, Tp, cols, causal);
        else rowstats_vec<4><<<rows, kRowThreads, 0, s>>>(Sp, Tp, cols, causal);
        return cudaGetLastError();
    }
    rowstats_kernel<<<rows, kRowThreads, 0, s>>>(Sp, Tp, cols, causal);
    return cudaGetLastError();
}

cudaError_t stats_combine(const void* const* parts, int n, void* out, int rows, cudaStream_t s) {
    if (n < 1 || n > kMaxParts) return cudaErrorInvalidValue;
    Parts a{};
    a.n = n;
    for (int i = 0; i < n; ++i) a.p[i] = static_cast<const float2*>(parts[i]);
    stats_combine_kernel<<<(rows + 255) / 256, 256, 0, s>>>(a, static_cast<float2*>(out), rows);
    return cudaGetLastError();
}

cudaError_t softmax_apply(const void* S, const void* st, void* P, int rows, int cols, int causal, cudaStream_t s) {
    if (rows <= 0) return cudaSuccess;
    static const char* env = std::getenv("TN_ROWOPS");
    const bool warp_rows = !(env && std::strcmp(env, "block") == 0);
    if (warp_rows && cols % 256 == 0 && al16(S) && al16(P)) {
        softmax_apply_warp<<<(rows + kWarpRows - 1) / kWarpRows, kRowThreads, 0, s>>>(
            static_cast<const __nv_bfloat16*>(S), static_cast<const float2*>(st), static_cast<__nv_bfloat16*>(P), rows,
            cols, causal);
        return cudaGetLastError();
    }
    softmax_apply_kernel<<<rows, kRowThreads, 0, s>>>(static_cast<const __nv_bfloat16*>(S),
                                                      static_cast<const float2*>(st), static_cast<__nv_bfloat16*>(P),
                                                      cols, causal);
    return cudaGetLastError();
}

}  // namespace tn::k
