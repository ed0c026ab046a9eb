// Backward / training tasks for the LoRA fine-tuning memgraph (BASELINE config
// 4): layout transposes, RMSNorm backward, SwiGLU backward, softmax backward,
// cross-entropy (loss and gradient). Row kernels: one CTA per row, warp-shuffle
// + shared-memory reductions in a fixed order (deterministic); elementwise
// kernels: grid-stride, 128-bit where aligned.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.hpp"

namespace tn::k {
namespace {

constexpr int kT = 256;

template <bool kMax>
__device__ __forceinline__ float block_reduce(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o /= 2) {
        float w = __shfl_xor_sync(0xffffffffu, v, o);
        v = kMax ? fmaxf(v, w) : v + w;
    }
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float r = red[0];
    for (int i = 1; i < kT / 32; ++i) r = kMax ? fmaxf(r, red[i]) : r + red[i];
    return r;
}

__device__ __forceinline__ float ldf(const void* p, std::int64_t i, int dt) {
    return dt == BF16 ? __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]) : static_cast<const float*>(p)[i];
}
__device__ __forceinline__ void stf(void* p, std::int64_t i, int dt, float v) {
    if (dt == BF16) static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
    else static_cast<float*>(p)[i] = v;
}

unsigned grid_for(std::int64_t work) {
    std::int64_t b = (work + kT - 1) / kT;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return static_cast<unsigned>(b);
}

// out[b][c][r] = in[b][r][c]  (32x32 smem tiles, 2- or 4-byte elements)
template <typename T>
__global__ void transpose_kernel(const T* __restrict__ in, T* __restrict__ out, int rows, int cols) {
    __shared__ T tile[32][33];
    const std::int64_t base = static_cast<std::int64_t>(blockIdx.z) * rows * cols;
    const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[base + static_cast<std::int64_t>(r) * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[base + static_cast<std::int64_t>(c) * rows + r] = tile[threadIdx.x][i];
    }
}

// 16-bit transpose with 128-bit global accesses: a 64x64 tile per 256-thread
// CTA; each thread loads two 8-element row chunks, scatters them transposed
// into shared memory (row pitch 72 elements: the 8 rows a warp writes per
// step land 2-way at most on a bank), then stores two 8-element chunks of
// the transposed tile. rows % 8 == 0, cols % 8 == 0, 16-byte aligned.
__global__ void __launch_bounds__(256) transpose16_vec(const std::uint16_t* __restrict__ in,
                                                       std::uint16_t* __restrict__ out, int rows, int cols) {
    constexpr int TP = 72;
    __shared__ __align__(16) std::uint16_t tile[64 * TP];
    const std::int64_t base = static_cast<std::int64_t>(blockIdx.z) * rows * cols;
    const int r0 = blockIdx.y * 64, c0 = blockIdx.x * 64;
    const int t = threadIdx.x;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int lr = t / 8 + 32 * k, lc = (t % 8) * 8;
        const int r = r0 + lr, c = c0 + lc;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r < rows && c < cols) v = __ldcs(reinterpret_cast<const uint4*>(in + base + static_cast<std::int64_t>(r) * cols + c));
        const std::uint16_t* e = reinterpret_cast<const std::uint16_t*>(&v);
#pragma unroll
        for (int j = 0; j < 8; ++j) tile[(lc + j) * TP + lr] = e[j];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int lc = t / 8 + 32 * k, lr = (t % 8) * 8;  // output row = input column
        const int c = c0 + lc, r = r0 + lr;
        if (c < cols && r < rows)
            __stcs(reinterpret_cast<uint4*>(out + base + static_cast<std::int64_t>(c) * rows + r),
                   *reinterpret_cast<const uint4*>(&tile[lc * TP + lr]));
    }
}

// dx = r*(w.dy) - x * r^3 * mean((w.dy).x),  r = rsqrt(mean(x^2) + eps)
__global__ void __launch_bounds__(kT) rmsnorm_bwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                         const __nv_bfloat16* __restrict__ w,
                                                         const __nv_bfloat16* __restrict__ dy,
                                                         __nv_bfloat16* __restrict__ dx, int cols, float eps) {
    __shared__ float red[kT / 32];
    const std::int64_t row = blockIdx.x;
    const __nv_bfloat16* xr = x + row * cols;
    const __nv_bfloat16* dr = dy + row * cols;
    float ss = 0.f, gx = 0.f;
    for (int c = threadIdx.x; c < cols; c += kT) {
        const float a = __bfloat162float(xr[c]);
        ss += a * a;
        gx += __bfloat162float(w[c]) * __bfloat162float(dr[c]) * a;
    }
    ss = block_reduce<false>(ss, red);
    gx = block_reduce<false>(gx, red);
    const float r = rsqrtf(ss / cols + eps);
    const float k = r * r * r * gx / cols;
    for (int c = threadIdx.x; c < cols; c += kT) {
        const float a = __bfloat162float(xr[c]);
        const float g = __bfloat162float(w[c]) * __bfloat162float(dr[c]);
        dx[row * cols + c] = __float2bfloat16_rn(r * g - a * k);
    }
}

// Same, 16-byte loads with the row held in registers between the two passes
// (NV chunks of 8 columns per thread; cols % 8 == 0, 16-byte aligned rows):
// x, w and dy are read from memory once instead of twice, as 2-byte scalars.
template <int NV>
__global__ void __launch_bounds__(kT) rmsnorm_bwd_vec(const __nv_bfloat16* __restrict__ x,
                                                      const __nv_bfloat16* __restrict__ w,
                                                      const __nv_bfloat16* __restrict__ dy,
                                                      __nv_bfloat16* __restrict__ dx, int cols, float eps) {
    __shared__ float red[kT / 32];
    const std::int64_t row = blockIdx.x;
    const int nc = cols / 8;
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * cols);
    const uint4* dr = reinterpret_cast<const uint4*>(dy + row * cols);
    const uint4* wr = reinterpret_cast<const uint4*>(w);
    float a[NV][8], g[NV][8];
    float ss = 0.f, gx = 0.f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int c = threadIdx.x + i * kT;
        if (c < nc) {
            const uint4 xv = __ldcs(xr + c), dv = __ldcs(dr + c), wv = __ldg(wr + c);
            const __nv_bfloat16* xh = reinterpret_cast<const __nv_bfloat16*>(&xv);
            const __nv_bfloat16* dh = reinterpret_cast<const __nv_bfloat16*>(&dv);
            const __nv_bfloat16* wh = reinterpret_cast<const __nv_bfloat16*>(&wv);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                a[i][j] = __bfloat162float(xh[j]);
                g[i][j] = __bfloat162float(wh[j]) * __bfloat162float(dh[j]);
                ss += a[i][j] * a[i][j];
                gx += g[i][j] * a[i][j];
            }
        }
    }
    ss = block_reduce<false>(ss, red);
    gx = block_reduce<false>(gx, red);
    const float r = rsqrtf(ss / cols + eps);
    const float k = r * r * r * gx / cols;
    uint4* orow = reinterpret_cast<uint4*>(dx + row * cols);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int c = threadIdx.x + i * kT;
        if (c < nc) {
            uint4 o;
            __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
            for (int j = 0; j < 4; ++j)
                oh[j] = __floats2bfloat162_rn(r * g[i][2 * j] - a[i][2 * j] * k, r * g[i][2 * j + 1] - a[i][2 * j + 1] * k);
            orow[c] = o;
        }
    }
}

// gu [rows, 2*cols] = [g | u]; da [rows, cols] -> dgu [rows, 2*cols]:
// dg = da * u * silu'(g), du = da * silu(g)
__global__ void swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ gu, const __nv_bfloat16* __restrict__ da,
                                  __nv_bfloat16* __restrict__ dgu, int rows, int cols) {
    const std::int64_t total = static_cast<std::int64_t>(rows) * cols;
    for (std::int64_t i = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t r = i / cols, c = i % cols;
        const float g = __bfloat162float(gu[r * 2 * cols + c]), u = __bfloat162float(gu[r * 2 * cols + cols + c]);
        const float d = __bfloat162float(da[i]);
        const float s = 1.0f / (1.0f + __expf(-g));
        dgu[r * 2 * cols + c] = __float2bfloat16_rn(d * u * s * (1.0f + g * (1.0f - s)));
        dgu[r * 2 * cols + cols + c] = __float2bfloat16_rn(d * g * s);
    }
}

// Same, 8 columns per thread with 16-byte loads / stores (cols % 8 == 0,
// 16-byte aligned rows): per element the scalar kernel's arithmetic.
__global__ void swiglu_bwd_vec(const __nv_bfloat16* __restrict__ gu, const __nv_bfloat16* __restrict__ da,
                               __nv_bfloat16* __restrict__ dgu, int rows, int cols) {
    const int nv = cols / 8;
    const std::int64_t total = static_cast<std::int64_t>(rows) * nv;
    for (std::int64_t w = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; w < total;
         w += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        const std::int64_t r = w / nv, c = w % nv;
        const uint4* row = reinterpret_cast<const uint4*>(gu + r * 2 * cols);
        const uint4 gv = __ldcs(row + c), uv = __ldcs(row + nv + c), dv = __ldcs(reinterpret_cast<const uint4*>(da) + w);
        const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&gv);
        const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&uv);
        const __nv_bfloat162* d2 = reinterpret_cast<const __nv_bfloat162*>(&dv);
        uint4 og, ou;
        __nv_bfloat162* og2 = reinterpret_cast<__nv_bfloat162*>(&og);
        __nv_bfloat162* ou2 = reinterpret_cast<__nv_bfloat162*>(&ou);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float2 g = __bfloat1622float2(g2[j]), u = __bfloat1622float2(u2[j]), d = __bfloat1622float2(d2[j]);
            const float s0 = 1.0f / (1.0f + __expf(-g.x)), s1 = 1.0f / (1.0f + __expf(-g.y));
            og2[j] = __floats2bfloat162_rn(d.x * u.x * s0 * (1.0f + g.x * (1.0f - s0)),
                                           d.y * u.y * s1 * (1.0f + g.y * (1.0f - s1)));
            ou2[j] = __floats2bfloat162_rn(d.x * g.x * s0, d.y * g.y * s1);
        }
        uint4* orow = reinterpret_cast<uint4*>(dgu + r * 2 * cols);
        orow[c] = og;
        orow[nv + c] = ou;
    }
}

// dS = P * (dP - sum_j P_j dP_j) per row; masked (causal) entries are 0.
__global__ void __launch_bounds__(kT) softmax_bwd_kernel(const __nv_bfloat16* __restrict__ P, const void* __restrict__ dP,
                                                         int dp_dt, __nv_bfloat16* __restrict__ dS, int rows, int cols,
                                                         int causal) {
    __shared__ float red[kT / 32];
    const std::int64_t r = blockIdx.x;
    const int i = static_cast<int>(r % rows);
    const int valid = causal ? min(cols, i + 1) : cols;
    const std::int64_t base = r * cols;
    float dot = 0.f;
    for (int c = threadIdx.x; c < valid; c += kT) dot += __bfloat162float(P[base + c]) * ldf(dP, base + c, dp_dt);
    dot = block_reduce<false>(dot, red);
    for (int c = threadIdx.x; c < cols; c += kT) {
        float v = 0.f;
        if (c < valid) v = __bfloat162float(P[base + c]) * (ldf(dP, base + c, dp_dt) - dot);
        dS[base + c] = __float2bfloat16_rn(v);
    }
}

// Cross entropy over a [rows, vocab] logits tile with int32 targets:
//   grad = (softmax(l) - onehot(t)) * scale ;  loss_row = logsumexp(l) - l_t
__global__ void __launch_bounds__(kT) xent_kernel(const void* __restrict__ logits, int lg_dt,
                                                  const int* __restrict__ tgt, void* __restrict__ out, int out_dt,
                                                  int vocab, float scale, int want_grad) {
    __shared__ float red[kT / 32];
    const std::int64_t r = blockIdx.x;
    const std::int64_t base = r * vocab;
    float mx = -INFINITY;
    for (int c = threadIdx.x; c < vocab; c += kT) mx = fmaxf(mx, ldf(logits, base + c, lg_dt));
    mx = block_reduce<true>(mx, red);
    float sum = 0.f;
    for (int c = threadIdx.x; c < vocab; c += kT) sum += __expf(ldf(logits, base + c, lg_dt) - mx);
    sum = block_reduce<false>(sum, red);
    int t = tgt[r];
    t = t < 0 ? 0 : (t >= vocab ? vocab - 1 : t);
    if (want_grad) {
        const float inv = 1.0f / sum;
        for (int c = threadIdx.x; c < vocab; c += kT) {
            float p = __expf(ldf(logits, base + c, lg_dt) - mx) * inv;
            if (c == t) p -= 1.0f;
            stf(out, base + c, out_dt, p * scale);
        }
    } else if (threadIdx.x == 0) {
        static_cast<float*>(out)[r] = (mx + __logf(sum) - ldf(logits, base + t, lg_dt)) * scale;
    }
}

// Fixed-order sum of per-row losses (single CTA).
__global__ void __launch_bounds__(kT) row_sum_kernel(const float* __restrict__ v, float* __restrict__ out, int n) {
    __shared__ float red[kT / 32];
    float s = 0.f;
    for (int i = threadIdx.x; i < n; i += kT) s += v[i];
    s = block_reduce<false>(s, red);
    if (threadIdx.x == 0) out[0] = s;
}

}  // namespace

cudaError_t transpose(const void* in, void* out, int batch, int rows, int cols, int esize, cudaStream_t s) {
    auto al16 = [](const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15) == 0; };
    if (esize == 2 && rows % 8 == 0 && cols % 8 == 0 && al16(in) && al16(out)) {
        dim3 g64((cols + 63) / 64, (rows + 63) / 64, batch);
        transpose16_vec<<<g64, 256, 0, s>>>(static_cast<const std::uint16_t*>(in), static_cast<std::uint16_t*>(out),
                                             rows, cols);
        return cudaGetLastError();
    }
    dim3 grid((cols + 31) / 32, (rows + 31) / 32, batch), block(32, 8);
    if (esize == 2)
        transpose_kernel<std::uint16_t><<<grid, block, 0, s>>>(static_cast<const std::uint16_t*>(in),
                                                               static_cast<std::uint16_t*>(out), rows, cols);
    else
        transpose_kernel<std::uint32_t><<<grid, block, 0, s>>>(static_cast<const std::uint32_t*>(in),
                                                               static_cast<std::uint32_t*>(out), rows, cols);
    return cudaGetLastError();
}

cudaError_t rmsnorm_bwd(const void* x, const void* w, const void* dy, void* dx, int rows, int cols, float eps,
                        cudaStream_t s) {
    auto al16 = [](const void* p) { return (reinterpret_cast<std::uintptr_t>(p) & 15) == 0; };
    const bool vec = cols % 8 == 0 && cols / 8 <= 4 * kT && al16(x) && al16(w) && al16(dy) && al16(dx);
    if (vec) {
        const int nv = (cols / 8 + kT - 1) / kT;
        auto* kern = nv == 1 ? rmsnorm_bwd_vec<1> : nv == 2 ? rmsnorm_bwd_vec<2> : rmsnorm_bwd_vec<4>;
        kern<<<rows, kT, 0, s>>>(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w),
                                 static_cast<const __nv_bfloat16*>(dy), static_cast<__nv_bfloat16*>(dx), cols, eps);
        return cudaGetLastError();
    }
    rmsnorm_bwd_kernel<<<rows, kT, 0, s>>>(static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w),
                                           static_cast<const __nv_bfloat16*>(dy), static_cast<__nv_bfloat16*>(dx), cols,
                                           eps);
    return cudaGetLastError();
}

cudaError_t swiglu_bwd(const void* gu, const void* da, void* dgu, int rows, int cols, cudaStream_t s) {
    auto al16 = [](const void* x) { return (reinterpret_cast<std::uintptr_t>(x) & 15) == 0; };
    if (cols % 8 == 0 && al16(gu) && al16(da) && al16(dgu)) {
        swiglu_bwd_vec<<<grid_for(static_cast<std::int64_t>(rows) * (cols / 8)), kT, 0, s>>>(
            static_cast<const __nv_bfloat16*>(gu), static_cast<const __nv_bfloat16*>(da),
            static_cast<__nv_bfloat16*>(dgu), rows, cols);
        return cudaGetLastError();
    }
    swiglu_bwd_kernel<<<grid_for(static_cast<std::int64_t>(rows) * cols), kT, 0, s>>>(
        static_cast<const __nv_bfloat16*>(gu), static_cast<const __nv_bfloat16*>(da), static_cast<__nv_bfloat16*>(dgu),
        rows, cols);
    return cudaGetLastError();
}

cudaError_t softmax_bwd(const void* P, const void* dP, int dp_dtype, void* dS, int batch, int rows, int cols,
                        int causal, cudaStream_t s) {
    const std::int64_t n = static_cast<std::int64_t>(batch) * rows;
    softmax_bwd_kernel<<<static_cast<unsigned>(n), kT, 0, s>>>(static_cast<const __nv_bfloat16*>(P), dP, dp_dtype,
                                                               static_cast<__nv_bfloat16*>(dS), rows, cols, causal);
    return cudaGetLastError();
}

cudaError_t xent(const void* logits, int lg_dtype, const void* targets, void* out, int out_dtype, int rows, int vocab,
                 float scale, int want_grad, void* scratch, cudaStream_t s) {
    if (want_grad) {
        xent_kernel<<<rows, kT, 0, s>>>(logits, lg_dtype, static_cast<const int*>(targets), out, out_dtype, vocab,
                                        scale, 1);
    } else {
        xent_kernel<<<rows, kT, 0, s>>>(logits, lg_dtype, static_cast<const int*>(targets), scratch, F32, vocab, scale,
                                        0);
        row_sum_kernel<<<1, kT, 0, s>>>(static_cast<const float*>(scratch), static_cast<float*>(out), rows);
    }
    return cudaGetLastError();
}

}  // namespace tn::k
