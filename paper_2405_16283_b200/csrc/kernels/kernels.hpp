// Host-side launch interface of the sm_100a task kernels. Every memgraph
// Kernel vertex maps to exactly one of these launches (op payload types in
// exec/ops.hpp). All kernels are deterministic: fixed reduction order, no
// atomics, so a vertex's output does not depend on the dispatch schedule.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tn::k {

enum DType : int { BF16 = 0, F32 = 1, I32 = 2 };

// Programmatic dependent launch for the next kernel launches of this host
// thread (the executor's dispatcher): the kernel may be scheduled while the
// previous kernel on its stream drains; every PDL-aware kernel calls
// griddepcontrol.wait before its first global-memory access.
void set_pdl(bool on);
bool pdl_enabled();

inline int dtype_size(int dt) { return dt == BF16 ? 2 : 4; }

// C[b][m][n] = alpha * sum_k A[b][m][k] * B[b][n][k] (+ R[b][m][n])
// A, B K-major (row-major [M,K] and [N,K]); C, R row-major with ldc.
// causal: 0 none; 1 "scores" (tiles strictly above the diagonal are
// skipped — their values are never read by a causal softmax); 2 "probs"
// (A must be lower triangular, A[b][m][k>m] == 0 as a causal softmax writes
// it, so the K loop stops at the diagonal block).
struct GemmArgs {
    const void* A = nullptr;
    const void* B = nullptr;
    const void* R = nullptr;
    void* C = nullptr;
    int M = 0, N = 0, K = 0, batch = 1;
    std::int64_t lda = 0, ldb = 0, ldc = 0;
    std::int64_t sa = 0, sb = 0, sc = 0;  // batch strides (elements)
    float alpha = 1.0f;
    int in_dtype = BF16;   // BF16 -> kind::f16, F32 -> kind::tf32
    int out_dtype = BF16;
    int causal = 0;
    int epi = 0;  // 1: SwiGLU epilogue, out [M, N/2]: out[:, 128b+j] = silu(C[:, 256b+j]) * C[:, 256b+128+j]
                  // 2: QKV + RoPE epilogue (hd 128): out = [rope(q) (H,M,128) | rope(k) | vᵀ (H,128,M)]
    const void* rope = nullptr;  // epi 2: fp32 [M, 64, 2] (cos, sin)
    int heads = 0;               // epi 2: heads per section, N = 3 * heads * 128
    // Fused RMSNorm, consumer side: row m is scaled by
    // rsqrt(sum_{c < rs_chunks} rs_P[(rs_row0 + m) * rs_ld + c] / dim + eps).
    const float* rs_P = nullptr;
    int rs_ld = 0, rs_row0 = 0, rs_chunks = 0;
    float rs_inv_dim = 0.f, rs_eps = 0.f;
    // Fused RMSNorm, producer side (plain epilogue with residual R, bf16 out,
    // batch 1): C = x = bf16(alpha*A·Bᵀ + R), then h = bf16(x * no_g) in the
    // M*ldc elements after C, and no_P[m * (N/32) + c] = sum of x[m, 32c..32c+31]^2.
    const void* no_g = nullptr;
    float* no_P = nullptr;
    int split = 0;               // fp32 inputs: 1 = 3xTF32 (A = Ahi + Alo, B = Bhi + Blo split in shared
                                 // memory, C += Alo·Bhi + Ahi·Blo + Ahi·Bhi; fp32-accurate), 0 = tf32
    int tile = 0;                // CTA-pair tile: 0 auto, 1 narrow (256x256), 2 wide (512x256),
                                 // 3 narrow with a stream-K tail (instead of half-width tail tiles)
    int a_mn = 0, b_mn = 0;      // MN-major operands (bf16): A stored [K, M] / B stored [K, N], row pitch lda /
                                 // ldb (>= M / N), batch strides sa / sb
    int ksplit = 0;              // 1-CTA split-K units per tile: 0 automatic, -1 off, n > 1 forced (needs a
                                 // GemmWorkspace with counters; plain epilogue, causal 0)
};

struct alignas(64) GemmPlan {
    CUtensorMap ta;  // A: (K, M, batch)
    CUtensorMap tb;  // B: (K, N, batch)
    CUtensorMap tbh; // B with 64-row boxes (2-way sliced tail tiles of the CTA-pair paths)
    CUtensorMap tbq; // B with 32-row boxes (4-way sliced tail tiles)
    CUtensorMap tc;  // C: {64 B x 32 rows} SWIZZLE_64B boxes for the TMA-store epilogue
    GemmArgs args;
    int path = 0;    // 0 tcgen05 1-CTA, 2 tcgen05 CTA pair (cta_group::2), 1 SIMT fallback
    int bn = 256;    // N tile of the tcgen05 path
    int tiles = 0;   // output tiles (all batches)
    int grid = 0;
    int sk_tiles = 0;          // path 2: trailing tiles split by K blocks across all pairs (stream-K)
    int sk_nk = 0;             // K blocks per stream-K tile
    std::size_t ws_bytes = 0;  // workspace the stream-K tail needs (0: none)
    int tail_split = 1;        // paths 2/3: tiles of the last partial wave split into this many N-slices
    int tail_units = 0;        // number of such slices
    int ksplit = 1;            // path 0: split-K units per tile (ws_bytes of partials + per-tile counters)
    bool tbh_ok = false;
    bool tc_ok = false;
};

// Stream-K scratch: per-pair fp32 partial slots + publication flags. One per
// stream (launches on a stream are ordered); `epoch` advances per launch so
// the flags never need resetting. Zero-initialised memory.
struct GemmWorkspace {
    void* p = nullptr;
    std::size_t bytes = 0;
    unsigned epoch = 0;
    unsigned* counters = nullptr;  // split-K per-tile arrival counters (zero-initialised, reset by each reducer)
    std::size_t counter_count = 0;
};

// 3-D tiled TMA descriptor (inner, rows, batch), 128-byte swizzle.
bool encode_tma_3d(CUtensorMap* map, const void* base, int esize, std::int64_t inner, std::int64_t rows,
                   std::int64_t ld, int batch, std::int64_t bstride, int box_inner, int box_rows);
bool encode_tma_3d_swz(CUtensorMap* map, const void* base, int esize, std::int64_t inner, std::int64_t rows,
                       std::int64_t ld, int batch, std::int64_t bstride, int box_inner, int box_rows,
                       CUtensorMapSwizzle swz);

// Encodes TMA descriptors (needs a CUDA context on the target device).
cudaError_t gemm_prepare(const GemmArgs& a, GemmPlan* plan, int num_sms);
cudaError_t gemm_launch(const GemmPlan& plan, cudaStream_t s, GemmWorkspace* ws = nullptr);
double gemm_flops(const GemmArgs& a);  // algorithmic FLOPs (causal-aware)

// Fused causal attention: q, k [H, seq, hd] bf16, vt [H, hd, seq] bf16,
// out [seq, ldo] bf16 with head h at columns h*hd. Online softmax in fp32,
// P rounded to bf16 for the P·V MMA. Fast path: hd == 128, seq % 128 == 0.
struct AttnArgs {
    const void* q = nullptr;
    const void* k = nullptr;
    const void* vt = nullptr;
    void* out = nullptr;
    int heads = 0, seq = 0, hd = 0;
    std::int64_t ldo = 0;
    float scale = 1.0f;
    int causal = 1;
    float* lse = nullptr;  // optional [heads][seq]: natural-log logsumexp of each scaled score row
};
struct alignas(64) AttnPlan {
    CUtensorMap tq, tk, tv, tv2;
    AttnArgs args;
    int path = 0;  // 0 tcgen05 fused (1 CTA per 128 rows), 1 SIMT fallback, 2 tcgen05 CTA pairs (seq % 256 == 0)
    int grid = 0;  // path 2: CTAs of the persistent launch
};
cudaError_t attention_prepare(const AttnArgs& a, AttnPlan* plan);

// Fused attention backward (attention_bwd.cu): q, k [heads][seq][hd]; v, o, dO
// row-major [seq][ld] with head h at columns h*hd (v may point into a packed
// qkv); lse [heads][seq] (natural log, written by the forward with
// AttnArgs::lse); D [heads][seq] fp32 scratch. Writes dq, dk, dv [seq][ldg]
// (head h at columns h*hd). hd 128, seq % 128 == 0.
struct AttnBwdArgs {
    const void *q = nullptr, *k = nullptr, *v = nullptr, *o = nullptr, *dout = nullptr;
    std::int64_t ldv = 0, ldo = 0, lddo = 0;
    const float* lse = nullptr;
    float* D = nullptr;
    const float* rope = nullptr;  // optional [seq][hd/2][cos, sin]: dq, dk inverse-rotated in the epilogue
    void *dq = nullptr, *dk = nullptr, *dv = nullptr;
    std::int64_t ldg = 0;
    int heads = 0, seq = 0, hd = 0;
    float scale = 1.0f;
    int causal = 1;
};
struct alignas(64) AttnBwdPlan {
    CUtensorMap tq, tk, tv, tdo;
    AttnBwdArgs args;
};
cudaError_t attention_bwd_prepare(const AttnBwdArgs& a, AttnBwdPlan* plan);
cudaError_t attention_bwd_launch(const AttnBwdPlan& plan, cudaStream_t s);
double attention_bwd_flops(const AttnBwdArgs& a);
cudaError_t attention_launch(const AttnPlan& plan, cudaStream_t s);
double attention_flops(const AttnArgs& a);

// y[r] = x[r] * rsqrt(mean(x[r]^2) + eps) * w        (bf16 in/out, fp32 math)
cudaError_t rmsnorm(const void* x, const void* w, void* y, int rows, int cols, float eps, cudaStream_t s);

// P[b][i][j] = softmax_j(scale * S[b][i][j]) over j <= i (causal) or all j;
// masked entries are written as exact zeros. S fp32, P bf16.
cudaError_t softmax(const void* S, void* P, int batch, int rows, int cols, float scale, int causal,
                    cudaStream_t s);

// Two-pass blockwise softmax over bf16 score tiles (stats in natural-log
// units, fp32 float2 (m, l) per row; `causal` = diagonal tile, j <= i valid).
cudaError_t rowstats(const void* S, void* st, int rows, int cols, int causal, cudaStream_t s);
cudaError_t stats_combine(const void* const* parts, int n, void* out, int rows, cudaStream_t s);
cudaError_t softmax_apply(const void* S, const void* st, void* P, int rows, int cols, int causal, cudaStream_t s);

// Rotate-half RoPE: src [seq, ld] bf16, head h at columns col_off + h*hd;
// table fp32 [seq, hd/2, 2] = (cos, sin); out [H, seq, hd] bf16 (head-major).
// inverse: rotate by -theta (RoPE backward); tokens_out: write [seq, heads*hd].
cudaError_t rope(const void* src, const void* table, void* out, int seq, std::int64_t ld, std::int64_t col_off,
                 int heads, int hd, cudaStream_t s, int inverse = 0, int tokens_out = 0);

// out[h][d][t] = src[t][col_off + h*hd + d]  (V^T per head, bf16)
cudaError_t transpose_heads(const void* src, void* out, int seq, std::int64_t ld, std::int64_t col_off, int heads,
                            int hd, cudaStream_t s);

// out[r][c] = silu(gu[r][c]) * gu[r][cols + c]   (bf16, fp32 math)
cudaError_t silu_mul(const void* gu, void* out, int rows, int cols, cudaStream_t s);

// out = sum_i in[i] in argument order, fp32 accumulate; dtypes per tensor.
cudaError_t sum_n(const void* const* ins, int n, int in_dtype, void* out, int out_dtype, std::int64_t count,
                  cudaStream_t s);

// out = parts[0] ++ parts[1] ++ ... (n equal parts of part_bytes bytes).
cudaError_t concat(const void* const* parts, int n, std::int64_t part_bytes, void* out, cudaStream_t s);

// out[t][:] = table[tokens[t]][:]   (tokens int32, table bf16 [vocab, dim])
cudaError_t embedding(const void* tokens, const void* table, void* out, int seq, int dim, int vocab,
                      cudaStream_t s);
// Embedding + fused-RMSNorm producer outputs: [x | h = x*g | P] (see GemmArgs::no_P).
cudaError_t embedding_norm(const void* tokens, const void* table, const void* g, void* out, int seq, int dim, int vocab,
                           cudaStream_t s);

// --- training (LoRA step) tasks ---------------------------------------------
// out[b][c][r] = in[b][r][c], esize 2 or 4 bytes.
cudaError_t transpose(const void* in, void* out, int batch, int rows, int cols, int esize, cudaStream_t s);
// dx = r*(w.dy) - x r^3 mean((w.dy).x), r = rsqrt(mean(x^2)+eps) (bf16).
cudaError_t rmsnorm_bwd(const void* x, const void* w, const void* dy, void* dx, int rows, int cols, float eps,
                        cudaStream_t s);
// gu = [g | u] per row; dgu = [da*u*silu'(g) | da*silu(g)] (bf16).
cudaError_t swiglu_bwd(const void* gu, const void* da, void* dgu, int rows, int cols, cudaStream_t s);
// dS = P * (dP - rowsum(P*dP)), causal-masked entries 0 (P bf16, dS bf16).
cudaError_t softmax_bwd(const void* P, const void* dP, int dp_dtype, void* dS, int batch, int rows, int cols,
                        int causal, cudaStream_t s);
// Cross entropy: want_grad -> out = (softmax - onehot) * scale [rows, vocab];
// else out = fp32 scalar sum_r (lse_r - l_r,t) * scale (scratch: rows floats).
cudaError_t xent(const void* logits, int lg_dtype, const void* targets, void* out, int out_dtype, int rows, int vocab,
                 float scale, int want_grad, void* scratch, cudaStream_t s);

// Elementwise dtype cast (bf16 <-> f32), RNE.
cudaError_t cast(const void* in, int in_dtype, void* out, int out_dtype, std::int64_t count, cudaStream_t s);

}  // namespace tn::k
