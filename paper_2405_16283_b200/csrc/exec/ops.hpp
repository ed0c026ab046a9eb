// Op payload schema: the extra per-vertex "op" key a generator puts on
// taskgraph vertices. The reference parser ignores unknown keys
// (proj/src/taskgraph.cpp:375-389), so a taskgraph carrying payloads is still
// a valid reference input and builds a bit-identical memgraph.
//
//   {"type": "gemm", "args": [A, B (, R)], "M":..,"N":..,"K":.., "batch":1,
//    "lda","ldb","ldc","sa","sb","sc", "a_off","b_off","c_off","r_off",
//    "alpha":1.0, "in_dtype":"bf16"|"f32", "out_dtype":"bf16"|"f32",
//    "causal":0|1|2, "epilogue": "none"|"swiglu", "tile": "auto"|"narrow"|"wide",
//    "precision": "tf32"|"3xtf32" (f32 inputs: one tf32 MMA, or the fp32-accurate
//    3xTF32 split)}   swiglu: out [M, N/2] with
//    out[:, 128b+j] = silu(C[:, 256b+j]) * C[:, 256b+128+j] (gate/up rows interleaved in 128-row blocks)
//    "qkv_rope": args [x, wqkv, rope_table], "heads", hd 128, N = 3*heads*128 -> out packed
//    [rope(q) (H,M,128) | rope(k) (H,M,128) | vᵀ (H,128,M)]
//   attention may take one packed arg [qkv] with "q_off", "k_off", "v_off" (elements)
//   rope: optional "inverse": 1 (rotate by -theta), "tokens_out": 1 (write [seq, heads*hd])
// training (LoRA step) tasks:
//   {"type": "transpose", "args": [x], "batch", "rows", "cols", "out_dtype"}   out[b][c][r] = x[b][r][c]
//   {"type": "rmsnorm_bwd", "args": [x, w, dy], "rows", "cols", "eps"}
//   {"type": "swiglu_bwd", "args": [gu, da], "rows", "cols"}   gu = [g | u] rows of 2*cols
//   {"type": "softmax_bwd", "args": [P, dP], "batch", "rows", "cols", "causal", "in_dtype" (dP)}
//   {"type": "xent_grad", "args": [logits, targets], "rows", "vocab", "scale", "in_dtype", "out_dtype"}
//   {"type": "xent_loss", "args": [logits, targets], "rows", "vocab", "scale", "in_dtype"} -> f32 scalar
//   {"type": "rmsnorm", "args": [x, w], "rows", "cols", "eps"}
//   {"type": "softmax", "args": [S], "batch", "rows", "cols", "scale", "causal"}
//   {"type": "rope", "args": [src, table], "seq", "ld", "col_off", "heads", "hd"}
//   {"type": "transpose_heads", "args": [src], "seq", "ld", "col_off", "heads", "hd"}
//   {"type": "silu_mul", "args": [gu], "rows", "cols"}
//   {"type": "sum", "args": [p0, p1, ...], "count", "in_dtype", "out_dtype",
//    "offs": [element offset per arg] (optional)}
//   {"type": "concat", "args": [t0, t1, ...], "count" (elements per part), "out_dtype"}
//   {"type": "embedding", "args": [tokens, table], "seq", "dim", "vocab"}
//   {"type": "cast", "args": [x], "count", "in_dtype", "out_dtype"}
//   {"type": "attention", "args": [q, k, vt], "heads", "seq", "hd", "ldo", "scale",
//    "causal", "lse": 0|1}   q,k [H,seq,hd], vt [H,hd,seq] -> out [seq, ldo] (head h at col h*hd);
//    lse 1: followed (byte offset seq*ldo*2) by the f32 [H, seq] natural-log logsumexp of each
//    scaled score row
//   {"type": "attention_bwd", "args": [q, k, v, o_lse, dO (, rope_table)], "heads", "seq", "hd", "scale", "causal",
//    "q_off", "k_off", "v_off", "v_ld", "ldo", "do_ld"}   q,k [H,seq,hd]; v [seq, v_ld] from v_off
//    (head h at col h*hd); o_lse = an attention output with lse 1 (pitch ldo); dO [seq, do_ld] ->
//    out [seq, 3*H*hd] = [dq | dk | dv] (bf16), then f32 [H, seq] D = rowsum(dO*O) (scratch);
//    with a rope_table [seq, hd/2, (cos, sin)] dq and dk are the pre-RoPE gradients (rotate-half,
//    rotation by -theta, like rope "inverse": 1)
//   {"type": "rowstats", "args": [S], "rows", "cols", "causal"}      bf16 S -> f32 (m,l) rows
//   {"type": "stats_combine", "args": [st0, st1, ...], "rows"}        fold (m,l) in arg order
//   {"type": "softmax_apply", "args": [S, st], "rows", "cols", "causal"}  P = exp(S-m)/l, bf16
// `args` are taskgraph producer ids; every arg must be a taskgraph edge into
// the vertex. Offsets/strides are in elements. Semantics are restated in fp32
// by oracle/ops_ref.py (the CPU oracle).
#pragma once

#include <cstdint>
#include <string>
#include <unordered_map>
#include <vector>

#include "../core/types.hpp"

namespace tn {

enum class OpType : std::uint8_t {
    Gemm, RmsNorm, Softmax, Rope, TransposeHeads, SiluMul, Sum, Embedding, Cast, Attention,
    RowStats, StatsCombine, SoftmaxApply, Concat,
    Transpose, RmsNormBwd, SwigluBwd, SoftmaxBwd, XentGrad, XentLoss, AttentionBwd
};

struct OpDesc {
    OpType type = OpType::Gemm;
    std::vector<VertexId> args;
    // integer and float parameters (absent keys default to 0 / listed defaults)
    std::int64_t M = 0, N = 0, K = 0, batch = 1;
    std::int64_t lda = 0, ldb = 0, ldc = 0, sa = 0, sb = 0, sc = 0;
    std::int64_t a_off = 0, b_off = 0, c_off = 0, r_off = 0;
    std::int64_t rows = 0, cols = 0, seq = 0, ld = 0, col_off = 0, heads = 0, hd = 0, count = 0, dim = 0,
                 vocab = 0, ldo = 0;
    int causal = 0;
    int epilogue = 0;  // gemm: 0 none, 1 swiglu, 2 qkv_rope
    int tile = 0;      // gemm: CTA-pair tile choice, 0 auto, 1 narrow 256x256, 2 wide 512x256
    int a_mn = 0, b_mn = 0;  // gemm "a_major" / "b_major": "k" (default: A [M, K], B [N, K]) | "mn" (A [K, M], B [K, N])
    int ksplit = 0;    // gemm: 1-CTA split-K units per tile: 0 automatic, 1 none, n > 1 forced (partials reduced
                       // in split order)
    int split = 0;     // gemm, f32 inputs: 0 tf32, 1 3xTF32
    int inverse = 0, tokens_out = 0;  // rope
    int in_dtype = 0, out_dtype = 0;  // k::DType
    double alpha = 1.0, eps = 1e-5, scale = 1.0;
    std::vector<std::int64_t> offs;  // sum: per-argument element offsets
    std::int64_t q_off = 0, k_off = 0, v_off = 0;  // attention on a packed qkv tensor
    int lse = 0;                                   // attention: also write the row logsumexp
    std::int64_t v_ld = 0, do_ld = 0;              // attention_bwd: v / dO row pitch
    // Fused RMSNorm. Producer (gemm with residual, embedding): "norm_out": 1
    // plus a trailing gamma argument; the output holds [x | h = x*gamma | P],
    // P[m][c] = sum of x[m, 32c..32c+31]^2 (fp32, [rows, dim/32]). Consumer
    // (gemm): row m scaled by rsqrt(sum_c P[rs_row0 + m][c] / rs_dim + eps),
    // P read from argument rs_arg at byte offset rs_off with leading dim rs_ld.
    int norm_out = 0;
    int rs_arg = -1;
    std::int64_t rs_off = 0, rs_ld = 0, rs_row0 = 0, rs_dim = 0;
};

// Parses the "op" payloads of a taskgraph JSON document (vertices without an
// "op" key are skipped).
std::unordered_map<VertexId, OpDesc> parse_ops(const std::string& taskgraph_json);

const char* to_string(OpType t);

}  // namespace tn
