// Parser for the per-vertex "op" payload (schema in ops.hpp).
#include "ops.hpp"

#include <nlohmann/json.hpp>

#include "../kernels/kernels.hpp"

namespace tn {

const char* to_string(OpType t) {
    switch (t) {
        case OpType::Gemm: return "gemm";
        case OpType::RmsNorm: return "rmsnorm";
        case OpType::Softmax: return "softmax";
        case OpType::Rope: return "rope";
        case OpType::TransposeHeads: return "transpose_heads";
        case OpType::SiluMul: return "silu_mul";
        case OpType::Sum: return "sum";
        case OpType::Embedding: return "embedding";
        case OpType::Cast: return "cast";
        case OpType::Attention: return "attention";
        case OpType::RowStats: return "rowstats";
        case OpType::StatsCombine: return "stats_combine";
        case OpType::SoftmaxApply: return "softmax_apply";
        case OpType::Concat: return "concat";
        case OpType::Transpose: return "transpose";
        case OpType::RmsNormBwd: return "rmsnorm_bwd";
        case OpType::SwigluBwd: return "swiglu_bwd";
        case OpType::SoftmaxBwd: return "softmax_bwd";
        case OpType::XentGrad: return "xent_grad";
        case OpType::XentLoss: return "xent_loss";
        case OpType::AttentionBwd: return "attention_bwd";
    }
    return "?";
}

namespace {

int dtype_of(const std::string& s) {
    if (s == "bf16") return k::BF16;
    if (s == "f32") return k::F32;
    if (s == "i32") return k::I32;
    throw ParseError("unknown dtype '" + s + "'");
}

OpType type_of(const std::string& s) {
    if (s == "gemm") return OpType::Gemm;
    if (s == "rmsnorm") return OpType::RmsNorm;
    if (s == "softmax") return OpType::Softmax;
    if (s == "rope") return OpType::Rope;
    if (s == "transpose_heads") return OpType::TransposeHeads;
    if (s == "silu_mul") return OpType::SiluMul;
    if (s == "sum") return OpType::Sum;
    if (s == "embedding") return OpType::Embedding;
    if (s == "cast") return OpType::Cast;
    if (s == "attention") return OpType::Attention;
    if (s == "rowstats") return OpType::RowStats;
    if (s == "stats_combine") return OpType::StatsCombine;
    if (s == "softmax_apply") return OpType::SoftmaxApply;
    if (s == "concat") return OpType::Concat;
    if (s == "transpose") return OpType::Transpose;
    if (s == "rmsnorm_bwd") return OpType::RmsNormBwd;
    if (s == "swiglu_bwd") return OpType::SwigluBwd;
    if (s == "softmax_bwd") return OpType::SoftmaxBwd;
    if (s == "xent_grad") return OpType::XentGrad;
    if (s == "xent_loss") return OpType::XentLoss;
    if (s == "attention_bwd") return OpType::AttentionBwd;
    throw ParseError("unknown op type '" + s + "'");
}

}  // namespace

std::unordered_map<VertexId, OpDesc> parse_ops(const std::string& text) {
    std::unordered_map<VertexId, OpDesc> out;
    nlohmann::json j;
    try {
        j = nlohmann::json::parse(text);
    } catch (const nlohmann::json::parse_error& e) {
        throw ParseError(std::string("invalid JSON: ") + e.what());
    }
    try {
        for (const auto& jv : j.at("vertices")) {
            if (!jv.contains("op") || jv["op"].is_null()) continue;
            const auto& o = jv["op"];
            OpDesc d;
            d.type = type_of(o.at("type").get<std::string>());
            d.args = o.value("args", std::vector<VertexId>{});
            auto I = [&](const char* k, std::int64_t dflt) { return o.value(k, dflt); };
            d.M = I("M", 0);
            d.N = I("N", 0);
            d.K = I("K", 0);
            d.batch = I("batch", 1);
            d.lda = I("lda", 0);
            d.ldb = I("ldb", 0);
            d.ldc = I("ldc", 0);
            d.sa = I("sa", 0);
            d.sb = I("sb", 0);
            d.sc = I("sc", 0);
            d.a_off = I("a_off", 0);
            d.b_off = I("b_off", 0);
            d.c_off = I("c_off", 0);
            d.r_off = I("r_off", 0);
            d.rows = I("rows", 0);
            d.cols = I("cols", 0);
            d.seq = I("seq", 0);
            d.ld = I("ld", 0);
            d.col_off = I("col_off", 0);
            d.heads = I("heads", 0);
            d.hd = I("hd", 0);
            d.count = I("count", 0);
            d.dim = I("dim", 0);
            d.vocab = I("vocab", 0);
            d.ldo = I("ldo", 0);
            d.offs = o.value("offs", std::vector<std::int64_t>{});
            d.inverse = static_cast<int>(I("inverse", 0));
            d.tokens_out = static_cast<int>(I("tokens_out", 0));
            d.q_off = I("q_off", 0);
            d.k_off = I("k_off", 0);
            d.v_off = I("v_off", 0);
            d.lse = static_cast<int>(I("lse", 0));
            d.v_ld = I("v_ld", 0);
            d.do_ld = I("do_ld", 0);
            d.causal = static_cast<int>(I("causal", 0));
            d.norm_out = static_cast<int>(I("norm_out", 0));
            d.rs_arg = static_cast<int>(I("rs_arg", -1));
            d.rs_off = I("rs_off", 0);
            d.rs_ld = I("rs_ld", 0);
            d.rs_row0 = I("rs_row0", 0);
            d.rs_dim = I("rs_dim", 0);
            {
                const std::string ep = o.value("epilogue", std::string("none"));
                if (ep == "none") d.epilogue = 0;
                else if (ep == "swiglu") d.epilogue = 1;
                else if (ep == "qkv_rope") d.epilogue = 2;
                else throw ParseError("unknown gemm epilogue '" + ep + "'");
                const std::string tl = o.value("tile", std::string("auto"));
                if (tl == "auto") d.tile = 0;
                else if (tl == "narrow") d.tile = 1;
                else if (tl == "wide") d.tile = 2;
                else if (tl == "streamk") d.tile = 3;
                else throw ParseError("gemm tile must be auto, narrow, wide or streamk");
                auto major = [&](const char* key) {
                    const std::string v = o.value(key, std::string("k"));
                    if (v != "k" && v != "mn") throw ParseError(std::string("gemm ") + key + " must be k or mn");
                    return v == "mn" ? 1 : 0;
                };
                d.a_mn = major("a_major");
                d.b_mn = major("b_major");
                d.ksplit = o.value("ksplit", 0);
                if (d.ksplit < 0 || d.ksplit > 16) throw ParseError("gemm ksplit must be in [0, 16]");
                const std::string pr = o.value("precision", std::string("tf32"));
                if (pr == "tf32") d.split = 0;
                else if (pr == "3xtf32") d.split = 1;
                else throw ParseError("gemm precision must be tf32 or 3xtf32");
            }
            d.in_dtype = dtype_of(o.value("in_dtype", std::string("bf16")));
            d.out_dtype = dtype_of(o.value("out_dtype", std::string("bf16")));
            d.alpha = o.value("alpha", 1.0);
            d.eps = o.value("eps", 1e-5);
            d.scale = o.value("scale", 1.0);
            out[jv.at("id").get<VertexId>()] = std::move(d);
        }
    } catch (const nlohmann::json::exception& e) {
        throw ParseError(std::string("invalid op payload: ") + e.what());
    }
    return out;
}

}  // namespace tn
