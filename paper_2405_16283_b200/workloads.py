"""Taskgraph generators with op payloads.

The reference generators (proj/src/taskgraph.cpp:418-616) emit unit-sized
opaque tasks. These emit byte-sized, device-assigned taskgraphs whose kernel
vertices carry an "op" payload (schema: csrc/exec/ops.hpp); the reference
parser ignores the extra key (taskgraph.cpp:375-389), so every graph here is
also a valid input of the reference memplan and builds a bit-identical
memgraph there.

Sizes are padded to a multiple of ALIGN bytes so the planner's first-fit
offsets (prefix sums of sizes, compiler.cpp:205-216) stay 1 KiB aligned for
TMA and 128-bit access (SURVEY hard part 4).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field

import numpy as np

ALIGN = 1024
DSIZE = {"bf16": 2, "f32": 4, "i32": 4}
# cost_hint model (abstract seconds) for the virtual-time simulator only.
_PEAK_FLOPS = 1.4e15
_HBM = 6.5e12


def _pad(n: int) -> int:
    return max(ALIGN, (n + ALIGN - 1) // ALIGN * ALIGN)


@dataclass
class Tensor:
    id: int
    name: str
    shape: tuple
    dtype: str
    device: int
    init: tuple | None = None  # inputs: ("normal", std) | ("uniform", lo, hi) | ("tokens", vocab) | ("rope", theta)

    @property
    def nbytes(self) -> int:
        return int(np.prod(self.shape)) * DSIZE[self.dtype]


@dataclass
class GraphBuilder:
    device_count: int = 1
    vertices: list = field(default_factory=list)
    edges: list = field(default_factory=list)
    tensors: dict = field(default_factory=dict)
    flops: float = 0.0

    def _add(self, kind, name, shape, dtype, device, cost, op=None, src_device=-1, init=None):
        vid = len(self.vertices)
        t = Tensor(vid, name, tuple(shape), dtype, device, init)
        v = {"id": vid, "kind": kind, "device": device}
        if kind == "transfer":
            v["src_device"] = src_device
        v["output_size"] = _pad(t.nbytes)
        v["cost_hint"] = float(cost)
        if op is not None:
            v["op"] = op
        self.vertices.append(v)
        self.tensors[vid] = t
        return vid

    def input(self, name, shape, dtype="bf16", device=0, init=("normal", 0.02)):
        return self._add("input", name, shape, dtype, device, 0.0, init=init)

    def kernel(self, name, op, shape, dtype, device=0, cost=None):
        for a in op["args"]:
            if self.tensors[a].device != device:
                raise ValueError(f"{name}: argument {a} lives on device {self.tensors[a].device}")
        if cost is None:
            cost = self._cost(op, shape, dtype)
        vid = self._add("kernel", name, shape, dtype, device, cost, op=op)
        for a in dict.fromkeys(op["args"]):
            self.edges.append([a, vid])
        return vid

    def transfer(self, src, device, name=None):
        t = self.tensors[src]
        vid = self._add("transfer", name or f"{t.name}@{device}", t.shape, t.dtype, device,
                        t.nbytes / 7.7e11, src_device=t.device)
        self.edges.append([src, vid])
        return vid

    def _cost(self, op, shape, dtype):
        if op["type"] == "gemm":
            f = 2.0 * op["M"] * op["N"] * op["K"] * op.get("batch", 1) * (0.5 if op.get("causal") else 1.0)
            self.flops += f
            return f / _PEAK_FLOPS
        byts = sum(self.tensors[a].nbytes for a in op["args"]) + int(np.prod(shape)) * DSIZE[dtype]
        return byts / _HBM

    # --- ops -----------------------------------------------------------------
    def gemm(self, name, a, b, M, N, K, *, r=None, out_dtype="bf16", in_dtype="bf16", device=0, **kw):
        op = {"type": "gemm", "args": [a, b] + ([r] if r is not None else []), "M": M, "N": N, "K": K,
              "in_dtype": in_dtype, "out_dtype": out_dtype}
        op.update({k: v for k, v in kw.items() if v is not None and k != "out_shape"})
        shape = kw.get("out_shape") or (op.get("batch", 1), M, N)
        return self.kernel(name, op, shape, out_dtype, device)

    def to_json(self) -> str:
        return json.dumps({"device_count": self.device_count, "vertices": self.vertices, "edges": self.edges})

    def meta(self) -> dict:
        return {vid: {"name": t.name, "shape": list(t.shape), "dtype": t.dtype, "device": t.device,
                      "init": list(t.init) if t.init else None} for vid, t in self.tensors.items()}

    def inputs(self):
        return [t for t in self.tensors.values() if t.init is not None]

    def outputs(self):
        consumed = {p for p, _ in self.edges}
        return [vid for vid in self.tensors if vid not in consumed]


# ------------------------------------------------------------ input data ---
def input_key(t: Tensor) -> int:
    import zlib

    return zlib.crc32(t.name.encode())


_CHUNK = 1 << 22  # elements per independently seeded chunk of a large input


def _to_bf16(x: np.ndarray) -> np.ndarray:
    u = x.view(np.uint32)
    return ((u + (((u >> 16) & 1) + 0x7FFF)) >> 16).astype(np.uint16)


def make_input(t: Tensor, seed: int) -> np.ndarray:
    """Deterministic synthetic bytes for an input tensor (host numpy), keyed by
    the tensor name so equal-named inputs of different graphs agree. Random
    tensors larger than one chunk are drawn chunk by chunk from independent
    streams (seed, name key, chunk index) on a thread pool, so multi-GB weight
    sets generate at memory speed; the values do not depend on the thread count."""
    n = int(np.prod(t.shape))
    kind = t.init[0]
    if kind in ("normal", "uniform") and n > _CHUNK:
        import os
        from concurrent.futures import ThreadPoolExecutor

        out = np.empty(n, dtype=np.uint16 if t.dtype == "bf16" else np.float32)

        def fill(c):
            lo, hi = c * _CHUNK, min(n, (c + 1) * _CHUNK)
            rng = np.random.default_rng([seed, input_key(t), c])
            if kind == "normal":
                x = rng.standard_normal(hi - lo, dtype=np.float32) * np.float32(t.init[1])
            else:
                x = rng.uniform(t.init[1], t.init[2], size=hi - lo).astype(np.float32)
            out[lo:hi] = _to_bf16(x) if t.dtype == "bf16" else x

        with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as pool:
            list(pool.map(fill, range((n + _CHUNK - 1) // _CHUNK)))
        return out
    rng = np.random.default_rng([seed, input_key(t)])
    if kind == "tokens":
        return rng.integers(0, t.init[1], size=n, dtype=np.int32)
    if kind == "rope":
        S, half = t.shape[0], t.shape[1]
        theta = float(t.init[1])
        inv = theta ** (-np.arange(half, dtype=np.float64) * 2.0 / (2 * half))
        ang = np.arange(S, dtype=np.float64)[:, None] * inv[None, :]
        tab = np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)
        return tab
    if kind in ("lora_a", "lora_b"):
        # rank-`r` adapter stored padded to the tensor's full rank dimension
        # (rows >= r of A and columns >= r of B are exactly zero)
        rows, cols = t.shape
        x = (rng.standard_normal(n, dtype=np.float32) * np.float32(t.init[1])).reshape(rows, cols)
        r = int(t.init[2])
        if kind == "lora_a":
            x[r:, :] = 0
        else:
            x[:, r:] = 0
        x = x.reshape(-1)
    elif kind == "ones":
        x = np.ones(n, dtype=np.float32)
    elif kind == "normal":
        x = rng.standard_normal(n, dtype=np.float32) * np.float32(t.init[1])
    elif kind == "uniform":
        x = rng.uniform(t.init[1], t.init[2], size=n).astype(np.float32)
    else:
        raise ValueError(kind)
    if t.dtype == "bf16":
        return _to_bf16(x)
    return x


# ---------------------------------------------------------------- LLaMA ---
@dataclass
class LlamaConfig:
    dim: int = 4096
    layers: int = 32
    heads: int = 32
    ffn: int = 11008
    vocab: int = 32000
    eps: float = 1e-5
    theta: float = 10000.0

    @property
    def hd(self) -> int:
        return self.dim // self.heads


LLAMA_7B = LlamaConfig()
LLAMA_65B = LlamaConfig(dim=8192, layers=80, heads=64, ffn=22016)


def llama_prefill(cfg: LlamaConfig, seq: int, layers: int | None = None, device: int = 0,
                  std: float = 0.02, fused_attention: bool = True, fused_swiglu: bool = True,
                  fused_qkv: bool = True, fused_norm: bool = False) -> GraphBuilder:
    """One forward prefill over `seq` tokens (causal), single device.

    Per layer: rmsnorm -> QKV gemm -> rope(q), rope(k), Vᵀ -> attention ->
    O-proj gemm with fused residual -> rmsnorm -> gate/up gemm -> silu·mul ->
    down gemm + residual. Attention is one fused blockwise vertex
    (`fused_attention`, S/P stay on chip) or three vertices with the n²
    intermediates materialised (batched causal QKᵀ in fp32 with the upper
    tiles skipped -> causal softmax to bf16 P -> batched P·V into [seq, dim]),
    which the planner may offload. With `fused_swiglu` the gate/up weight
    rows are stored interleaved in 128-row blocks (gate_b, up_b, ...) and the
    gate_up GEMM's epilogue applies silu(g)*u, so the [seq, 2*ffn]
    intermediate never reaches HBM (requires ffn % 128 == 0). With
    `fused_qkv` (hd 128, fused attention) the QKV GEMM's epilogue applies RoPE
    to q/k and transposes v, writing one packed [q | k | vᵀ] tensor that the
    attention vertex reads by offset.
    With `fused_norm` (on top of fused_qkv and fused_swiglu) there are no
    RMSNorm vertices: every producer of the residual stream (the embedding,
    each attn_out / ffn_out GEMM) writes [x | h = x*gamma | P] where gamma is
    the next norm's weight and P the per-32-column sums of x^2; the consuming
    GEMM reads h and scales its output rows by rsqrt(sum P / dim + eps) in
    the epilogue (see _llama_fused_norm). Off by default: it removes the 65
    RMSNorm launches (1.5 ms of the 7B step) but the extra h / P stores and
    row-scale loads in the GEMM epilogues cost more — paired A/B on one B200
    (tools/ab_fused_norm.py): 51.24 ms unfused vs 52.62 ms fused per step.
    Head: final rmsnorm -> last-token logits (fp32). Weights are graph inputs
    (cold in host RAM, materialised by H2D at dispatch).
    """
    L = cfg.layers if layers is None else layers
    d, H, hd, f, V, S = cfg.dim, cfg.heads, cfg.hd, cfg.ffn, cfg.vocab, seq
    if (fused_norm and fused_qkv and fused_swiglu and fused_attention and hd == 128 and f % 128 == 0
            and d % 256 == 0 and S >= 256):  # norm_out producers need the CTA-pair GEMM path (M >= 256)
        return _llama_fused_norm(cfg, S, L, device, std)
    g = GraphBuilder(device_count=1)
    dev = device
    tok = g.input("tokens", (S,), "i32", dev, init=("tokens", V))
    emb = g.input("tok_embeddings", (V, d), "bf16", dev, init=("normal", std))
    rope_tab = g.input("rope_table", (S, hd // 2, 2), "f32", dev, init=("rope", cfg.theta))
    x = g.kernel("embed", {"type": "embedding", "args": [tok, emb], "seq": S, "dim": d, "vocab": V}, (S, d), "bf16", dev)
    for l in range(L):
        p = f"layers.{l}."
        wn1 = g.input(p + "attention_norm", (d,), "bf16", dev, init=("normal", 1.0))
        wqkv = g.input(p + "wqkv", (3 * d, d), "bf16", dev, init=("normal", std))
        wo = g.input(p + "wo", (d, d), "bf16", dev, init=("normal", std))
        wn2 = g.input(p + "ffn_norm", (d,), "bf16", dev, init=("normal", 1.0))
        w13 = g.input(p + "w13", (2 * f, d), "bf16", dev, init=("normal", std))
        w2 = g.input(p + "w2", (d, f), "bf16", dev, init=("normal", std))
        h = g.kernel(p + "attn_norm_out", {"type": "rmsnorm", "args": [x, wn1], "rows": S, "cols": d, "eps": cfg.eps},
                     (S, d), "bf16", dev)
        if fused_qkv and fused_attention and hd == 128:
            qkv = g.gemm(p + "qkv_rope", h, wqkv, S, 3 * d, d, r=rope_tab, epilogue="qkv_rope", heads=H,
                         out_shape=(3, H, S, hd), device=dev)
            sec = H * S * hd
            op = {"type": "attention", "args": [qkv], "q_off": 0, "k_off": sec, "v_off": 2 * sec, "heads": H,
                  "seq": S, "hd": hd, "ldo": d, "scale": 1.0 / math.sqrt(hd), "causal": 1}
            o = g.kernel(p + "attn", op, (S, d), "bf16", dev, cost=2.0 * S * S * hd * H / _PEAK_FLOPS)
            g.flops += 2.0 * S * S * hd * H * (1 + 1 / S)
            x = g.gemm(p + "attn_out", o, wo, S, d, d, r=x, out_shape=(S, d), device=dev)
            h2 = g.kernel(p + "ffn_norm_out", {"type": "rmsnorm", "args": [x, wn2], "rows": S, "cols": d,
                                               "eps": cfg.eps}, (S, d), "bf16", dev)
            x = _ffn(g, p, h2, w13, w2, x, S, d, f, dev, fused_swiglu)
            continue
        qkv = g.gemm(p + "qkv", h, wqkv, S, 3 * d, d, out_shape=(S, 3 * d), device=dev)
        q = g.kernel(p + "q_rope", {"type": "rope", "args": [qkv, rope_tab], "seq": S, "ld": 3 * d, "col_off": 0,
                                    "heads": H, "hd": hd}, (H, S, hd), "bf16", dev)
        k = g.kernel(p + "k_rope", {"type": "rope", "args": [qkv, rope_tab], "seq": S, "ld": 3 * d, "col_off": d,
                                    "heads": H, "hd": hd}, (H, S, hd), "bf16", dev)
        vt = g.kernel(p + "v_t", {"type": "transpose_heads", "args": [qkv], "seq": S, "ld": 3 * d, "col_off": 2 * d,
                                  "heads": H, "hd": hd}, (H, hd, S), "bf16", dev)
        if fused_attention:
            op = {"type": "attention", "args": [q, k, vt], "heads": H, "seq": S, "hd": hd, "ldo": d,
                  "scale": 1.0 / math.sqrt(hd), "causal": 1}
            o = g.kernel(p + "attn", op, (S, d), "bf16", dev, cost=2.0 * S * S * hd * H / _PEAK_FLOPS)
            g.flops += 2.0 * S * S * hd * H * (1 + 1 / S)
        else:
            sc = g.gemm(p + "scores", q, k, S, S, hd, batch=H, sa=S * hd, sb=S * hd, sc=S * S, out_dtype="f32",
                        causal=1, out_shape=(H, S, S), device=dev)
            pr = g.kernel(p + "probs", {"type": "softmax", "args": [sc], "batch": H, "rows": S, "cols": S,
                                        "scale": 1.0 / math.sqrt(hd), "causal": 1}, (H, S, S), "bf16", dev)
            o = g.gemm(p + "attn", pr, vt, S, hd, S, batch=H, lda=S, ldb=S, ldc=d, sa=S * S, sb=hd * S, sc=hd,
                       causal=2, out_shape=(S, d), device=dev)
        x = g.gemm(p + "attn_out", o, wo, S, d, d, r=x, out_shape=(S, d), device=dev)
        h2 = g.kernel(p + "ffn_norm_out", {"type": "rmsnorm", "args": [x, wn2], "rows": S, "cols": d, "eps": cfg.eps},
                      (S, d), "bf16", dev)
        x = _ffn(g, p, h2, w13, w2, x, S, d, f, dev, fused_swiglu)
    wn = g.input("norm", (d,), "bf16", dev, init=("normal", 1.0))
    wout = g.input("output", (V, d), "bf16", dev, init=("normal", std))
    hn = g.kernel("final_norm", {"type": "rmsnorm", "args": [x, wn], "rows": S, "cols": d, "eps": cfg.eps},
                  (S, d), "bf16", dev)
    g.gemm("logits", hn, wout, 1, V, d, a_off=(S - 1) * d, out_dtype="f32", out_shape=(1, V), device=dev)
    return g


def _ffn(g, p, h2, w13, w2, x, S, d, f, dev, fused_swiglu):
    if fused_swiglu and f % 128 == 0:
        a = g.gemm(p + "act", h2, w13, S, 2 * f, d, epilogue="swiglu", out_shape=(S, f), device=dev)
    else:
        gu = g.gemm(p + "gate_up", h2, w13, S, 2 * f, d, out_shape=(S, 2 * f), device=dev)
        a = g.kernel(p + "act", {"type": "silu_mul", "args": [gu], "rows": S, "cols": f}, (S, f), "bf16", dev)
    return g.gemm(p + "ffn_out", a, w2, S, d, f, r=x, out_shape=(S, d), device=dev)


def _llama_fused_norm(cfg: LlamaConfig, S: int, L: int, dev: int, std: float) -> GraphBuilder:
    """llama_prefill with every RMSNorm fused into its producer / consumer
    (same inputs and names as the unfused graph). Residual-stream vertices
    hold [x (S x d bf16) | h = bf16(x * gamma) | P (S x d/32 fp32)]:
      embed:    x = table rows                 (gamma: layer 0 attention_norm)
      attn_out: x = o·woᵀ + x_prev             (gamma: ffn_norm)
      ffn_out:  x = act·w2ᵀ + x_prev           (gamma: next attention_norm / final norm)
    and the consumers (qkv_rope, swiglu, the last-token head) read h and
    scale row m by rsqrt(sum_c P[c][m] / d + eps) — RMSNorm(x) W^T =
    diag(r) (x * gamma) W^T."""
    d, H, hd, f, V = cfg.dim, cfg.heads, cfg.hd, cfg.ffn, cfg.vocab
    g = GraphBuilder(device_count=1)
    xn_shape = (2 * S * d + 2 * S * (d // 32),)  # [x | h | P] in bf16-sized units
    p_off = 2 * S * d * 2                          # byte offset of P
    rs = {"rs_arg": 0, "rs_off": p_off, "rs_ld": d // 32, "rs_dim": d, "eps": cfg.eps}
    tok = g.input("tokens", (S,), "i32", dev, init=("tokens", V))
    emb = g.input("tok_embeddings", (V, d), "bf16", dev, init=("normal", std))
    rope_tab = g.input("rope_table", (S, hd // 2, 2), "f32", dev, init=("rope", cfg.theta))
    wn1 = g.input("layers.0.attention_norm", (d,), "bf16", dev, init=("normal", 1.0))
    x = g.kernel("embed", {"type": "embedding", "args": [tok, emb, wn1], "seq": S, "dim": d, "vocab": V,
                           "norm_out": 1}, xn_shape, "bf16", dev)
    for l in range(L):
        p = f"layers.{l}."
        wqkv = g.input(p + "wqkv", (3 * d, d), "bf16", dev, init=("normal", std))
        wo = g.input(p + "wo", (d, d), "bf16", dev, init=("normal", std))
        wn2 = g.input(p + "ffn_norm", (d,), "bf16", dev, init=("normal", 1.0))
        w13 = g.input(p + "w13", (2 * f, d), "bf16", dev, init=("normal", std))
        w2 = g.input(p + "w2", (d, f), "bf16", dev, init=("normal", std))
        qkv = g.gemm(p + "qkv_rope", x, wqkv, S, 3 * d, d, r=rope_tab, epilogue="qkv_rope", heads=H,
                     a_off=S * d, out_shape=(3, H, S, hd), device=dev, **rs)
        sec = H * S * hd
        op = {"type": "attention", "args": [qkv], "q_off": 0, "k_off": sec, "v_off": 2 * sec, "heads": H,
              "seq": S, "hd": hd, "ldo": d, "scale": 1.0 / math.sqrt(hd), "causal": 1}
        o = g.kernel(p + "attn", op, (S, d), "bf16", dev, cost=2.0 * S * S * hd * H / _PEAK_FLOPS)
        g.flops += 2.0 * S * S * hd * H * (1 + 1 / S)
        x = g.kernel(p + "attn_out", {"type": "gemm", "args": [o, wo, x, wn2], "M": S, "N": d, "K": d,
                                      "in_dtype": "bf16", "out_dtype": "bf16", "norm_out": 1},
                     xn_shape, "bf16", dev, cost=2.0 * S * d * d / _PEAK_FLOPS)
        g.flops += 2.0 * S * d * d
        a = g.gemm(p + "act", x, w13, S, 2 * f, d, epilogue="swiglu", a_off=S * d, out_shape=(S, f), device=dev, **rs)
        gn = (g.input(f"layers.{l + 1}.attention_norm", (d,), "bf16", dev, init=("normal", 1.0)) if l + 1 < L
              else g.input("norm", (d,), "bf16", dev, init=("normal", 1.0)))
        x = g.kernel(p + "ffn_out", {"type": "gemm", "args": [a, w2, x, gn], "M": S, "N": d, "K": f,
                                     "in_dtype": "bf16", "out_dtype": "bf16", "norm_out": 1},
                     xn_shape, "bf16", dev, cost=2.0 * S * d * f / _PEAK_FLOPS)
        g.flops += 2.0 * S * d * f
    wout = g.input("output", (V, d), "bf16", dev, init=("normal", std))
    g.gemm("logits", x, wout, 1, V, d, a_off=S * d + (S - 1) * d, out_dtype="f32", out_shape=(1, V), device=dev,
           rs_row0=S - 1, **rs)
    return g


def llama_prefill_tp(cfg: LlamaConfig, seq: int, tp: int, layers: int | None = None,
                     std: float = 0.02, fused_qkv: bool = True) -> GraphBuilder:
    """Config 3: tensor-parallel prefill over `tp` memgraph devices (Megatron
    layout). QKV / gate-up are column-parallel (each device owns
    heads / ffn columns), O / down are row-parallel and produce per-device
    partial sums. The all-reduce is explicit memgraph vertices — no NCCL:
      reduce-scatter: device r receives row block r of every other device's
        partial (Transfer, NVLink peer copy) and adds them in fixed device
        order plus its residual rows (`sum` with per-arg offsets);
      all-gather: every device receives the other reduced row blocks
        (Transfer) and concatenates them (`concat`) into its replica of x.
    The residual stream x is replicated; weights are per-device inputs
    (host-resident, sliced exactly like a TP checkpoint shard). The final norm
    and last-token logits run on device 0. With `fused_qkv` (hd 128) each
    device's QKV GEMM applies RoPE and transposes V in its epilogue (packed
    [q | k | vᵀ] read by offset in attention), as in llama_prefill."""
    L = cfg.layers if layers is None else layers
    d, H, hd, f, V, S = cfg.dim, cfg.heads, cfg.hd, cfg.ffn, cfg.vocab, seq
    assert H % tp == 0 and f % tp == 0 and S % tp == 0
    Hl, fl, Sb = H // tp, f // tp, S // tp
    dl = Hl * hd
    g = GraphBuilder(device_count=tp)
    x = {}
    tab = {}
    for r in range(tp):
        tok = g.input(f"tokens@{r}", (S,), "i32", r, init=("tokens", V))
        emb = g.input(f"tok_embeddings@{r}", (V, d), "bf16", r, init=("normal", std))
        tab[r] = g.input(f"rope_table@{r}", (S, hd // 2, 2), "f32", r, init=("rope", cfg.theta))
        x[r] = g.kernel(f"embed@{r}", {"type": "embedding", "args": [tok, emb], "seq": S, "dim": d, "vocab": V},
                        (S, d), "bf16", r)

    def allreduce(name, partial, resid, need=None):
        """partial[r][b]: [Sb, d] row block b of device r's partial sum;
        `need`: devices that receive the gathered result (default all)."""
        red = {}
        for b in range(tp):
            args = [partial[r][b] if r == b else g.transfer(partial[r][b], b, f"{name}.rs[{r}->{b}]") for r in range(tp)]
            args.append(resid[b])
            red[b] = g.kernel(f"{name}.reduced[{b}]", {"type": "sum", "args": args, "count": Sb * d,
                                                        "offs": [0] * tp + [b * Sb * d], "in_dtype": "bf16",
                                                        "out_dtype": "bf16"}, (Sb, d), "bf16", b)
        out = {}
        for r in (range(tp) if need is None else need):
            parts = [red[b] if b == r else g.transfer(red[b], r, f"{name}.ag[{b}->{r}]") for b in range(tp)]
            out[r] = g.kernel(f"{name}.x@{r}", {"type": "concat", "args": parts, "count": Sb * d, "out_dtype": "bf16"},
                              (S, d), "bf16", r)
        return out

    for l in range(L):
        p = f"layers.{l}."
        o = {}
        for r in range(tp):
            wn1 = g.input(p + f"attention_norm@{r}", (d,), "bf16", r, init=("normal", 1.0))
            wqkv = g.input(p + f"wqkv@{r}", (3 * dl, d), "bf16", r, init=("normal", std))
            h = g.kernel(p + f"attn_norm_out@{r}", {"type": "rmsnorm", "args": [x[r], wn1], "rows": S, "cols": d,
                                                     "eps": cfg.eps}, (S, d), "bf16", r)
            if fused_qkv and hd == 128:
                qkv = g.gemm(p + f"qkv_rope@{r}", h, wqkv, S, 3 * dl, d, r=tab[r], epilogue="qkv_rope", heads=Hl,
                             out_shape=(3, Hl, S, hd), device=r)
                sec = Hl * S * hd
                o[r] = g.kernel(p + f"attn@{r}", {"type": "attention", "args": [qkv], "q_off": 0, "k_off": sec,
                                                  "v_off": 2 * sec, "heads": Hl, "seq": S, "hd": hd, "ldo": dl,
                                                  "scale": 1.0 / math.sqrt(hd), "causal": 1}, (S, dl), "bf16", r,
                                cost=2.0 * S * S * hd * Hl / _PEAK_FLOPS)
                g.flops += 2.0 * S * S * hd * Hl * (1 + 1 / S)
                continue
            qkv = g.gemm(p + f"qkv@{r}", h, wqkv, S, 3 * dl, d, out_shape=(S, 3 * dl), device=r)
            q = g.kernel(p + f"q_rope@{r}", {"type": "rope", "args": [qkv, tab[r]], "seq": S, "ld": 3 * dl, "col_off": 0,
                                             "heads": Hl, "hd": hd}, (Hl, S, hd), "bf16", r)
            k = g.kernel(p + f"k_rope@{r}", {"type": "rope", "args": [qkv, tab[r]], "seq": S, "ld": 3 * dl,
                                             "col_off": dl, "heads": Hl, "hd": hd}, (Hl, S, hd), "bf16", r)
            vt = g.kernel(p + f"v_t@{r}", {"type": "transpose_heads", "args": [qkv], "seq": S, "ld": 3 * dl,
                                           "col_off": 2 * dl, "heads": Hl, "hd": hd}, (Hl, hd, S), "bf16", r)
            o[r] = g.kernel(p + f"attn@{r}", {"type": "attention", "args": [q, k, vt], "heads": Hl, "seq": S, "hd": hd,
                                              "ldo": dl, "scale": 1.0 / math.sqrt(hd), "causal": 1}, (S, dl), "bf16", r,
                            cost=2.0 * S * S * hd * Hl / _PEAK_FLOPS)
            g.flops += 2.0 * S * S * hd * Hl * (1 + 1 / S)
        partial = {}
        for r in range(tp):
            wo = g.input(p + f"wo@{r}", (d, dl), "bf16", r, init=("normal", std))
            partial[r] = {b: g.gemm(p + f"attn_out_partial@{r}[{b}]", o[r], wo, Sb, d, dl, a_off=b * Sb * dl,
                                    out_shape=(Sb, d), device=r) for b in range(tp)}
        x = allreduce(p + "attn_ar", partial, x)
        a = {}
        for r in range(tp):
            wn2 = g.input(p + f"ffn_norm@{r}", (d,), "bf16", r, init=("normal", 1.0))
            w13 = g.input(p + f"w13@{r}", (2 * fl, d), "bf16", r, init=("normal", std))
            h2 = g.kernel(p + f"ffn_norm_out@{r}", {"type": "rmsnorm", "args": [x[r], wn2], "rows": S, "cols": d,
                                                     "eps": cfg.eps}, (S, d), "bf16", r)
            gu = g.gemm(p + f"gate_up@{r}", h2, w13, S, 2 * fl, d, out_shape=(S, 2 * fl), device=r)
            a[r] = g.kernel(p + f"act@{r}", {"type": "silu_mul", "args": [gu], "rows": S, "cols": fl}, (S, fl), "bf16", r)
        partial = {}
        for r in range(tp):
            w2 = g.input(p + f"w2@{r}", (d, fl), "bf16", r, init=("normal", std))
            partial[r] = {b: g.gemm(p + f"ffn_out_partial@{r}[{b}]", a[r], w2, Sb, d, fl, a_off=b * Sb * fl,
                                    out_shape=(Sb, d), device=r) for b in range(tp)}
        x = allreduce(p + "ffn_ar", partial, x, need=[0] if l == L - 1 else None)
    wn = g.input("norm", (d,), "bf16", 0, init=("normal", 1.0))
    wout = g.input("output", (V, d), "bf16", 0, init=("normal", std))
    hn = g.kernel("final_norm", {"type": "rmsnorm", "args": [x[0], wn], "rows": S, "cols": d, "eps": cfg.eps},
                  (S, d), "bf16", 0)
    g.gemm("logits", hn, wout, 1, V, d, a_off=(S - 1) * d, out_dtype="f32", out_shape=(1, V), device=0)
    return g


def llama_lora_step(cfg: LlamaConfig, seq: int, layers: int | None = None, rank: int = 16, rank_pad: int = 64,
                    lora_alpha: float = 16.0, std: float = 0.02, device: int = 0,
                    recompute_attention: bool = True, recompute_ffn: bool = True,
                    recompute_qkv: bool = True, mn_major: bool = True, prefetch: int = 0,
                    recompute_norms: bool = True, bwd_prefetch: int = 0,
                    fused_attention: bool | None = None) -> GraphBuilder:
    """Config 4: one LoRA fine-tuning step (forward + backward) of a LLaMA
    model over `seq` tokens, rank-`rank` adapters on the fused QKV projection
    and on both FFN projections ("rank 16 on Q,K,V,FFN"), frozen
    base weights, mean token cross-entropy. Every activation the backward
    needs is a vertex output that stays live from the forward to the
    backward, so under an HBM cap the planner offloads it to host RAM and
    reloads it (activation offload). Outputs: the loss and dA/dB of every
    adapter. Adapters are stored zero-padded to `rank_pad` (the tensor-core
    K atom); padding rows/columns are exactly zero.

    Backward GEMMs need transposed operands (dX = dY·W, dW = dYᵀ·X): read in
    place MN-major (`mn_major`, default) or, with mn_major=False, through
    explicit `transpose` vertices. The attention backward is one fused
    `attention_bwd` vertex (`fused_attention`, default) or, with
    fused_attention=False, dP = dO·Vᵀ -> softmax_bwd -> dQ = dS·K,
    dK = dSᵀ·Q, dV = Pᵀ·dO over materialised n² tiles.

    With `recompute_attention` (default; SURVEY §8d "fwd + bwd with
    recompute") the backward recomputes P = softmax(scale·QKᵀ) from the saved
    q and k instead of keeping the forward's P (H·S² bf16 = 1 GB per 7B layer)
    live across the step: the planner then never offloads the n² tensor, at the
    cost of one more causal scores GEMM + softmax per layer. The recomputed P
    is bitwise the forward's (same kernels, same inputs).

    `recompute_ffn` / `recompute_qkv` (defaults) extend the recompute to the
    gate/up projection + SwiGLU (gu, act from the saved h2 and U2) and to the
    QKV projection + RoPE (qkv, q, k from the saved h and U1): each layer then
    keeps only the norm inputs / outputs and the rank-R adapter activations
    live across the step. On the 7B step under 16 GiB this cuts the planned
    activation offload from 20.6 to 6.9 GB (simulated step 0.82 -> 0.38 s) for
    +28 % FLOPs (one more gate/up and QKV GEMM per layer).

    `mn_major` (default): the backward GEMMs read transposed operands in place
    ("a_major" / "b_major": "mn", e.g. dX = dY·W with W stored [out, in]) instead
    of through explicit transpose vertices (≈1,000 vertices and ~3 GB of
    transposed copies per layer on the 7B step, n² probability tiles included).

    `recompute_norms` (default): the backward recomputes both RMSNorm outputs
    from the saved residual stream (x, x1), so only x, x1 and the rank-R
    adapter activations stay live across the step. `prefetch` /
    `bwd_prefetch`: list the next layers' weight inputs / recompute GEMMs
    that many layers early in the taskgraph order (planner-visible prefetch;
    measured neutral on the 7B step, default 0).

    `fused_attention` (default when hd == 128 and seq % 128 == 0): the
    forward runs the fused attention kernel, and the backward recomputes it
    with the per-row logsumexp ("lse": 1) and takes dq|dk|dv from ONE fused
    `attention_bwd` vertex (csrc/kernels/attention_bwd.cu) instead of the
    materialised scores / probs / dP / dS chain: no n² tensor exists at all,
    so the 7B step under 16 GiB needs no activation offload (step 0.52 ->
    0.39 s)."""
    if fused_attention is None:
        fused_attention = mn_major and cfg.hd == 128 and seq % 128 == 0
    g = GraphBuilder(device_count=1)
    _lora_step_into(g, cfg, seq, layers, rank, rank_pad, lora_alpha, std, device, "", recompute_attention,
                    recompute_ffn, recompute_qkv, mn_major, prefetch, recompute_norms, bwd_prefetch,
                    fused_attention)
    return g


def llama_lora_step_dp(cfg: LlamaConfig, seq: int, dp: int, layers: int | None = None, rank: int = 16,
                       rank_pad: int = 64, lora_alpha: float = 16.0, std: float = 0.02,
                       recompute_attention: bool = True, recompute_ffn: bool = True,
                       recompute_qkv: bool = True, mn_major: bool = True, prefetch: int = 0,
                    recompute_norms: bool = True, bwd_prefetch: int = 0,
                    fused_attention: bool | None = None) -> GraphBuilder:
    """Config 4 over `dp` devices (data parallel): every memgraph
    device runs the full LoRA step on its own sequence (tokens/targets
    `@r`; the frozen weights and adapters are the same tensors on every device,
    each device materialising its copy from host), then the per-device loss
    and adapter gradients are summed on device 0 in fixed device order — the
    gradient all-reduce as explicit Transfer vertices (NVLink peer copies)
    into `sum` combines, no NCCL. Outputs: the summed loss and gradients
    (same names as llama_lora_step's). Global batch = dp sequences."""
    if fused_attention is None:
        fused_attention = mn_major and cfg.hd == 128 and seq % 128 == 0
    g = GraphBuilder(device_count=dp)
    outs = [_lora_step_into(g, cfg, seq, layers, rank, rank_pad, lora_alpha, std, r, f"@{r}" if r else "",
                            recompute_attention, recompute_ffn, recompute_qkv, mn_major, prefetch,
                            recompute_norms, bwd_prefetch, fused_attention) for r in range(dp)]
    for name, v0 in outs[0].items():
        t = g.tensors[v0]
        n = int(np.prod(t.shape))
        args = [v0] + [g.transfer(outs[r][name], 0, f"{name}@{r}->0") for r in range(1, dp)]
        g.kernel(f"{name}.sum", {"type": "sum", "args": args, "count": n, "in_dtype": t.dtype,
                                 "out_dtype": t.dtype}, t.shape, t.dtype, 0)
    return g


def _lora_step_into(g: GraphBuilder, cfg: LlamaConfig, seq: int, layers, rank, rank_pad, lora_alpha, std, device,
                    data_sfx, recompute_attention=True, recompute_ffn=False, recompute_qkv=False,
                    mn_major=False, prefetch=0, recompute_norms=False, bwd_prefetch=0,
                    fused_attention=False) -> dict:
    """Appends one LoRA step on `device` to `g`; returns {output name: vid}
    (the loss and every adapter gradient)."""
    L = cfg.layers if layers is None else layers
    d, H, hd, f, V, S = cfg.dim, cfg.heads, cfg.hd, cfg.ffn, cfg.vocab, seq
    R, sc = rank_pad, lora_alpha / rank
    scale = 1.0 / math.sqrt(hd)
    dev = device
    results = {}
    if fused_attention and not (mn_major and hd == 128 and S % 128 == 0):
        raise ValueError("fused_attention needs mn_major, hd 128 and seq % 128 == 0")
    attn_flops = 2.0 * S * S * hd * H * (1 + 1 / S)  # causal: QKᵀ and PV, half each

    def tr(name, x, rows, cols, batch=1, dt="bf16"):
        return g.kernel(name, {"type": "transpose", "args": [x], "batch": batch, "rows": rows, "cols": cols,
                               "out_dtype": dt}, (batch, cols, rows), dt, dev)

    def rms(name, x, w):
        return g.kernel(name, {"type": "rmsnorm", "args": [x, w], "rows": S, "cols": d, "eps": cfg.eps}, (S, d),
                        "bf16", dev)

    def rms_bwd(name, x, w, dy):
        return g.kernel(name, {"type": "rmsnorm_bwd", "args": [x, w, dy], "rows": S, "cols": d, "eps": cfg.eps},
                        (S, d), "bf16", dev)

    def add(name, a, b):
        return g.kernel(name, {"type": "sum", "args": [a, b], "count": S * d, "in_dtype": "bf16",
                               "out_dtype": "bf16"}, (S, d), "bf16", dev)

    tok = g.input("tokens" + data_sfx, (S,), "i32", dev, init=("tokens", V))
    tgt = g.input("targets" + data_sfx, (S,), "i32", dev, init=("tokens", V))
    emb = g.input("tok_embeddings", (V, d), "bf16", dev, init=("normal", std))
    rope_tab = g.input("rope_table", (S, hd // 2, 2), "f32", dev, init=("rope", cfg.theta))
    x = g.kernel("embed", {"type": "embedding", "args": [tok, emb], "seq": S, "dim": d, "vocab": V}, (S, d), "bf16", dev)

    saved = []
    ws = {}

    def layer_weights(l):
        p = f"layers.{l}."
        return {
            "wn1": g.input(p + "attention_norm", (d,), "bf16", dev, init=("normal", 1.0)),
            "wqkv": g.input(p + "wqkv", (3 * d, d), "bf16", dev, init=("normal", std)),
            "wo": g.input(p + "wo", (d, d), "bf16", dev, init=("normal", std)),
            "wn2": g.input(p + "ffn_norm", (d,), "bf16", dev, init=("normal", 1.0)),
            "w13": g.input(p + "w13", (2 * f, d), "bf16", dev, init=("normal", std)),
            "w2": g.input(p + "w2", (d, f), "bf16", dev, init=("normal", std)),
            "A1": g.input(p + "lora_qkv.A", (R, d), "bf16", dev, init=("lora_a", std, rank)),
            "B1": g.input(p + "lora_qkv.B", (3 * d, R), "bf16", dev, init=("lora_b", std, rank)),
            "A2": g.input(p + "lora_w13.A", (R, d), "bf16", dev, init=("lora_a", std, rank)),
            "B2": g.input(p + "lora_w13.B", (2 * f, R), "bf16", dev, init=("lora_b", std, rank)),
            "A3": g.input(p + "lora_w2.A", (R, f), "bf16", dev, init=("lora_a", std, rank)),
            "B3": g.input(p + "lora_w2.B", (d, R), "bf16", dev, init=("lora_b", std, rank)),
        }

    for l in range(L):
        p = f"layers.{l}."
        for j in range(l, min(L, l + 1 + prefetch)):
            if j not in ws:
                ws[j] = layer_weights(j)
        w = ws.pop(l)
        a = {"x": x}
        a["h"] = rms(p + "attn_norm_out", x, w["wn1"])
        base = g.gemm(p + "qkv_base", a["h"], w["wqkv"], S, 3 * d, d, out_shape=(S, 3 * d), device=dev)
        a["U1"] = g.gemm(p + "lora_qkv.U", a["h"], w["A1"], S, R, d, out_shape=(S, R), device=dev)
        a["qkv"] = g.gemm(p + "qkv", a["U1"], w["B1"], S, 3 * d, R, r=base, alpha=sc, out_shape=(S, 3 * d), device=dev)
        a["q"] = g.kernel(p + "q_rope", {"type": "rope", "args": [a["qkv"], rope_tab], "seq": S, "ld": 3 * d,
                                         "col_off": 0, "heads": H, "hd": hd}, (H, S, hd), "bf16", dev)
        a["k"] = g.kernel(p + "k_rope", {"type": "rope", "args": [a["qkv"], rope_tab], "seq": S, "ld": 3 * d,
                                         "col_off": d, "heads": H, "hd": hd}, (H, S, hd), "bf16", dev)
        vt = g.kernel(p + "v_t", {"type": "transpose_heads", "args": [a["qkv"]], "seq": S, "ld": 3 * d,
                                  "col_off": 2 * d, "heads": H, "hd": hd}, (H, hd, S), "bf16", dev)
        if fused_attention:  # the fused kernel; the backward recomputes it with the row logsumexp
            o = g.kernel(p + "attn", {"type": "attention", "args": [a["q"], a["k"], vt], "heads": H, "seq": S,
                                      "hd": hd, "ldo": d, "scale": scale, "causal": 1}, (S, d), "bf16", dev,
                         cost=attn_flops / _PEAK_FLOPS)
            g.flops += attn_flops
        else:
            scr = g.gemm(p + "scores", a["q"], a["k"], S, S, hd, batch=H, sa=S * hd, sb=S * hd, sc=S * S,
                         out_dtype="f32", causal=1, out_shape=(H, S, S), device=dev)
            a["P"] = g.kernel(p + "probs", {"type": "softmax", "args": [scr], "batch": H, "rows": S, "cols": S,
                                            "scale": scale, "causal": 1}, (H, S, S), "bf16", dev)
            o = g.gemm(p + "attn", a["P"], vt, S, hd, S, batch=H, lda=S, ldb=S, ldc=d, sa=S * S, sb=hd * S, sc=hd,
                       causal=2, out_shape=(S, d), device=dev)
        a["x1"] = g.gemm(p + "attn_out", o, w["wo"], S, d, d, r=x, out_shape=(S, d), device=dev)
        a["h2"] = rms(p + "ffn_norm_out", a["x1"], w["wn2"])
        gub = g.gemm(p + "gate_up_base", a["h2"], w["w13"], S, 2 * f, d, out_shape=(S, 2 * f), device=dev)
        a["U2"] = g.gemm(p + "lora_w13.U", a["h2"], w["A2"], S, R, d, out_shape=(S, R), device=dev)
        a["gu"] = g.gemm(p + "gate_up", a["U2"], w["B2"], S, 2 * f, R, r=gub, alpha=sc, out_shape=(S, 2 * f), device=dev)
        a["act"] = g.kernel(p + "act", {"type": "silu_mul", "args": [a["gu"]], "rows": S, "cols": f}, (S, f), "bf16", dev)
        y0 = g.gemm(p + "ffn_base", a["act"], w["w2"], S, d, f, r=a["x1"], out_shape=(S, d), device=dev)
        a["U3"] = g.gemm(p + "lora_w2.U", a["act"], w["A3"], S, R, f, out_shape=(S, R), device=dev)
        x = g.gemm(p + "ffn_out", a["U3"], w["B3"], S, d, R, r=y0, alpha=sc, out_shape=(S, d), device=dev)
        saved.append((p, w, a))
    wn = g.input("norm", (d,), "bf16", dev, init=("normal", 1.0))
    wout = g.input("output", (V, d), "bf16", dev, init=("normal", std))
    xL = x
    hn = rms("final_norm", xL, wn)
    logits = g.gemm("logits", hn, wout, S, V, d, out_shape=(S, V), device=dev)
    results["loss"] = g.kernel("loss", {"type": "xent_loss", "args": [logits, tgt], "rows": S, "vocab": V,
                                        "scale": 1.0 / S, "in_dtype": "bf16"}, (1,), "f32", dev)
    dlog = g.kernel("dlogits", {"type": "xent_grad", "args": [logits, tgt], "rows": S, "vocab": V, "scale": 1.0 / S,
                                "in_dtype": "bf16", "out_dtype": "bf16"}, (S, V), "bf16", dev)
    if mn_major:  # B = wout stored [V = K, d = N]
        dhn = g.gemm("d_final_norm_out", dlog, wout, S, d, V, b_major="mn", out_shape=(S, d), device=dev)
    else:
        woutT = tr("output.T", wout, V, d)
        dhn = g.gemm("d_final_norm_out", dlog, woutT, S, d, V, out_shape=(S, d), device=dev)
    dx = rms_bwd("d_x_final", xL, wn, dhn)

    def lora_grads(p, nm, dY, n_out, k_in, U, X, A, B):
        """dY [S, n_out] of Y = X Wᵀ + s U Bᵀ with U = X Aᵀ: returns V = dY·B and emits
        dB = s dYᵀU [n_out, R], dA = s VᵀX [R, k_in] as graph outputs."""
        if mn_major:  # B [n_out, R], dY [S, n_out], U [S, R], X [S, k_in], V [S, R] read in place
            Vv = g.gemm(p + nm + ".V", dY, B, S, R, n_out, b_major="mn", out_shape=(S, R), device=dev)
            results[p + nm + ".dB"] = g.gemm(p + nm + ".dB", dY, U, n_out, R, S, a_major="mn", b_major="mn",
                                             alpha=sc, out_shape=(n_out, R), device=dev)
            dAT = g.gemm(p + nm + ".dA.T", X, Vv, k_in, R, S, a_major="mn", b_major="mn", alpha=sc,
                         out_shape=(k_in, R), device=dev)
            results[p + nm + ".dA"] = tr(p + nm + ".dA", dAT, k_in, R)
            return Vv
        BT = tr(p + nm + ".B.T", B, n_out, R)
        Vv = g.gemm(p + nm + ".V", dY, BT, S, R, n_out, out_shape=(S, R), device=dev)
        dYT = tr(p + nm + ".dY.T", dY, S, n_out)
        UT = tr(p + nm + ".U.T", U, S, R)
        results[p + nm + ".dB"] = g.gemm(p + nm + ".dB", dYT, UT, n_out, R, S, alpha=sc, out_shape=(n_out, R),
                                         device=dev)
        VT = tr(p + nm + ".V.T", Vv, S, R)
        XT = tr(p + nm + ".X.T", X, S, k_in)
        # dAᵀ = s·Xᵀ·V keeps M = k_in on the tensor cores (R rows would be a GEMV)
        dAT = g.gemm(p + nm + ".dA.T", XT, VT, k_in, R, S, alpha=sc, out_shape=(k_in, R), device=dev)
        results[p + nm + ".dA"] = tr(p + nm + ".dA", dAT, k_in, R)
        return Vv

    def recompute(l):
        """Layer l's forward activations again from the saved residual stream /
        adapter activations (bitwise the forward's); depends on no gradient."""
        p, w, a = saved[l]
        if recompute_norms:  # h, h2 again from the saved x, x1 (bitwise the forward's): only the
            # residual stream is kept across the step
            a = dict(a, h2=rms(p + "ffn_norm_out.re", a["x1"], w["wn2"]), h=rms(p + "attn_norm_out.re", a["x"],
                                                                                   w["wn1"]))
        if recompute_ffn:  # gu and act again from the saved h2, U2 (bitwise the forward's)
            gub_r = g.gemm(p + "gate_up_base.re", a["h2"], w["w13"], S, 2 * f, d, out_shape=(S, 2 * f), device=dev)
            gu_r = g.gemm(p + "gate_up.re", a["U2"], w["B2"], S, 2 * f, R, r=gub_r, alpha=sc, out_shape=(S, 2 * f),
                          device=dev)
            a = dict(a, gu=gu_r, act=g.kernel(p + "act.re", {"type": "silu_mul", "args": [gu_r], "rows": S, "cols": f},
                                              (S, f), "bf16", dev))
        if recompute_qkv:  # qkv, q, k again from the saved h, U1
            base_r = g.gemm(p + "qkv_base.re", a["h"], w["wqkv"], S, 3 * d, d, out_shape=(S, 3 * d), device=dev)
            qkv_r = g.gemm(p + "qkv.re", a["U1"], w["B1"], S, 3 * d, R, r=base_r, alpha=sc, out_shape=(S, 3 * d),
                           device=dev)
            a = dict(a, qkv=qkv_r,
                     q=g.kernel(p + "q_rope.re", {"type": "rope", "args": [qkv_r, rope_tab], "seq": S, "ld": 3 * d,
                                                  "col_off": 0, "heads": H, "hd": hd}, (H, S, hd), "bf16", dev),
                     k=g.kernel(p + "k_rope.re", {"type": "rope", "args": [qkv_r, rope_tab], "seq": S, "ld": 3 * d,
                                                  "col_off": d, "heads": H, "hd": hd}, (H, S, hd), "bf16", dev))
        return a

    def attention_grads(p, a, do):
        """dq, dk, dv of the materialised attention (scores / probs / softmax_bwd)."""
        dP = g.gemm(p + "d_probs", do, a["qkv"], S, S, hd, batch=H, lda=d, sa=hd, ldb=3 * d, b_off=2 * d, sb=hd,
                    sc=S * S, out_dtype="f32", causal=1, out_shape=(H, S, S), device=dev)
        if recompute_attention:  # P again from the saved q, k (bitwise the forward's)
            scr_b = g.gemm(p + "scores.re", a["q"], a["k"], S, S, hd, batch=H, sa=S * hd, sb=S * hd, sc=S * S,
                           out_dtype="f32", causal=1, out_shape=(H, S, S), device=dev)
            P = g.kernel(p + "probs.re", {"type": "softmax", "args": [scr_b], "batch": H, "rows": S, "cols": S,
                                          "scale": scale, "causal": 1}, (H, S, S), "bf16", dev)
        else:
            P = a["P"]
        dS = g.kernel(p + "d_scores", {"type": "softmax_bwd", "args": [P, dP], "batch": H, "rows": S, "cols": S,
                                       "causal": 1, "in_dtype": "f32"}, (H, S, S), "bf16", dev)
        if mn_major:  # k, q [H, S, hd], dS / P [H, queries, keys], do [S, d] read in place
            dq_r = g.gemm(p + "d_q_rot", dS, a["k"], S, hd, S, batch=H, lda=S, ldb=hd, ldc=d, sa=S * S, sb=hd * S,
                          sc=hd, alpha=scale, causal=2, b_major="mn", out_shape=(S, d), device=dev)
            dk_r = g.gemm(p + "d_k_rot", dS, a["q"], S, hd, S, batch=H, lda=S, ldb=hd, ldc=d, sa=S * S, sb=hd * S,
                          sc=hd, alpha=scale, a_major="mn", b_major="mn", out_shape=(S, d), device=dev)
            dv = g.gemm(p + "d_v", P, do, S, hd, S, batch=H, lda=S, ldb=d, ldc=d, sa=S * S, sb=hd, sc=hd,
                        a_major="mn", b_major="mn", out_shape=(S, d), device=dev)
        else:
            kT = tr(p + "k.T", a["k"], S, hd, batch=H)
            dq_r = g.gemm(p + "d_q_rot", dS, kT, S, hd, S, batch=H, lda=S, ldb=S, ldc=d, sa=S * S, sb=hd * S, sc=hd,
                          alpha=scale, causal=2, out_shape=(S, d), device=dev)
            dST = tr(p + "d_scores.T", dS, S, S, batch=H)
            qT = tr(p + "q.T", a["q"], S, hd, batch=H)
            dk_r = g.gemm(p + "d_k_rot", dST, qT, S, hd, S, batch=H, lda=S, ldb=S, ldc=d, sa=S * S, sb=hd * S,
                          sc=hd, alpha=scale, out_shape=(S, d), device=dev)
            PT = tr(p + "probs.T", P, S, S, batch=H)
            doT = g.kernel(p + "d_attn.T", {"type": "transpose_heads", "args": [do], "seq": S, "ld": d, "col_off": 0,
                                            "heads": H, "hd": hd}, (H, hd, S), "bf16", dev)
            dv = g.gemm(p + "d_v", PT, doT, S, hd, S, batch=H, lda=S, ldb=S, ldc=d, sa=S * S, sb=hd * S, sc=hd,
                        out_shape=(S, d), device=dev)
        dq = g.kernel(p + "d_q", {"type": "rope", "args": [dq_r, rope_tab], "seq": S, "ld": d, "col_off": 0,
                                  "heads": H, "hd": hd, "inverse": 1, "tokens_out": 1}, (S, d), "bf16", dev)
        dk = g.kernel(p + "d_k", {"type": "rope", "args": [dk_r, rope_tab], "seq": S, "ld": d, "col_off": 0,
                                  "heads": H, "hd": hd, "inverse": 1, "tokens_out": 1}, (S, d), "bf16", dev)
        return dq, dk, ((dq, None, None), (dk, None, None), (dv, None, None))

    rec = {}
    for l in reversed(range(L)):
        # the recompute of layers l-1 .. l-bwd_prefetch is listed ahead of layer l's
        # gradient GEMMs, so the planner reloads their frozen weights one or more
        # layers early and the H2D of layer l-1 overlaps layer l's backward
        for j2 in range(l, max(-1, l - 1 - bwd_prefetch), -1):
            if j2 not in rec:
                rec[j2] = recompute(j2)
        p, w, _ = saved[l]
        a = rec.pop(l)
        dy = dx  # gradient of x_{l+1}
        # x_{l+1} = act·W2ᵀ + s·U3·B3ᵀ + x1
        V3 = lora_grads(p, "lora_w2", dy, d, f, a["U3"], a["act"], w["A3"], w["B3"])
        if mn_major:  # W2 [d, f], A3 [R, f] read MN-major
            da0 = g.gemm(p + "d_act_base", dy, w["w2"], S, f, d, b_major="mn", out_shape=(S, f), device=dev)
            da = g.gemm(p + "d_act", V3, w["A3"], S, f, R, r=da0, alpha=sc, b_major="mn", out_shape=(S, f),
                        device=dev)
        else:
            w2T = tr(p + "w2.T", w["w2"], d, f)
            A3T = tr(p + "lora_w2.A.T", w["A3"], R, f)
            da0 = g.gemm(p + "d_act_base", dy, w2T, S, f, d, out_shape=(S, f), device=dev)
            da = g.gemm(p + "d_act", V3, A3T, S, f, R, r=da0, alpha=sc, out_shape=(S, f), device=dev)
        dgu = g.kernel(p + "d_gate_up", {"type": "swiglu_bwd", "args": [a["gu"], da], "rows": S, "cols": f},
                       (S, 2 * f), "bf16", dev)
        V2 = lora_grads(p, "lora_w13", dgu, 2 * f, d, a["U2"], a["h2"], w["A2"], w["B2"])
        if mn_major:
            dh2_0 = g.gemm(p + "d_ffn_norm_out_base", dgu, w["w13"], S, d, 2 * f, b_major="mn", out_shape=(S, d),
                           device=dev)
            dh2 = g.gemm(p + "d_ffn_norm_out", V2, w["A2"], S, d, R, r=dh2_0, alpha=sc, b_major="mn",
                         out_shape=(S, d), device=dev)
        else:
            w13T = tr(p + "w13.T", w["w13"], 2 * f, d)
            A2T = tr(p + "lora_w13.A.T", w["A2"], R, d)
            dh2_0 = g.gemm(p + "d_ffn_norm_out_base", dgu, w13T, S, d, 2 * f, out_shape=(S, d), device=dev)
            dh2 = g.gemm(p + "d_ffn_norm_out", V2, A2T, S, d, R, r=dh2_0, alpha=sc, out_shape=(S, d), device=dev)
        dx1 = add(p + "d_x1", dy, rms_bwd(p + "d_x1_norm", a["x1"], w["wn2"], dh2))
        # x1 = o·Woᵀ + x ; o[:, head h] = P_h·V_h
        if mn_major:
            do = g.gemm(p + "d_attn", dx1, w["wo"], S, d, d, b_major="mn", out_shape=(S, d), device=dev)
        else:
            woT = tr(p + "wo.T", w["wo"], d, d)
            do = g.gemm(p + "d_attn", dx1, woT, S, d, d, out_shape=(S, d), device=dev)
        if fused_attention:
            # O and the row logsumexp again (fused forward), then dq|dk|dv in one fused kernel
            vt_r = g.kernel(p + "v_t.re", {"type": "transpose_heads", "args": [a["qkv"]], "seq": S, "ld": 3 * d,
                                           "col_off": 2 * d, "heads": H, "hd": hd}, (H, hd, S), "bf16", dev)
            o_lse = g.kernel(p + "attn.re", {"type": "attention", "args": [a["q"], a["k"], vt_r], "heads": H,
                                             "seq": S, "hd": hd, "ldo": d, "scale": scale, "causal": 1, "lse": 1},
                             (S * d + 2 * H * S,), "bf16", dev, cost=attn_flops / _PEAK_FLOPS)
            g.flops += attn_flops
            # dqkv = [dq | dk | dv] rows of 3d, dq and dk already rotated back (pre-RoPE)
            dqkv = g.kernel(p + "d_attn_qkv", {"type": "attention_bwd",
                                                "args": [a["q"], a["k"], a["qkv"], o_lse, do, rope_tab],
                                                "heads": H, "seq": S, "hd": hd, "scale": scale, "causal": 1,
                                                "v_off": 2 * d, "v_ld": 3 * d, "ldo": d, "do_ld": d},
                            (S * 3 * d + 2 * H * S,), "bf16", dev, cost=2.5 * attn_flops / _PEAK_FLOPS)
            g.flops += 2.5 * attn_flops
            parts = None
        else:
            dq, dk, parts = attention_grads(p, a, do)
        # qkv = h·Wqkvᵀ + s·U1·B1ᵀ with dqkv = [dq | dk | dv]
        V1 = None
        dBs = []
        if parts is None:  # one [S, 3d] gradient: each product over all of q|k|v at once
            V1 = g.gemm(p + "lora_qkv.V", dqkv, w["B1"], S, R, 3 * d, ldb=R, b_major="mn", out_shape=(S, R),
                        device=dev)
            results[p + "lora_qkv.dB"] = g.gemm(p + "lora_qkv.dB", dqkv, a["U1"], 3 * d, R, S, alpha=sc,
                                                a_major="mn", lda=3 * d, b_major="mn", out_shape=(3 * d, R),
                                                device=dev)
            dA1T = g.gemm(p + "lora_qkv.dA.T", a["h"], V1, d, R, S, alpha=sc, a_major="mn", b_major="mn",
                          out_shape=(d, R), device=dev)
        elif mn_major:  # B1 [3d, R] (part j: rows j*d..), U1 [S, R], dq/dk/dv [S, d], h [S, d], V1 [S, R]
            for j, (dpart, off, ld) in enumerate(parts):
                V1 = g.gemm(p + f"lora_qkv.V{j}", dpart, w["B1"], S, R, d, ldb=R, b_off=j * d * R, r=V1,
                            b_major="mn", a_off=off, lda=ld, out_shape=(S, R), device=dev)
                dBs.append(g.gemm(p + f"lora_qkv.dB{j}", dpart, a["U1"], d, R, S, alpha=sc, a_major="mn",
                                  b_major="mn", a_off=off, lda=ld, out_shape=(d, R), device=dev))
            results[p + "lora_qkv.dB"] = g.kernel(p + "lora_qkv.dB", {"type": "concat", "args": dBs, "count": d * R,
                                                                      "out_dtype": "bf16"}, (3 * d, R), "bf16", dev)
            dA1T = g.gemm(p + "lora_qkv.dA.T", a["h"], V1, d, R, S, alpha=sc, a_major="mn", b_major="mn",
                          out_shape=(d, R), device=dev)
        else:
            B1T = tr(p + "lora_qkv.B.T", w["B1"], 3 * d, R)
            U1T = tr(p + "lora_qkv.U.T", a["U1"], S, R)
            for j, (dpart, _, _) in enumerate(parts):
                V1 = g.gemm(p + f"lora_qkv.V{j}", dpart, B1T, S, R, d, ldb=3 * d, b_off=j * d, r=V1,
                            out_shape=(S, R), device=dev)
                dT = tr(p + f"lora_qkv.dY{j}.T", dpart, S, d)
                dBs.append(g.gemm(p + f"lora_qkv.dB{j}", dT, U1T, d, R, S, alpha=sc, out_shape=(d, R), device=dev))
            results[p + "lora_qkv.dB"] = g.kernel(p + "lora_qkv.dB", {"type": "concat", "args": dBs, "count": d * R,
                                                                      "out_dtype": "bf16"}, (3 * d, R), "bf16", dev)
            V1T = tr(p + "lora_qkv.V.T", V1, S, R)
            hT = tr(p + "lora_qkv.X.T", a["h"], S, d)
            dA1T = g.gemm(p + "lora_qkv.dA.T", hT, V1T, d, R, S, alpha=sc, out_shape=(d, R), device=dev)
        results[p + "lora_qkv.dA"] = tr(p + "lora_qkv.dA", dA1T, d, R)
        if l == 0:
            break  # no gradient is needed below the first layer
        dh = None
        if parts is None:
            dh = g.gemm(p + "d_attn_norm_out_base", dqkv, w["wqkv"], S, d, 3 * d, ldb=d, b_major="mn",
                        out_shape=(S, d), device=dev)
            dh = g.gemm(p + "d_attn_norm_out", V1, w["A1"], S, d, R, r=dh, alpha=sc, b_major="mn",
                        out_shape=(S, d), device=dev)
        elif mn_major:  # Wqkv [3d, d] (part j: rows j*d..), A1 [R, d]
            for j, (dpart, off, ld) in enumerate(parts):
                dh = g.gemm(p + f"d_attn_norm_out{j}", dpart, w["wqkv"], S, d, d, ldb=d, b_off=j * d * d, r=dh,
                            b_major="mn", a_off=off, lda=ld, out_shape=(S, d), device=dev)
            dh = g.gemm(p + "d_attn_norm_out", V1, w["A1"], S, d, R, r=dh, alpha=sc, b_major="mn",
                        out_shape=(S, d), device=dev)
        else:
            wqkvT = tr(p + "wqkv.T", w["wqkv"], 3 * d, d)
            A1T = tr(p + "lora_qkv.A.T", w["A1"], R, d)
            for j, (dpart, _, _) in enumerate(parts):
                dh = g.gemm(p + f"d_attn_norm_out{j}", dpart, wqkvT, S, d, d, ldb=3 * d, b_off=j * d, r=dh,
                            out_shape=(S, d), device=dev)
            dh = g.gemm(p + "d_attn_norm_out", V1, A1T, S, d, R, r=dh, alpha=sc, out_shape=(S, d), device=dev)
        dx = add(p + "d_x", dx1, rms_bwd(p + "d_x_norm", a["x"], w["wn1"], dh))
    return results


def prefill_flops(cfg: LlamaConfig, seq: int, layers: int | None = None) -> float:
    """Algorithmic FLOPs of llama_prefill (causal attention counted as half)."""
    L = cfg.layers if layers is None else layers
    d, f, S, hd, H = cfg.dim, cfg.ffn, seq, cfg.hd, cfg.heads
    lin = 2.0 * S * (3 * d * d + d * d + 2 * f * d + f * d)
    attn = 2 * (2.0 * S * S * hd * H) * 0.5 * (1 + 1 / S)
    return L * (lin + attn) + 2.0 * cfg.vocab * d


# ------------------------------------------ long-context blockwise attention (cfg 5) ---
def blockwise_attention(seq: int = 65536, heads: int = 32, hd: int = 128, tile: int = 4096,
                        device: int = 0, lag: int | None = None, interleave: str = "head",
                        pv_ksplit: int = 0) -> GraphBuilder:
    """Config 5: causal attention over `seq` tokens with the n^2 score tiles
    materialised as vertices and kept live across a two-pass softmax, so a
    capped plan must offload them to host RAM.

    Pass 1, for every head h and query block i, key block j <= i:
        S_hij = scale * Q_hi K_hjᵀ (bf16 tile)      st_hij = rowstats(S_hij)
    then m/l per (h, i) = stats_combine(st_hi0..st_hii) in fixed j order.
    Pass 2 (after ALL of pass 1, as listed):
        P_hij = softmax_apply(S_hij, ml_hi); O_hi = P_hi0 V_h0 + ... (a chain of
        gemms with fused fp32 residual, j ascending); out_hi = bf16(O_hi).
    Q/K/Vᵀ blocks are graph inputs (cold in host RAM).

    `lag` (default: all heads) is the listing distance between a head's pass 1
    and its pass 2: pass 2 of head h is listed right after pass 1 of head
    h + lag, so `lag` heads of score tiles are live at once — enough to force
    offloads under a cap while letting the D2H of new tiles overlap the H2D of
    old ones (duplex PCIe). `interleave="block"` lists the two passes query
    block by query block (pass 1 of (h + lag, i), then pass 2 of (h, i)), so
    the tiles being produced (offloaded) and the tiles being consumed
    (reloaded) alternate at tile granularity instead of head granularity.
    `pv_ksplit` > 1 asks the executor to split the K (= tile keys) of each
    P·V GEMM into that many ranges (M = tile, N = hd fills only tile/128
    CTAs); the partials are reduced in split order."""
    assert seq % tile == 0
    nb = seq // tile
    T = tile
    g = GraphBuilder(device_count=1)
    dev = device
    scale = 1.0 / math.sqrt(hd)
    q = {(h, i): g.input(f"q[{h},{i}]", (T, hd), "bf16", dev, init=("normal", 1.0)) for h in range(heads) for i in range(nb)}
    k = {(h, j): g.input(f"k[{h},{j}]", (T, hd), "bf16", dev, init=("normal", 1.0)) for h in range(heads) for j in range(nb)}
    vt = {(h, j): g.input(f"vt[{h},{j}]", (hd, T), "bf16", dev, init=("normal", 1.0)) for h in range(heads) for j in range(nb)}
    S, ml = {}, {}
    lag = heads if lag is None else max(0, min(lag, heads))

    def pass1(h, blocks=None):
        for i in (range(nb) if blocks is None else blocks):
            parts = []
            for j in range(i + 1):
                S[(h, i, j)] = g.gemm(f"S[{h},{i},{j}]", q[(h, i)], k[(h, j)], T, T, hd, alpha=scale,
                                      out_shape=(T, T), device=dev)
                parts.append(g.kernel(f"st[{h},{i},{j}]", {"type": "rowstats", "args": [S[(h, i, j)]], "rows": T,
                                                            "cols": T, "causal": int(i == j)}, (T, 2), "f32", dev))
            ml[(h, i)] = g.kernel(f"ml[{h},{i}]", {"type": "stats_combine", "args": parts, "rows": T}, (T, 2), "f32", dev)

    def pass2(h, blocks=None):
        for i in (range(nb) if blocks is None else blocks):
            acc = None
            for j in range(i + 1):
                P = g.kernel(f"P[{h},{i},{j}]", {"type": "softmax_apply", "args": [S[(h, i, j)], ml[(h, i)]], "rows": T,
                                                 "cols": T, "causal": int(i == j)}, (T, T), "bf16", dev)
                acc = g.gemm(f"O[{h},{i},{j}]", P, vt[(h, j)], T, hd, T, r=acc, out_dtype="f32", out_shape=(T, hd),
                             device=dev, ksplit=pv_ksplit or None)
            g.kernel(f"out[{h},{i}]", {"type": "cast", "args": [acc], "count": T * hd, "in_dtype": "f32",
                                       "out_dtype": "bf16"}, (T, hd), "bf16", dev)

    assert interleave in ("head", "block")
    for step in range(heads + lag):
        if interleave == "block" and step < heads and step - lag >= 0:
            for i in range(nb):
                pass1(step, [i])
                pass2(step - lag, [i])
            continue
        if step < heads:
            pass1(step)
        if step - lag >= 0:
            pass2(step - lag)
    return g


def blockwise_attention_flops(seq, heads, hd, tile):
    nb = seq // tile
    return heads * (nb * (nb + 1) // 2) * 2 * (2.0 * tile * tile * hd)


# ------------------------------------------------- tiled matmul chain (cfg 1) ---
def matmul_chain(n: int = 4096, tile: int = 1024, chain: int = 4, devices: int = 2,
                 dtype: str = "f32", precision: str = "3xtf32") -> GraphBuilder:
    """Config 1: X·W1·W2·…·WL, n×n fp32, tiled `tile`×`tile`.

    Row panels of X are split over devices; each device holds its own copy of
    every weight tile (inputs), computes per-tile partial products (one gemm
    vertex per (i, j, k)) and a fixed-order combine (`sum` of the k partials,
    so the reduction order never depends on the schedule). Between links the
    activation row panels are exchanged with Transfer vertices (all-gather of
    panels), which exercises the move path across devices.
    Weights are stored transposed per tile (B operand is K-major). fp32 tiles
    multiply with `precision` "3xtf32" (fp32-accurate split on the tensor
    cores, the default) or "tf32" (one tf32 MMA, ~1e-3 relative)."""
    T = n // tile
    g = GraphBuilder(device_count=devices)
    rows_per_dev = [list(range(d * T // devices, (d + 1) * T // devices)) for d in range(devices)]
    owner = {i: d for d in range(devices) for i in rows_per_dev[d]}
    X = {(i, k): g.input(f"X[{i},{k}]", (tile, tile), dtype, owner[i], init=("uniform", -1 / 64, 1 / 64))
         for i in range(T) for k in range(T)}
    cur = X
    for l in range(chain):
        Wt = {}
        for d in range(devices):
            for j in range(T):
                for k in range(T):
                    Wt[(d, j, k)] = g.input(f"W{l}T[{j},{k}]@{d}", (tile, tile), dtype, d,
                                            init=("uniform", -1 / 64, 1 / 64))
        nxt = {}
        for i in range(T):
            d = owner[i]
            for j in range(T):
                parts = []
                for k in range(T):
                    parts.append(g.gemm(f"P{l}[{i},{j},{k}]", cur[(i, k)], Wt[(d, j, k)], tile, tile, tile,
                                        in_dtype=dtype, out_dtype="f32", out_shape=(tile, tile), device=d,
                                        precision=precision if dtype == "f32" else None))
                nxt[(i, j)] = g.kernel(f"Y{l}[{i},{j}]", {"type": "sum", "args": parts, "count": tile * tile,
                                                          "in_dtype": "f32", "out_dtype": dtype},
                                       (tile, tile), dtype, d)
        if l + 1 < chain and devices > 1:
            # Row panels stay with their owner; nothing moves for X·W. To
            # exercise NVLink moves, rotate panel ownership each link.
            moved = {}
            new_owner = {i: (owner[i] + 1) % devices for i in range(T)}
            for (i, j), vid in nxt.items():
                moved[(i, j)] = g.transfer(vid, new_owner[i])
            owner = new_owner
            nxt = moved
        cur = nxt
    return g


# ------------------------------------------------------------- memgraph ---
def plan(g: GraphBuilder, capacity, *, alloc_horizon="greedy", victim_policy="farthest-next-use",
         order_policy="as-listed", seed=0, keep_superfluous=True):
    """Builds the memgraph with this package's bit-exact planner."""
    from . import memplan

    caps = capacity if isinstance(capacity, (list, tuple)) else [int(capacity)] * g.device_count
    return memplan.build_memgraph(g.to_json(), list(caps), mode="byte", order_policy=order_policy,
                                  victim_policy=victim_policy, seed=seed, alloc_horizon=alloc_horizon,
                                  keep_superfluous=keep_superfluous)


def working_set_floor(g: GraphBuilder) -> list[int]:
    """Per-device lower bound for a plan: permanent outputs plus the largest
    single working set (a vertex's output + same-device inputs), like
    tests/test_helpers.hpp:55-74 in byte mode (without its 1.5x slack)."""
    cons = {}
    prods = {v["id"]: [] for v in g.vertices}
    for p, c in g.edges:
        cons[p] = cons.get(p, 0) + 1
        prods[c].append(p)
    size = {v["id"]: v["output_size"] for v in g.vertices}
    dev = {v["id"]: v["device"] for v in g.vertices}
    outs = [0] * g.device_count
    ws = [0] * g.device_count
    for v in g.vertices:
        if cons.get(v["id"], 0) == 0:
            outs[v["device"]] += v["output_size"]
        w = v["output_size"] + sum(size[p] for p in prods[v["id"]] if dev[p] == v["device"])
        ws[v["device"]] = max(ws[v["device"]], w)
    return [o + w for o, w in zip(outs, ws)]
