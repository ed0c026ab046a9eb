"""CPU restatement of the op payload semantics in fp32 (numpy).

TEST INFRASTRUCTURE ONLY — the checker, never the product: only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import this.

Parity status: the reference has no tensor math at all (vertices are opaque
tasks; "real GPU execution, CUDA/cuTensor
kernels" out of scope), so tensor values are "parity unpinned":
these functions DEFINE the op semantics of our payload schema
(paper_2405_16283_b200/csrc/exec/ops.hpp) and the GPU kernels are checked
against them within stated tolerances. Every op reduces in fp32 and rounds
once to the output dtype (bf16 round-to-nearest-even), like the kernels.
"""
from __future__ import annotations

import numpy as np

DT = {"bf16": 2, "f32": 4, "i32": 4}


# ---------------------------------------------------------------- bf16 ---
def bf16_to_f32(u16: np.ndarray) -> np.ndarray:
    return (u16.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + r) >> 16).astype(np.uint16)


def load(buf: np.ndarray, dtype: str, count: int, off_elems: int = 0) -> np.ndarray:
    """Reads `count` elements of `dtype` from a uint8 buffer as fp32 (or int32)."""
    es = DT[dtype]
    raw = buf[off_elems * es:(off_elems + count) * es]
    if dtype == "bf16":
        return bf16_to_f32(raw.view(np.uint16))
    if dtype == "f32":
        return raw.view(np.float32).astype(np.float32)
    return raw.view(np.int32)


def store(buf: np.ndarray, dtype: str, values: np.ndarray, off_elems: int = 0) -> None:
    es = DT[dtype]
    v = np.ascontiguousarray(values).reshape(-1)
    if dtype == "bf16":
        b = f32_to_bf16(v.astype(np.float32)).view(np.uint8)
    elif dtype == "f32":
        b = v.astype(np.float32).view(np.uint8)
    else:
        b = v.astype(np.int32).view(np.uint8)
    buf[off_elems * es:off_elems * es + b.size] = b


def typed(buf: np.ndarray, dtype: str) -> np.ndarray:
    es = DT[dtype]
    raw = buf[: (buf.size // es) * es]
    return raw.view({"bf16": np.uint16, "f32": np.float32, "i32": np.int32}[dtype])


def strided(buf, dtype, off, batch, bs, rows, ld, cols):
    """[batch, rows, cols] fp32 copy of an element-strided region."""
    t = typed(buf, dtype)
    span = off + (batch - 1) * bs + (rows - 1) * ld + cols
    if span > t.size:
        raise ValueError(f"strided view needs {span} elements, region has {t.size}")
    es = t.itemsize
    v = np.lib.stride_tricks.as_strided(t[off:], shape=(batch, rows, cols), strides=(bs * es, ld * es, es))
    return bf16_to_f32(v) if dtype == "bf16" else v.astype(np.float32)


def scatter(buf, dtype, off, bs, ld, values, mask=None):
    """Writes values[batch, rows, cols] into an element-strided region."""
    t = typed(buf, dtype)
    Bn, R, Cc = values.shape
    es = t.itemsize
    v = np.lib.stride_tricks.as_strided(t[off:], shape=(Bn, R, Cc), strides=(bs * es, ld * es, es),
                                        writeable=True)
    conv = f32_to_bf16(values) if dtype == "bf16" else values.astype(t.dtype)
    if mask is None:
        v[...] = conv
    else:
        np.copyto(v, conv, where=mask)


# ------------------------------------------------------------------ ops ---
def op_gemm(op, args, out):
    """C[b] = alpha * A[b] @ B[b]^T (+ R[b]).

    causal 1: only C[b][i][j<=i] is defined (the upper triangle is left
    untouched; a causal softmax never reads it). causal 2: A is lower
    triangular (A[b][i][k>i] == 0, e.g. causal softmax probabilities), which
    lets the kernel skip the all-zero K blocks; the product is the plain one."""
    M, N, K, B = op["M"], op["N"], op["K"], op.get("batch", 1)
    a_mn, b_mn = op.get("a_major", "k") == "mn", op.get("b_major", "k") == "mn"
    # MN-major operands: A stored [K, M], B stored [K, N] (row pitch lda / ldb)
    lda = op.get("lda") or (M if a_mn else K)
    ldb = op.get("ldb") or (N if b_mn else K)
    ldc = op.get("ldc") or N
    ind, outd = op.get("in_dtype", "bf16"), op.get("out_dtype", "bf16")
    if a_mn:
        A = np.transpose(strided(args[0], ind, op.get("a_off", 0), B, op.get("sa", 0), K, lda, M), (0, 2, 1))
    else:
        A = strided(args[0], ind, op.get("a_off", 0), B, op.get("sa", 0), M, lda, K)
    if b_mn:
        Bm = np.transpose(strided(args[1], ind, op.get("b_off", 0), B, op.get("sb", 0), K, ldb, N), (0, 2, 1))
    else:
        Bm = strided(args[1], ind, op.get("b_off", 0), B, op.get("sb", 0), N, ldb, K)
    causal = op.get("causal", 0)
    C = np.matmul(A, np.transpose(Bm, (0, 2, 1))) * np.float32(op.get("alpha", 1.0))
    if op.get("rs_arg", -1) >= 0:  # fused RMSNorm consumer: row m *= rsqrt(sum_c P[c][row0+m] / dim + eps)
        C = C * row_scale(op, args)[None, :, None]
    if op.get("epilogue", "none") == "qkv_rope":
        # packed [rope(q) (H,M,128) | rope(k) | vT (H,128,M)] from C = x W^T
        H, Mm = op["heads"], op["M"]
        tab = load(args[2], "f32", Mm * 64 * 2).reshape(Mm, 64, 2)
        c, s_ = tab[:, None, :, 0], tab[:, None, :, 1]
        X = C[0].reshape(Mm, 3, H, 128)

        def rope(x):  # x [M, H, 128]
            a, b = x[..., :64], x[..., 64:]
            return np.concatenate([a * c - b * s_, b * c + a * s_], axis=-1).transpose(1, 0, 2)

        packed = np.concatenate([rope(X[:, 0]).reshape(-1), rope(X[:, 1]).reshape(-1),
                                 X[:, 2].transpose(1, 2, 0).reshape(-1)])
        store(out, "bf16", packed)
        return
    if op.get("epilogue", "none") == "swiglu":
        # out[:, 128b + j] = silu(C[:, 256b + j]) * C[:, 256b + 128 + j]
        Bn, Mm, Nn = C.shape
        blk = C.reshape(Bn, Mm, Nn // 256, 2, 128)
        g, u = blk[:, :, :, 0, :], blk[:, :, :, 1, :]
        C = (g / (1.0 + np.exp(-g)) * u).reshape(Bn, Mm, Nn // 2)
        ldc = op.get("ldc") or Nn // 2
    if len(args) >= 3:
        C = C + strided(args[2], outd, op.get("r_off", 0), B, op.get("sc", 0), M, ldc, N)
    if op.get("norm_out", 0):  # fused RMSNorm producer: [x | h = x*gamma | P]
        store_norm_out(out, C[0], load(args[3], "bf16", N))
        return
    mask = None
    if causal == 1:
        mask = np.broadcast_to((np.arange(N)[None, :] <= np.arange(M)[:, None])[None], C.shape)
    scatter(out, outd, op.get("c_off", 0), op.get("sc", 0), ldc, C.astype(np.float32), mask)


def chunk_sumsq(x: np.ndarray) -> np.ndarray:
    """P[m][c] = sum over the 32 columns of chunk c of x[m]^2, accumulated in
    column order in fp32 (the fused-norm producers' partial sums, [rows, cols/32])."""
    R, Cc = x.shape
    xc = x.reshape(R, Cc // 32, 32)
    ss = np.zeros((R, Cc // 32), dtype=np.float32)
    for j in range(32):
        ss += xc[:, :, j] * xc[:, :, j]
    return ss


def store_norm_out(out, C2d, g):
    """Writes the fused-RMSNorm producer output [x | h | P] for fp32 values
    C2d [rows, cols]: x = bf16(C2d), h = bf16(x * g), P = chunk_sumsq(x)."""
    R, Cc = C2d.shape
    x = bf16_to_f32(f32_to_bf16(C2d))
    store(out, "bf16", x)
    store(out, "bf16", x * g[None, :], R * Cc)
    store(out, "f32", chunk_sumsq(x), R * Cc)  # f32 element offset R*Cc == byte offset 2*R*Cc*2


def row_scale(op, args) -> np.ndarray:
    """Per-row factor of a fused-RMSNorm consumer: rsqrt(sum_c P[row0+m][c] /
    dim + eps), c summed in order (P [rows, ld] fp32 read from args[rs_arg]
    at byte rs_off)."""
    M, dim, ld, row0 = op["M"], op["rs_dim"], op["rs_ld"], op.get("rs_row0", 0)
    buf = args[op["rs_arg"]][op.get("rs_off", 0):]
    P = buf[: (row0 + M) * ld * 4].view(np.float32).reshape(row0 + M, ld)[row0:row0 + M, : dim // 32]
    ss = np.zeros(M, dtype=np.float32)
    for c in range(dim // 32):
        ss += P[:, c]
    return (np.float32(1.0) / np.sqrt(ss / np.float32(dim) + np.float32(op.get("eps", 1e-5)))).astype(np.float32)


def op_rmsnorm(op, args, out):
    R, Cc, eps = op["rows"], op["cols"], op.get("eps", 1e-5)
    x = load(args[0], "bf16", R * Cc).reshape(R, Cc)
    w = load(args[1], "bf16", Cc)
    ms = np.mean(x * x, axis=1, keepdims=True, dtype=np.float32)
    y = x * (1.0 / np.sqrt(ms + np.float32(eps))).astype(np.float32) * w[None, :]
    store(out, "bf16", y)


def _pool():
    import os
    from concurrent.futures import ThreadPoolExecutor

    global _POOL
    if _POOL is None:
        _POOL = ThreadPoolExecutor(max_workers=os.cpu_count() or 1)
    return _POOL


_POOL = None


def op_softmax(op, args, out):
    """Row softmax of scale*S over j <= i (causal) or all j; masked entries
    are exact zeros. Heads run on a thread pool (numpy ufuncs drop the GIL)."""
    B, R, Cc, scale, causal = op.get("batch", 1), op["rows"], op["cols"], op.get("scale", 1.0), op.get("causal", 0)
    S = typed(args[0], "f32")[: B * R * Cc].reshape(B, R, Cc)
    P = typed(out, "bf16")[: B * R * Cc].reshape(B, R, Cc)
    keep = (np.arange(Cc)[None, :] <= np.arange(R)[:, None]) if causal else None

    def one(b):
        x = S[b] * np.float32(scale)
        if keep is not None:
            np.copyto(x, np.float32(-np.inf), where=~keep)
        x -= x.max(axis=1, keepdims=True)
        np.exp(x, out=x)
        x /= x.sum(axis=1, keepdims=True, dtype=np.float32)
        P[b] = f32_to_bf16(x)

    list(_pool().map(one, range(B)))


def op_attention(op, args, out):
    """O[i, h*hd:(h+1)*hd] = softmax_j(scale * q_i . k_j, j <= i if causal) @ v,
    fp32 throughout (the fused GPU kernel rounds P to bf16 for its MMA)."""
    H, S, hd, scale, causal = op["heads"], op["seq"], op["hd"], op.get("scale", 1.0), op.get("causal", 1)
    ldo = op.get("ldo") or H * hd
    n = H * S * hd
    aq, ak, av = (args[0], args[1], args[2]) if len(args) == 3 else (args[0], args[0], args[0])
    q = load(aq, "bf16", n, op.get("q_off", 0)).reshape(H, S, hd)
    k = load(ak, "bf16", n, op.get("k_off", 0)).reshape(H, S, hd)
    vt = load(av, "bf16", n, op.get("v_off", 0)).reshape(H, hd, S)
    keep = (np.arange(S)[None, :] <= np.arange(S)[:, None]) if causal else None
    O = np.empty((S, H, hd), dtype=np.float32)
    lse = np.empty((H, S), dtype=np.float32)

    def one(h):
        s = (q[h] @ k[h].T) * np.float32(scale)
        if keep is not None:
            np.copyto(s, np.float32(-np.inf), where=~keep)
        mx = s.max(axis=1, keepdims=True)
        s -= mx
        np.exp(s, out=s)
        tot = s.sum(axis=1, keepdims=True, dtype=np.float32)
        lse[h] = (mx + np.log(tot))[:, 0]
        s /= tot
        O[:, h, :] = s @ vt[h].T

    list(_pool().map(one, range(H)))
    scatter(out, "bf16", 0, 0, ldo, O.reshape(1, S, H * hd))
    if op.get("lse", 0):  # natural-log logsumexp of each scaled score row, after the [S, ldo] output
        store(out, "f32", lse, S * ldo // 2)


def op_attention_bwd(op, args, out):
    """Attention gradient (attention_bwd.cu): P = exp(scale q k^T - lse) from the
    forward's lse, D = rowsum(dO * O), dS = P * (dP - D), dP = dO v^T;
    out = [dq | dk | dv] rows of 3*H*hd (dq = scale dS k, dk = scale dS^T q,
    dv = P^T dO), then D (f32 [H, S]). fp32 throughout (the kernel rounds P and
    dS to bf16 for its MMAs)."""
    H, S, hd, scale, causal = op["heads"], op["seq"], op["hd"], op.get("scale", 1.0), op.get("causal", 1)
    w = H * hd
    ldo, vld, dld = op.get("ldo") or w, op.get("v_ld") or w, op.get("do_ld") or w
    n = H * S * hd
    q = load(args[0], "bf16", n, op.get("q_off", 0)).reshape(H, S, hd)
    k = load(args[1], "bf16", n, op.get("k_off", 0)).reshape(H, S, hd)
    v = strided(args[2], "bf16", op.get("v_off", 0), 1, 0, S, vld, w)[0].reshape(S, H, hd)
    o = strided(args[3], "bf16", 0, 1, 0, S, ldo, w)[0].reshape(S, H, hd)
    lse = load(args[3], "f32", H * S, S * ldo // 2).reshape(H, S)
    do = strided(args[4], "bf16", 0, 1, 0, S, dld, w)[0].reshape(S, H, hd)
    keep = (np.arange(S)[None, :] <= np.arange(S)[:, None]) if causal else np.ones((S, S), bool)
    G = np.empty((S, 3, H, hd), dtype=np.float32)
    D = np.empty((H, S), dtype=np.float32)

    def one(h):
        s = (q[h] @ k[h].T) * np.float32(scale)
        P = np.where(keep, np.exp(s - lse[h][:, None]), np.float32(0.0)).astype(np.float32)
        dOh = do[:, h, :]
        D[h] = np.sum(dOh * o[:, h, :], axis=1, dtype=np.float32)
        dS = P * (dOh @ v[:, h, :].T - D[h][:, None])
        G[:, 0, h, :] = np.float32(scale) * (dS @ k[h])
        G[:, 1, h, :] = np.float32(scale) * (dS.T @ q[h])
        G[:, 2, h, :] = P.T @ dOh

    list(_pool().map(one, range(H)))
    if len(args) == 6:  # pre-RoPE dq, dk: rotate-half by -theta at each position (op_rope "inverse")
        tab = load(args[5], "f32", S * (hd // 2) * 2).reshape(S, hd // 2, 2)
        c, sn = tab[:, None, None, :, 0], tab[:, None, None, :, 1]
        a, b = G[:, :2, :, : hd // 2], G[:, :2, :, hd // 2:]
        G[:, :2] = np.concatenate([a * c + b * sn, b * c - a * sn], axis=-1)
    store(out, "bf16", G.reshape(-1))
    store(out, "f32", D, S * 3 * w // 2)


def _valid_mask(rows, cols, causal):
    return (np.arange(cols)[None, :] <= np.arange(rows)[:, None]) if causal else np.ones((rows, cols), bool)


def op_rowstats(op, args, out):
    """(m, l) per row of a bf16 score tile: m = max_j s_ij, l = sum_j exp(s_ij - m)
    over valid j (j <= i on a causal diagonal tile)."""
    R, Cc, causal = op["rows"], op["cols"], op.get("causal", 0)
    S = load(args[0], "bf16", R * Cc).reshape(R, Cc)
    keep = _valid_mask(R, Cc, causal)
    x = np.where(keep, S, -np.inf)
    m = x.max(axis=1)
    l = np.exp(x - m[:, None]).sum(axis=1, dtype=np.float32)
    store(out, "f32", np.stack([m, l], axis=1).astype(np.float32))


def op_stats_combine(op, args, out):
    """Folds per-tile (m, l) in argument order: m = max, l = sum l_k exp(m_k - m)."""
    R = op["rows"]
    acc = load(args[0], "f32", 2 * R).reshape(R, 2).copy()
    for a in args[1:]:
        x = load(a, "f32", 2 * R).reshape(R, 2)
        m = np.maximum(acc[:, 0], x[:, 0])
        acc[:, 1] = acc[:, 1] * np.exp(acc[:, 0] - m) + x[:, 1] * np.exp(x[:, 0] - m)
        acc[:, 0] = m
    store(out, "f32", acc)


def op_softmax_apply(op, args, out):
    """P = exp(S - m) / l (bf16), masked entries 0."""
    R, Cc, causal = op["rows"], op["cols"], op.get("causal", 0)
    S = load(args[0], "bf16", R * Cc).reshape(R, Cc)
    st = load(args[1], "f32", 2 * R).reshape(R, 2)
    P = np.exp(S - st[:, :1]) / st[:, 1:]
    store(out, "bf16", np.where(_valid_mask(R, Cc, causal), P, 0.0).astype(np.float32))


def op_rope(op, args, out):
    """Rotate-half RoPE; "inverse" rotates by -theta (the backward), "tokens_out"
    writes [seq, heads*hd] instead of head-major [heads, seq, hd]."""
    S, ld, co, H, hd = op["seq"], op["ld"], op.get("col_off", 0), op["heads"], op["hd"]
    half = hd // 2
    x = strided(args[0], "bf16", co, 1, 0, S, ld, H * hd)[0].reshape(S, H, hd)
    tab = load(args[1], "f32", S * half * 2).reshape(S, half, 2)
    sgn = np.float32(-1.0 if op.get("inverse", 0) else 1.0)
    c, s = tab[:, None, :, 0], sgn * tab[:, None, :, 1]
    a, b = x[..., :half], x[..., half:]
    y = np.concatenate([a * c - b * s, b * c + a * s], axis=-1)  # [S, H, hd]
    store(out, "bf16", y if op.get("tokens_out", 0) else np.transpose(y, (1, 0, 2)))


def op_transpose(op, args, out):
    Bn, R, Cc, dt = op.get("batch", 1), op["rows"], op["cols"], op.get("out_dtype", "bf16")
    t = typed(args[0], dt)[: Bn * R * Cc].reshape(Bn, R, Cc)
    o = typed(out, dt)
    o[: Bn * R * Cc] = np.transpose(t, (0, 2, 1)).reshape(-1)


def op_rmsnorm_bwd(op, args, out):
    """dx = r (w.dy) - x r^3 mean((w.dy).x), r = 1/sqrt(mean(x^2) + eps)."""
    R, Cc, eps = op["rows"], op["cols"], op.get("eps", 1e-5)
    x = load(args[0], "bf16", R * Cc).reshape(R, Cc)
    w = load(args[1], "bf16", Cc)
    dy = load(args[2], "bf16", R * Cc).reshape(R, Cc)
    r = (1.0 / np.sqrt(np.mean(x * x, axis=1, keepdims=True, dtype=np.float32) + np.float32(eps))).astype(np.float32)
    g = w[None, :] * dy
    k = r ** 3 * np.mean(g * x, axis=1, keepdims=True, dtype=np.float32)
    store(out, "bf16", r * g - x * k)


def op_swiglu_bwd(op, args, out):
    R, Cc = op["rows"], op["cols"]
    gu = load(args[0], "bf16", R * 2 * Cc).reshape(R, 2 * Cc)
    da = load(args[1], "bf16", R * Cc).reshape(R, Cc)
    g, u = gu[:, :Cc], gu[:, Cc:]
    sg = 1.0 / (1.0 + np.exp(-g))
    store(out, "bf16", np.concatenate([da * u * sg * (1.0 + g * (1.0 - sg)), da * g * sg], axis=1))


def op_softmax_bwd(op, args, out):
    Bn, R, Cc, causal = op.get("batch", 1), op["rows"], op["cols"], op.get("causal", 0)
    P = load(args[0], "bf16", Bn * R * Cc).reshape(Bn, R, Cc)
    dP = load(args[1], op.get("in_dtype", "f32"), Bn * R * Cc).reshape(Bn, R, Cc)
    keep = _valid_mask(R, Cc, causal)[None]
    P = np.where(keep, P, 0.0)
    dot = np.sum(P * np.where(keep, dP, 0.0), axis=2, keepdims=True, dtype=np.float32)
    store(out, "bf16", np.where(keep, P * (dP - dot), 0.0).astype(np.float32))


def _xent_parts(op, args):
    R, V = op["rows"], op["vocab"]
    lg = load(args[0], op.get("in_dtype", "bf16"), R * V).reshape(R, V)
    t = np.clip(load(args[1], "i32", R), 0, V - 1)
    mx = lg.max(axis=1, keepdims=True)
    e = np.exp(lg - mx)
    ssum = e.sum(axis=1, keepdims=True, dtype=np.float32)
    return lg, t, mx, e, ssum


def op_xent_grad(op, args, out):
    lg, t, mx, e, ssum = _xent_parts(op, args)
    g = e / ssum
    g[np.arange(len(t)), t] -= 1.0
    store(out, op.get("out_dtype", "bf16"), g * np.float32(op.get("scale", 1.0)))


def op_xent_loss(op, args, out):
    lg, t, mx, e, ssum = _xent_parts(op, args)
    rows = (mx[:, 0] + np.log(ssum[:, 0]) - lg[np.arange(len(t)), t]) * np.float32(op.get("scale", 1.0))
    store(out, "f32", np.array([np.sum(rows, dtype=np.float32)], dtype=np.float32))


def op_transpose_heads(op, args, out):
    S, ld, co, H, hd = op["seq"], op["ld"], op.get("col_off", 0), op["heads"], op["hd"]
    x = strided(args[0], "bf16", co, 1, 0, S, ld, H * hd)[0].reshape(S, H, hd)
    store(out, "bf16", np.transpose(x, (1, 2, 0)))


def op_silu_mul(op, args, out):
    R, Cc = op["rows"], op["cols"]
    gu = load(args[0], "bf16", R * 2 * Cc).reshape(R, 2 * Cc)
    g, u = gu[:, :Cc], gu[:, Cc:]
    store(out, "bf16", g / (1.0 + np.exp(-g)) * u)


def op_sum(op, args, out):
    """out = sum_i in_i[offs_i : offs_i + count], fp32, argument order."""
    n, ind, outd = op["count"], op.get("in_dtype", "bf16"), op.get("out_dtype", "bf16")
    offs = op.get("offs") or [0] * len(args)
    acc = load(args[0], ind, n, offs[0]).astype(np.float32).copy()
    for a, o in zip(args[1:], offs[1:]):
        acc += load(a, ind, n, o)
    store(out, outd, acc)


def op_concat(op, args, out):
    """out = args[0] ++ args[1] ++ ... (count elements of out_dtype each)."""
    nb = op["count"] * DT[op.get("out_dtype", "bf16")]
    for i, a in enumerate(args):
        out[i * nb:(i + 1) * nb] = a[:nb]


def op_embedding(op, args, out):
    S, Dm, V = op["seq"], op["dim"], op["vocab"]
    tok = np.clip(load(args[0], "i32", S), 0, V - 1)
    tab = args[1][: V * Dm * 2].view(np.uint16).reshape(V, Dm)
    if op.get("norm_out", 0):  # fused RMSNorm producer: [x | h = x*gamma | P]
        store_norm_out(out, bf16_to_f32(tab[tok]), load(args[2], "bf16", Dm))
        return
    out[: S * Dm * 2] = tab[tok].reshape(-1).view(np.uint8)


def op_cast(op, args, out):
    n = op["count"]
    store(out, op.get("out_dtype", "bf16"), load(args[0], op.get("in_dtype", "f32"), n))


OPS = {
    "gemm": op_gemm,
    "rmsnorm": op_rmsnorm,
    "softmax": op_softmax,
    "rope": op_rope,
    "transpose_heads": op_transpose_heads,
    "silu_mul": op_silu_mul,
    "sum": op_sum,
    "embedding": op_embedding,
    "cast": op_cast,
    "attention": op_attention,
    "attention_bwd": op_attention_bwd,
    "rowstats": op_rowstats,
    "stats_combine": op_stats_combine,
    "softmax_apply": op_softmax_apply,
    "concat": op_concat,
    "transpose": op_transpose,
    "rmsnorm_bwd": op_rmsnorm_bwd,
    "swiglu_bwd": op_swiglu_bwd,
    "softmax_bwd": op_softmax_bwd,
    "xent_grad": op_xent_grad,
    "xent_loss": op_xent_loss,
}


def gemm_flops(op) -> float:
    f = 2.0 * op["M"] * op["N"] * op["K"] * op.get("batch", 1)
    return f * 0.5 * (1 + 1 / op["M"]) if op.get("causal", 0) else f
