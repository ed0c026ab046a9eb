"""Shared fixtures: small op-payload graphs, their inputs and comparisons."""
import json
import os

import numpy as np

from oracle import ops_ref
from oracle.cpu_executor import CpuExecutor, linear_extension
from paper_2405_16283_b200 import workloads as W

SMALL = W.LlamaConfig(dim=512, layers=2, heads=4, ffn=1024, vocab=1000)


def small_llama(seq=256, layers=2, cap_factor=1.5, hz="lazy"):
    g = W.llama_prefill(SMALL, seq, layers=layers)
    cap = int(W.working_set_floor(g)[0] * cap_factor) // 1024 * 1024
    mg, stats = W.plan(g, cap, alloc_horizon=hz)
    return g, mg, stats


def inputs_of(g, seed=0):
    return {t.id: W.make_input(t, seed) for t in g.inputs()}


def as_f32(raw: bytes, dtype: str, n: int) -> np.ndarray:
    b = np.frombuffer(raw, dtype=np.uint8)
    return ops_ref.load(b, dtype, n).astype(np.float32)


def out_values(g, vid, raw):
    t = g.tensors[vid]
    return as_f32(raw, t.dtype, int(np.prod(t.shape)))


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def oracle_outputs(g, mg, inputs, schedule="total_order", seed=0):
    ex = CpuExecutor(mg, g.to_json())
    for vid, a in inputs.items():
        ex.set_input(vid, a)
    sched = linear_extension(json.loads(mg), schedule, seed)
    return ex.run(sched, outputs=g.outputs())


def direct_forward(g, inputs):
    """Evaluates the taskgraph straight (no memgraph, no arena reuse)."""
    bufs = {}
    for v in g.vertices:
        vid = v["id"]
        out = np.zeros(v["output_size"], dtype=np.uint8)
        if v["kind"] == "input":
            b = np.frombuffer(inputs[vid].tobytes(), dtype=np.uint8)
            out[: b.size] = b
        elif v["kind"] == "transfer":
            (src,) = [p for p, c in g.edges if c == vid]
            out[:] = bufs[src][: out.size]
        else:
            op = v["op"]
            ops_ref.OPS[op["type"]](op, [bufs[a] for a in op["args"]], out)
        bufs[vid] = out
    return {o: bufs[o].tobytes() for o in g.outputs()}


def replay_capacity(mg_json, order):
    """Restates verifier.cpp:198-288 check_capacity for an arbitrary order."""
    m = json.loads(mg_json)
    pos = {v: i for i, v in enumerate(order)}
    readers = {}
    for e in m["edges"]:
        if e["kind"] == "data":
            readers.setdefault(e["from"], []).append(e["to"])
    iv = []
    for k, p in m["placement"].items():
        vid = int(k)
        rs = readers.get(vid, [])
        end = max(pos[r] for r in rs) if rs else None
        iv.append((vid, p["device"], p["offset"], p["size"], pos[vid], end))
    for i in range(len(iv)):
        for j in range(i + 1, len(iv)):
            a, b = iv[i], iv[j]
            if a[1] != b[1] or not (a[2] < b[2] + b[3] and b[2] < a[2] + a[3]):
                continue
            disjoint = (a[5] is not None and a[5] < b[4]) or (b[5] is not None and b[5] < a[4])
            assert disjoint, f"regions of {a[0]} and {b[0]} overlap while both live"


def tp_inputs_from_full(g_tp, g_full, full_inputs, cfg, tp):
    """Shards single-device LLaMA inputs into the TP graph's per-device inputs
    (Megatron slicing: QKV / gate-up rows by head / ffn column, O / down by K)."""
    by_name = {g_full.tensors[v].name: a for v, a in full_inputs.items()}
    d, hd, f = cfg.dim, cfg.hd, cfg.ffn
    Hl, fl = cfg.heads // tp, f // tp
    dl = Hl * hd
    out = {}
    for t in g_tp.inputs():
        base, _, dev = t.name.partition("@")
        r = int(dev) if dev else 0
        a = by_name[base]
        if base.endswith("wqkv"):
            w = a.reshape(3 * d, d)
            a = np.concatenate([w[j * d + r * dl: j * d + (r + 1) * dl] for j in range(3)])
        elif base.endswith("w13"):
            w = a.reshape(2 * f, d)
            a = np.concatenate([w[r * fl:(r + 1) * fl], w[f + r * fl: f + (r + 1) * fl]])
        elif base.endswith(".wo"):
            a = a.reshape(d, d)[:, r * dl:(r + 1) * dl]
        elif base.endswith(".w2"):
            a = a.reshape(d, f)[:, r * fl:(r + 1) * fl]
        out[t.id] = np.ascontiguousarray(a).reshape(-1)
    return out


def inputs_with_in_edges(mg_json) -> int:
    """Input vertices that must wait for earlier vertices (memory edges into
    an input reusing a freed region; SURVEY hard part 3)."""
    m = json.loads(mg_json)
    ins = {v["id"] for v in m["vertices"] if v["op"] == "input"}
    return len({e["to"] for e in m["edges"] if e["to"] in ins})


def record_err(test, **kw):
    """Appends measured errors to $PARITY_LOG (JSON lines) when set: the
    evidence the stated tolerances are derived from (about 2x the measured)."""
    p = os.environ.get("PARITY_LOG")
    if p:
        with open(p, "a") as f:
            f.write(json.dumps({"test": test, **kw}) + "\n")
