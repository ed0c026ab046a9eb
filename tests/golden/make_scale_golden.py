"""Scale goldens: bit-exact memgraph construction at thousands of vertices,
generated from the UNMODIFIED reference build (oracle/_ref/_memplan).

Run here (the reference sources exist only in this container):
    make -C oracle ref && python tests/golden/make_scale_golden.py
Writes tests/golden/scale_corpus.json: for each BASELINE-shaped plan
(config 4 LoRA step, config 5 blockwise attention, config 3 TP8 prefill) the
sha256 of the taskgraph JSON our generator emits, the sha256 of the
reference's serialize_memgraph bytes, its stats and the reference's build
time. tests/test_planner_golden.py rebuilds each with our planner and
compares bytes (compiler.cpp:487-585 at 4k-9k vertices, where
the windowed prune and the rank-ordered ghost map could diverge).
"""
import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.join(HERE, "..", "..")
sys.path.insert(0, ROOT)
from paper_2405_16283_b200 import workloads as W  # noqa: E402

GIB = 1 << 30


def cases():
    """(name, taskgraph builder, capacities, build kwargs) — shared with the test."""
    return [
        ("lora7b_seq4096_cap16GiB_lazy", lambda: W.llama_lora_step(W.LLAMA_7B, 4096, recompute_ffn=False,
                                                                    recompute_qkv=False, mn_major=False,
                                                                    recompute_norms=False), [16 * GIB],
         {"alloc_horizon": "lazy"}),
        ("lora7b_seq4096_cap16GiB_lazy_saveP", lambda: W.llama_lora_step(W.LLAMA_7B, 4096, recompute_attention=False,
                                                                         recompute_ffn=False, recompute_qkv=False,
                                                                         mn_major=False, recompute_norms=False),
         [16 * GIB], {"alloc_horizon": "lazy"}),
        ("lora7b_seq4096_cap16GiB_lazy_recompute", lambda: W.llama_lora_step(W.LLAMA_7B, 4096), [16 * GIB],
         {"alloc_horizon": "lazy"}),
        ("lora7b_seq4096_cap12GiB_lazy_fused", lambda: W.llama_lora_step(W.LLAMA_7B, 4096), [12 * GIB],
         {"alloc_horizon": "lazy"}),
        ("blockwise_seq65536_h32_tile4096_lag8_cap16GiB_lazy",
         lambda: W.blockwise_attention(65536, 32, 128, 4096, lag=8), [16 * GIB], {"alloc_horizon": "lazy"}),
        ("llama65b_tp8_seq8192_layers10_cap0.9GiB_lazy", lambda: W.llama_prefill_tp(W.LLAMA_65B, 8192, 8, layers=10),
         [int(0.9 * GIB) // 1024 * 1024] * 8, {"alloc_horizon": "lazy"}),
        ("llama7b_prefill_seq4096_cap16GiB_greedy", lambda: W.llama_prefill(W.LLAMA_7B, 4096), [16 * GIB],
         {"alloc_horizon": "greedy"}),
    ]


def h(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()


def main(only=None):
    """Rebuilds every case with the reference (or only the named ones, keeping
    the other entries of the existing corpus)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
    import _memplan as ref

    out = []
    old = {}
    if only:
        old = {c["name"]: c for c in json.load(open(os.path.join(HERE, "scale_corpus.json")))["cases"]}
    for name, mk, caps, kw in cases():
        if only and name not in only:
            out.append(old[name])
            continue
        tg = mk().to_json()
        t0 = time.perf_counter()
        mg, stats = ref.build_memgraph(tg, caps, mode="byte", **kw)
        dt = time.perf_counter() - t0
        m = json.loads(mg)
        out.append({"name": name, "taskgraph_sha256": h(tg), "memgraph_sha256": h(mg), "stats": stats,
                    "vertices": len(m["vertices"]), "edges": len(m["edges"]), "reference_build_s": round(dt, 1)})
        print(json.dumps(out[-1]), flush=True)
    with open(os.path.join(HERE, "scale_corpus.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_scale_golden.py (reference: oracle/_ref/_memplan)",
                   "cases": out}, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or None)
