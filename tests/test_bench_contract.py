"""bench.py helpers that do not need a GPU: the roofline bookkeeping over a
trace, and the reference arm's live planner leg (oracle/_ref)."""
import json
import os

import pytest

import bench
from paper_2405_16283_b200 import workloads as W


def test_roofline_from_trace_counts_gemm_flops_and_bytes():
    cfg = W.LlamaConfig(dim=512, layers=2, heads=4, ffn=1024, vocab=1000)
    g = W.llama_prefill(cfg, 256)
    rows = [{"vertex": v["id"], "start": 0.0, "end": 1e-3} for v in g.vertices]
    roof, by_type = bench.roofline_from_trace(g, {"rows": rows}, 1000.0)
    gemms = [v for v in g.vertices if (v.get("op") or {}).get("type") == "gemm"]
    assert roof["launches_per_step"] == len(gemms)
    assert roof["algorithmic_flops_per_step"] == pytest.approx(sum(bench.gemm_flops(v["op"]) for v in gemms))
    assert roof["unit"] == "TFLOP/s" and roof["bound"] == "tensor"
    assert sum(c["n"] for c in roof["gemm_classes"].values()) == len(gemms)
    assert roof["algorithmic_bytes_per_launch"] > 0
    assert by_type["gemm"] == pytest.approx(1e-3 * len(gemms))


def test_attention_roofline_flops_and_bytes():
    cfg = W.LlamaConfig(dim=512, layers=2, heads=4, ffn=1024, vocab=1000)
    S = 256
    g = W.llama_prefill(cfg, S)
    rows = [{"vertex": v["id"], "start": 0.0, "end": 1e-9} for v in g.vertices]  # TF/s rounded to 0.1
    att = bench.attention_roofline(g, {"rows": rows}, 1000.0)
    assert att["launches_per_step"] == cfg.layers
    hd = cfg.dim // cfg.heads
    per = 4.0 * cfg.heads * S * S * hd * 0.5 * (1 + 1 / S)  # causal
    assert att["achieved"] == pytest.approx(per / 1e-9 / 1e12, rel=1e-3)
    assert att["frac"] == pytest.approx(att["achieved"] / 1000.0, rel=1e-3)
    assert att["algorithmic_bytes_per_launch"] == 4 * cfg.heads * S * hd * 2  # q, k, vT in; O out
    no_attn = W.GraphBuilder()
    no_attn.input("x", (4, 4), "bf16")
    assert bench.attention_roofline(no_attn, {"rows": []}, 1000.0) is None


def test_planner_parity_leg_is_byte_identical():
    if not os.path.isdir(os.path.join(bench.ROOT, "oracle", "_ref")):
        pytest.skip("oracle/_ref not built")
    cfg = W.LlamaConfig(dim=512, layers=2, heads=4, ffn=1024, vocab=1000)
    g = W.llama_prefill(cfg, 256)
    leg = bench.planner_parity(g, [64 << 20], "greedy")
    if "unavailable" in leg:
        pytest.skip(leg["unavailable"])
    assert leg["memgraph_bytes_identical"]
    assert leg["vertices"] == len(json.loads(W.plan(g, 64 << 20)[0])["vertices"])


def test_both_arms_share_the_config():
    import argparse
    a = argparse.Namespace(layers=None, seq=4096, cap_gib=16.0, horizon="greedy", mode="tp", quick=False)
    c1, c8 = bench.bench_config(a, 1), bench.bench_config(a, 8)
    assert c1["workload"] == "llama7b_prefill_seq4096_cap16GiB" and c1["layers"] == 32
    assert c8["workload"].endswith("_tp8") and c8["global_batch"] == 1
    _, g = bench.make_graph(argparse.Namespace(**{**vars(a), "seq": 256, "layers": 1}), 2)
    assert g.device_count == 2  # N > 1: the partitioned (TP) memgraph


def test_input_h2d_bytes_per_device():
    cfg = W.LlamaConfig(dim=512, layers=2, heads=4, ffn=1024, vocab=1000)
    g = W.llama_prefill_tp(cfg, 256, 2)
    mg, _ = W.plan(g, [64 << 20] * 2)
    per = bench.input_h2d_bytes_per_device(g, mg, 2)
    tables = sum(t.nbytes for t in g.inputs() if t.name.startswith("tok_embeddings"))
    assert sum(per) == sum(t.nbytes for t in g.inputs()) - tables + 2 * 256 * 512 * 2
