"""Memgraph construction is bit-exact with the reference.

Pinned three ways: (1) the committed golden corpus generated from the
unmodified reference build (tests/golden/make_golden.py), (2) the paper's
worked examples (proj/tests/test_compiler.cpp:48-110, acceptance_main.cpp:47-94),
(3) a live differential run against oracle/_ref when it is present.
"""
import hashlib
import json
import os

import pytest

from corpus import corpus_cases, taskgraph
from paper_2405_16283_b200 import memplan

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "planner_corpus.json")))


def sha(s):
    return hashlib.sha256(s.encode()).hexdigest()


def test_golden_corpus_bit_exact():
    cases = GOLD["cases"]
    mine = list(corpus_cases())
    assert len(mine) == len(cases)
    n_err = 0
    for want, case in zip(cases, mine):
        assert case["gen_args"] == want["gen_args"] and case["kw"] == want["kw"] and case["caps"] == want["caps"]
        g = taskgraph(case["gen"], case["gen_args"])
        try:
            mg, stats = memplan.build_memgraph(g, case["caps"], **case["kw"])
        except memplan.MemplanError as e:
            assert "error" in want, (case, str(e))
            assert str(e) == want["error"]
            n_err += 1
            continue
        assert "error" not in want, (case, want["error"])
        assert sha(mg) == want["memgraph_sha256"], case
        assert stats == want["stats"], case
        for key, hsum in want.get("simulate_sha256", {}).items():
            pol, tb, prof = key.split("|", 2)
            assert sha(memplan.simulate(mg, prof, pol, tb, case["kw"]["seed"])) == hsum, (case, key)
        assert sha(memplan.verify(g, mg, 0) + memplan.verify(g, mg, 200)) == want["verify_sha256"], case
        m = json.loads(mg)
        req = [i for i, e in enumerate(m["edges"]) if e["kind"] == "memory" and not e["superfluous"]][:2]
        for i, hsum in zip(req, want["mutant_verify_sha256"]):
            mm = dict(m)
            mm["edges"] = m["edges"][:i] + m["edges"][i + 1:]
            rep = memplan.verify(g, json.dumps(mm), 50)
            assert sha(rep) == hsum, case
            assert json.loads(rep)["all_passed"] is False  # every required memory edge matters
        if "compare_sha256" in want:
            assert sha(memplan.compare_policies(mg, "", 4, case["kw"]["seed"])) == want["compare_sha256"]
    assert n_err > 50  # the corpus deliberately includes wedged / too-small capacities


def test_worked_example_five_slots():
    g = taskgraph("gen_matmul", [3])
    mg, stats = memplan.build_memgraph(g, [5, 5, 5])
    assert mg == GOLD["worked"]["five_slots"]
    assert stats == {"offloads": 0, "reloads": 0, "memory_edges": 2, "required_memory_edges": 1,
                     "peak_usage": [5, 5, 3]}
    m = json.loads(mg)
    pl = m["placement"]
    assert pl["0"]["offset"] == pl["13"]["offset"] and pl["1"]["offset"] == pl["14"]["offset"]
    mem = {(e["from"], e["to"]): e for e in m["edges"] if e["kind"] == "memory"}
    assert not mem[(2, 13)]["superfluous"] and mem[(2, 14)]["superfluous"]
    assert memplan.simulate(mg, seed=7) == GOLD["worked"]["five_slots_trace_seed7"]


def test_worked_example_four_slots():
    g = taskgraph("gen_matmul", [3])
    order = [0, 1, 6, 7, 8, 9, 3, 4, 5, 10, 11, 12, 13, 2, 14]
    mg, stats = memplan.build_memgraph(g, [4, 5, 5], order=order, alloc_horizon="lazy")
    assert mg == GOLD["worked"]["four_slots"]
    assert stats["offloads"] == 1 and stats["reloads"] == 1
    m = json.loads(mg)
    off = [v for v in m["vertices"] if v["origin"]["kind"] == "offload"]
    rel = [v for v in m["vertices"] if v["origin"]["kind"] == "reload"]
    assert off[0]["origin"]["ref"] == 0 and rel[0]["origin"]["ref"] == 0
    mem = {(e["from"], e["to"]) for e in m["edges"] if e["kind"] == "memory"}
    assert (off[0]["id"], 13) in mem and (13, rel[0]["id"]) in mem


def test_verifier_cycle_witness():
    cyc = json.loads(GOLD["worked"]["five_slots"])
    cyc["edges"].append({"from": 14, "to": 0, "kind": "memory", "superfluous": False})
    assert memplan.verify(taskgraph("gen_matmul", [3]), json.dumps(cyc), 0) == GOLD["worked"]["cyclic_verify"]


def test_byte_mode_first_fit_offsets():
    """proj/tests/test_compiler.cpp:150-182."""
    g = json.dumps({"device_count": 1, "vertices": [
        {"id": 0, "kind": "input", "device": 0, "output_size": 20},
        {"id": 1, "kind": "input", "device": 0, "output_size": 25},
        {"id": 2, "kind": "kernel", "device": 0, "output_size": 5},
        {"id": 3, "kind": "kernel", "device": 0, "output_size": 15},
        {"id": 4, "kind": "kernel", "device": 0, "output_size": 5}], "edges": [[0, 2], [2, 3], [1, 4]]})
    mg, _ = memplan.build_memgraph(g, [50], mode="byte", order=[0, 1, 2, 3, 4])
    pl = json.loads(mg)["placement"]
    assert [pl[str(i)]["offset"] for i in range(5)] == [0, 20, 45, 0, 15]
    e = [x for x in json.loads(mg)["edges"] if x["kind"] == "memory" and (x["from"], x["to"]) == (2, 4)]
    assert e and not e[0]["superfluous"]


def test_errors_match_reference_taxonomy():
    g = json.dumps({"device_count": 1, "vertices": [{"id": 0, "kind": "input", "device": 0, "output_size": 10}],
                    "edges": []})
    with pytest.raises(memplan.MemplanError, match="exceeds device 0 capacity 5"):
        memplan.build_memgraph(g, [5], mode="byte", order=[0])
    chain = json.dumps({"device_count": 1, "vertices": [{"id": 0, "kind": "input", "device": 0},
                                                        {"id": 1, "kind": "kernel", "device": 0}], "edges": [[0, 1]]})
    with pytest.raises(memplan.MemplanError, match="linear extension"):
        memplan.build_memgraph(chain, [4], order=[1, 0])
    with pytest.raises(memplan.MemplanError, match="one entry per device"):
        memplan.build_memgraph(taskgraph("gen_matmul", [2]), [4])
    bounce = json.dumps({"device_count": 2, "vertices": [
        {"id": 0, "kind": "input", "device": 0}, {"id": 1, "kind": "input", "device": 1},
        {"id": 2, "kind": "transfer", "device": 0, "src_device": 1},
        {"id": 3, "kind": "transfer", "device": 1, "src_device": 0},
        {"id": 4, "kind": "transfer", "device": 1, "src_device": 0}], "edges": [[1, 2], [2, 3], [0, 4]]})
    with pytest.raises(memplan.MemplanError, match="host capacity exceeded"):
        memplan.build_memgraph(bounce, [1, 8], order=[0, 1, 2, 3, 4], host_capacity=0)
    with pytest.raises(memplan.MemplanError):
        memplan.build_memgraph("{}", [1])


def test_live_differential_vs_reference(ref_memplan):
    """Same corpus recipe, fresh seeds, byte-compared against oracle/_ref."""
    n = 0
    for seed in range(200, 260):
        from corpus import gen_args
        name, args = gen_args(seed)
        g = getattr(ref_memplan, name)(*args)
        assert ref_memplan.validate_taskgraph(g) == memplan.validate_taskgraph(g)
        for pol in ("as-listed", "depth-first", "min-memory-greedy"):
            assert ref_memplan.topological_order(g, pol, seed) == memplan.topological_order(g, pol, seed)
        for caps_scale in (1, 2):
            gj = json.loads(g)
            caps = [caps_scale * 3 + 2] * gj["device_count"]
            for hz in ("greedy", "lazy"):
                kw = dict(alloc_horizon=hz, victim_policy=["farthest-next-use", "last-allocated",
                                                           "seeded-random"][seed % 3], seed=seed)
                try:
                    a = ref_memplan.build_memgraph(g, caps, **kw)
                except Exception as e:
                    with pytest.raises(memplan.MemplanError, match=None) as ei:
                        memplan.build_memgraph(g, caps, **kw)
                    assert str(ei.value) == str(e)
                    continue
                b = memplan.build_memgraph(g, caps, **kw)
                assert a == b
                assert ref_memplan.memgraph_to_dot(a[0]) == memplan.memgraph_to_dot(a[0])
                n += 1
    assert n > 100


def test_large_llama_plan_matches_reference(ref_memplan):
    """A LLaMA-shaped byte-mode graph (with op payloads the reference
    ignores) plans identically; the reference takes seconds, we take less."""
    from paper_2405_16283_b200 import workloads as W

    g = W.llama_prefill(W.LlamaConfig(dim=1024, layers=6, heads=8, ffn=2816, vocab=4000), 512,
                        fused_attention=False).to_json()
    for caps, hz, spills in (([54 << 20], "greedy", False), ([26 << 20], "lazy", True), ([35 << 20], "lazy", True)):
        a = ref_memplan.build_memgraph(g, caps, mode="byte", alloc_horizon=hz)
        b = memplan.build_memgraph(g, caps, mode="byte", alloc_horizon=hz)
        assert a == b
        assert (a[1]["offloads"] > 0) == spills
    gf = W.llama_prefill(W.LlamaConfig(dim=1024, layers=6, heads=8, ffn=2816, vocab=4000), 512).to_json()
    for caps, hz in (([20 << 20], "lazy"), ([40 << 20], "greedy")):
        assert ref_memplan.build_memgraph(gf, caps, mode="byte", alloc_horizon=hz) == \
            memplan.build_memgraph(gf, caps, mode="byte", alloc_horizon=hz)


def test_verifier_certifies_large_plans():
    """The scalable verifier certifies BASELINE-size plans the reference's
    O(P^2 * BFS) checks cannot finish."""
    import time
    from paper_2405_16283_b200 import workloads as W
    for g, cap, hz in ((W.llama_prefill(W.LLAMA_7B, 4096), 16 << 30, "greedy"),
                       (W.blockwise_attention(65536, 32, 128, 8192, lag=8), 16 << 30, "lazy")):
        mg, st = W.plan(g, cap, alloc_horizon=hz)
        t0 = time.time()
        rep = json.loads(memplan.verify(g.to_json(), mg, 0))
        assert rep["all_passed"], rep
        assert time.time() - t0 < 30


def test_scale_goldens_bit_exact():
    """BASELINE-shaped plans of 424 to 27,104 vertices (LoRA 7B step with 656
    offloads, 64k blockwise attention with 3,568 offloads, 65B TP8 over 8
    devices, the 7B bench plan) are byte-identical to the reference build
    (tests/golden/scale_corpus.json from make_scale_golden.py; the reference
    needed up to 183 s for one of them)."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_scale_golden import cases

    gold = {c["name"]: c for c in json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                                               "scale_corpus.json")))["cases"]}
    assert len(gold) == len(cases())
    for name, mk, caps, kw in cases():
        want = gold[name]
        tg = mk().to_json()
        assert sha(tg) == want["taskgraph_sha256"], name  # the generator itself is unchanged
        mg, stats = memplan.build_memgraph(tg, caps, mode="byte", **kw)
        assert stats == want["stats"], name
        assert sha(mg) == want["memgraph_sha256"], name
