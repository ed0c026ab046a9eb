"""Generates the golden fixtures from the UNMODIFIED reference build.

Run here (the reference exists only in this container):
    make -C oracle ref && python tests/golden/make_golden.py
Writes tests/golden/planner_corpus.json: for a corpus following the
reference acceptance recipe (proj/tests/acceptance_main.cpp:107-164, plus
order/victim/horizon/mode/keep_superfluous sweeps), the sha256 of the
reference's serialize_memgraph bytes, its stats, and the sha256 of
simulate()/compare_policies() outputs on each memgraph; plus the full
memgraph JSON of the paper's worked examples (test_compiler.cpp:48-110).
"""
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle", "_ref"))
import _memplan as ref  # noqa: E402

sys.path.insert(0, os.path.join(HERE, ".."))
from corpus import corpus_cases  # noqa: E402


def h(s: str) -> str:
    return hashlib.sha256(s.encode()).hexdigest()


def main():
    cases = []
    for case in corpus_cases():
        g = getattr(ref, case["gen"])(*case["gen_args"])
        entry = dict(case)
        try:
            mg, stats = ref.build_memgraph(g, case["caps"], **case["kw"])
        except Exception as e:  # the error message is part of the contract
            entry["error"] = str(e)
            cases.append(entry)
            continue
        entry["memgraph_sha256"] = h(mg)
        entry["stats"] = stats
        entry["verify_sha256"] = h(ref.verify(g, mg, 0) + ref.verify(g, mg, 200))
        m = json.loads(mg)
        req = [i for i, e in enumerate(m["edges"]) if e["kind"] == "memory" and not e["superfluous"]][:2]
        mut = []
        for i in req:  # racing mutants (acceptance_main.cpp:236-259)
            mm = dict(m)
            mm["edges"] = m["edges"][:i] + m["edges"][i + 1:]
            mut.append(h(ref.verify(g, json.dumps(mm), 50)))
        entry["mutant_verify_sha256"] = mut
        if case.get("simulate"):
            sims = {}
            for pol, tb, prof in case["simulate"]:
                sims[f"{pol}|{tb}|{prof}"] = h(ref.simulate(mg, prof, pol, tb, case["kw"]["seed"]))
            entry["simulate_sha256"] = sims
            entry["compare_sha256"] = h(ref.compare_policies(mg, "", 4, case["kw"]["seed"]))
        cases.append(entry)
    g = ref.gen_matmul(3)
    worked = {
        "five_slots": ref.build_memgraph(g, [5, 5, 5])[0],
        "four_slots": ref.build_memgraph(g, [4, 5, 5], order=[0, 1, 6, 7, 8, 9, 3, 4, 5, 10, 11, 12, 13, 2, 14],
                                         alloc_horizon="lazy")[0],
        "five_slots_trace_seed7": ref.simulate(ref.build_memgraph(g, [5, 5, 5])[0], seed=7),
    }
    cyc = json.loads(worked["five_slots"])
    cyc["edges"].append({"from": 14, "to": 0, "kind": "memory", "superfluous": False})
    worked["cyclic_verify"] = ref.verify(g, json.dumps(cyc), 0)
    out = {"generator": "tests/golden/make_golden.py (reference: oracle/_ref/_memplan)", "cases": cases,
           "worked": worked}
    with open(os.path.join(HERE, "planner_corpus.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print(len(cases), "cases;", sum("error" in c for c in cases), "reference errors")


if __name__ == "__main__":
    main()
