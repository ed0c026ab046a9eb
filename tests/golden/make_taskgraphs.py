"""Generates tests/golden/taskgraphs.json: the toy taskgraphs the planner
corpus builds from, emitted by the UNMODIFIED reference generators
(oracle/_ref/_memplan.gen_matmul / gen_layered / gen_random_dag,
proj/src/taskgraph.cpp:418-616). The generators are out of scope for the
product, so the tests read their outputs from this fixture.

    make -C oracle ref && python tests/golden/make_taskgraphs.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle", "_ref"))
sys.path.insert(0, os.path.join(HERE, ".."))
import _memplan as ref  # noqa: E402

from corpus import gen_args  # noqa: E402


def wanted():
    keys = [gen_args(seed) for seed in range(90)]
    keys += [("gen_random_dag", [14, 0.3, 2, seed]) for seed in range(12)]
    keys += [("gen_layered", [2, 2, 2, 3])] + [("gen_matmul", [p]) for p in (1, 2, 3)]
    return keys


def main():
    out = {}
    for name, args in wanted():
        out[f"{name}{json.dumps(args)}"] = getattr(ref, name)(*args)
    with open(os.path.join(HERE, "taskgraphs.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_taskgraphs.py (reference: oracle/_ref/_memplan gen_*)",
                   "graphs": out}, f, indent=0, sort_keys=True)
    print(len(out), "taskgraphs")


if __name__ == "__main__":
    main()
