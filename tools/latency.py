"""Dispatch latency microbenchmark: a chain of small kernels."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_2405_16283_b200 import workloads as W
from paper_2405_16283_b200.executor import Executor

g = W.GraphBuilder()
x = g.input("x", (1024,), "f32", init=("normal", 1.0))
for i in range(300):
    x = g.kernel(f"c{i}", {"type": "cast", "args": [x], "count": 1024, "in_dtype": "f32", "out_dtype": "f32"}, (1024,), "f32")
mg, _ = W.plan(g, 1 << 24)
for comp in ["callback", "poll"]:
    ex = Executor(mg, g.to_json(), {"completion": comp})
    ex.set_input(0, W.make_input(g.tensors[0], 0))
    for r in range(3):
        t = json.loads(ex.run())
    rows = sorted(t["rows"], key=lambda r: r["start"])
    ks = [r for r in rows if r["vertex"] != 0]
    gaps = [b["start"] - a["end"] for a, b in zip(ks, ks[1:])]
    print(comp, "makespan %.2f ms" % (t["makespan"] * 1e3), "median gap %.1f us" % (np.median(gaps) * 1e6),
          "median dur %.1f us" % (np.median([r["end"] - r["start"] for r in ks]) * 1e6), ex.stats()["wall_s"])
