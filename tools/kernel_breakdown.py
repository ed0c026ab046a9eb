"""Per-op kernel time breakdown of a traced config-5 step (bench_longctx.py --dump)."""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_16283_b200 import workloads as W  # noqa: E402

d = json.load(open(sys.argv[1]))
heads, lag, tile, inter = (int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]) if len(sys.argv) > 5 else (8, 1, 4096, "head")
m, t = d["memgraph"], d["trace"]
R = {r["vertex"]: r for r in t["rows"]}
g = W.blockwise_attention(65536, heads, 128, tile, lag=lag, interleave=inter)
ops = {v["id"]: v.get("op", {}) for v in g.vertices}
agg = collections.defaultdict(list)
for v in m["vertices"]:
    if v["op"] != "kernel":
        continue
    r = R[v["id"]]
    o = ops[v["origin"]["ref"]]
    key = o.get("type")
    if key == "gemm":
        key += f"_{o['M']}x{o['N']}x{o['K']}"
    agg[key].append(r["end"] - r["start"])
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    v = sorted(v)
    print(f"{k:28s} n={len(v):5d} total={sum(v)*1e3:8.2f} ms median={v[len(v)//2]*1e6:8.1f} us p90={v[int(.9*len(v))]*1e6:8.1f}")
