"""Per-op kernel time of a traced config-4 LoRA step (tools/bench_lora.py
--dump FILE, default builder options), split at the loss vertex into the
forward (hidden under the weights' H2D stream) and the backward (the step's
compute tail): python tools/lora_breakdown.py FILE [layers]."""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2405_16283_b200 import workloads as W  # noqa: E402

d = json.load(open(sys.argv[1]))
layers = int(sys.argv[2]) if len(sys.argv) > 2 else None
g = W.llama_lora_step(W.LLAMA_7B, 4096, layers=layers)
m, t = d["memgraph"], d["trace"]
R = {r["vertex"]: r for r in t["rows"]}
ops = {v["id"]: v.get("op", {}) for v in g.vertices}
names = {vid: t.name for vid, t in g.tensors.items()}
loss_end = max(R[v["id"]]["end"] for v in m["vertices"]
               if v["op"] == "kernel" and "loss" in names.get(v["origin"]["ref"], ""))
agg = {"forward": collections.defaultdict(list), "backward": collections.defaultdict(list)}
for v in m["vertices"]:
    if v["op"] != "kernel":
        continue
    r = R[v["id"]]
    o = ops[v["origin"]["ref"]]
    key = o.get("type")
    if key == "gemm":
        key += f"_{o['M']}x{o['N']}x{o['K']}" + (f"_{o['epilogue']}" if o.get("epilogue") else "")
    agg["backward" if r["start"] >= loss_end else "forward"][key].append(r["end"] - r["start"])
print(f"loss done at {loss_end:.4f} s, step end {t['makespan']:.4f} s")
for ph, a in agg.items():
    tot = sum(sum(v) for v in a.values())
    print(f"== {ph}: kernel busy {tot * 1e3:.1f} ms")
    for k, v in sorted(a.items(), key=lambda x: -sum(x[1]))[:25]:
        v = sorted(v)
        print(f"  {k:40s} n={len(v):4d} total={sum(v) * 1e3:7.2f} ms median={v[len(v) // 2] * 1e6:7.1f} us")
