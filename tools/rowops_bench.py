"""RMSNorm micro-benchmark through the executor: a chain of R rmsnorm
vertices over a [rows, cols] bf16 activation (each reads the previous
output, so inputs are L2-hot as inside the 7B step). Reports the per-vertex
CUDA-event time and the implied HBM-equivalent GB/s (read + write)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_2405_16283_b200 import workloads as W
from paper_2405_16283_b200.executor import Executor

rows, cols, R = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 4096, 16)))
g = W.GraphBuilder()
x = g.input("x", (rows, cols), "bf16", init=("normal", 1.0))
w = g.input("w", (cols,), "bf16", init=("normal", 1.0))
for i in range(R):
    x = g.kernel(f"n{i}", {"type": "rmsnorm", "args": [x, w], "rows": rows, "cols": cols, "eps": 1e-5}, (rows, cols), "bf16")
mg, _ = W.plan(g, 1 << 32)
with Executor(mg, g.to_json(), {"input_residency": "device"}) as ex:
    for t in g.inputs():
        ex.set_input(t.id, torch.randn(*t.shape, device="cuda").to(torch.bfloat16))
    best = None
    for _ in range(5):
        tr = json.loads(ex.run())
        ks = sorted(r["end"] - r["start"] for r in tr["rows"] if r["vertex"] > 1)
        med = ks[len(ks) // 2]
        best = med if best is None else min(best, med)
print(json.dumps({"rows": rows, "cols": cols, "us": round(best * 1e6, 2), "gbs": round(4 * rows * cols / best / 1e9, 1)}))
