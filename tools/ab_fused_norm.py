"""Paired A/B of the 7B prefill step with and without the fused-RMSNorm graph
option (same process, same box, alternating blocks of timed steps), so the
clock / power-cap drift between runs does not decide the comparison."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import torch  # noqa: E402

from paper_2405_16283_b200 import workloads as W  # noqa: E402
from paper_2405_16283_b200.executor import Executor  # noqa: E402


def make(fused):
    g = W.llama_prefill(W.LLAMA_7B, 4096, fused_norm=fused)
    mg, _ = W.plan(g, 16 << 30)
    ex = Executor(mg, g.to_json(), {"devices": [0], "input_residency": "device"})
    for k, v in bench.device_inputs(g, 0, torch.device("cuda", 0)).items():
        ex.set_input(k, v)
    return ex


def block(ex, n):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        ex.run(trace=False)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


exs = {"unfused": make(False), "fused": make(True)}
for ex in exs.values():
    for _ in range(3):
        ex.run(trace=False)
res = {k: [] for k in exs}
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    for k, ex in (exs.items() if rep % 2 == 0 else reversed(list(exs.items()))):
        res[k].append(block(ex, 10))
print(json.dumps({k: {"median_ms": round(statistics.median(v), 3), "all": [round(x, 2) for x in v]} for k, v in res.items()}))
