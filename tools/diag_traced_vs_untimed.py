import json, sys, os
sys.path.insert(0, '/root/repo')
import bench, torch
from paper_2405_16283_b200 import workloads as W
from paper_2405_16283_b200.executor import Executor
g = W.llama_prefill(W.LLAMA_7B, 4096)
mg, _ = W.plan(g, 16 << 30)
ex = Executor(mg, g.to_json(), {"devices": [0], "input_residency": "device"})
for k, v in bench.device_inputs(g, 0, torch.device("cuda", 0)).items():
    ex.set_input(k, v)
for _ in range(3):
    ex.run(trace=False)
seq = [False]*5 + [True]*3 + [False]*30 + [True]*3 + [False]*3 + [True]*2
out = []
for tr in seq:
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    r = ex.run(trace=tr)
    e.record()
    torch.cuda.synchronize()
    d = {"traced": tr, "event_ms": round(s.elapsed_time(e), 2)}
    if tr:
        t = json.loads(r)
        rows = t["rows"]
        d["makespan_ms"] = round(t["makespan"] * 1e3, 2)
        d["first_start_ms"] = round(min(x["start"] for x in rows if x["end"] > 0) * 1e3, 3)
        d["rows"] = len(rows)
    out.append(d)
for d in out:
    print(json.dumps(d))
