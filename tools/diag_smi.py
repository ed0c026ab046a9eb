"""Does the nvidia-smi clock sampler (bench.Clocks) perturb the timed step?
Alternates blocks of untimed 7B steps with and without the sampler running."""
import json, sys, statistics, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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


def block(n=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(n):
        ex.run(trace=False)
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / n


res = {"no_smi": [], "smi_100ms": [], "smi_1000ms": []}
for rep in range(3):
    res["no_smi"].append(block())
    with bench.Clocks(0) as c:
        res["smi_100ms"].append(block())
    print(json.dumps(c.summary()))
    bench.Clocks.PERIOD_MS = 1000
    with bench.Clocks(0) as c:
        res["smi_1000ms"].append(block())
    bench.Clocks.PERIOD_MS = 100
tr = json.loads(ex.run())
print(json.dumps({k: [round(x, 2) for x in v] for k, v in res.items()} | {"traced_makespan_ms": round(tr["makespan"] * 1e3, 2)}))
