"""Event-driven vs fixed-order dispatch ON HARDWARE (the paper's Fig. 10
experiment; reference compare_policies, simulator.cpp:391-417):
the same memgraph executed with both policies, alternating, cold inputs in
pinned host memory. speedup = (fixed - event) / fixed per trial pair."""
import argparse, json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_2405_16283_b200 import memplan, workloads as W
from paper_2405_16283_b200.executor import Executor

ap = argparse.ArgumentParser()
ap.add_argument("--cap-gib", type=float, default=4.0)
ap.add_argument("--seq", type=int, default=4096)
ap.add_argument("--layers", type=int, default=32)
ap.add_argument("--horizon", default="lazy")
ap.add_argument("--trials", type=int, default=5)
ap.add_argument("--residency", default="host")
ap.add_argument("--unfused", action="store_true")
a = ap.parse_args()
g = W.llama_prefill(W.LLAMA_7B, a.seq, layers=a.layers, fused_attention=not a.unfused)
mg, st = W.plan(g, int(a.cap_gib * (1 << 30)), alloc_horizon=a.horizon)
inputs = bench.device_inputs(g, 0, torch.device("cuda", 0))
ex = Executor(mg, g.to_json(), {"input_residency": a.residency})
for k, v in inputs.items():
    ex.set_input(k, v)
del inputs
(o,) = g.outputs()
ex.run(trace=False); ex.run("fixed-order", trace=False)
ev, fx, outs = [], [], set()
for t in range(a.trials):
    e = json.loads(ex.run("event-driven", "fifo", t))["makespan"]; outs.add(ex.get_output(o, 128000))
    f = json.loads(ex.run("fixed-order", "fifo", t))["makespan"]; outs.add(ex.get_output(o, 128000))
    ev.append(e); fx.append(f)
sp = [(f - e) / f for e, f in zip(ev, fx)]
sim = json.loads(memplan.compare_policies(mg, "", 20, 0))
print(json.dumps({"cap_gib": a.cap_gib, "horizon": a.horizon, "residency": a.residency, "plan": st,
                  "event_driven_ms": [round(x * 1e3, 2) for x in ev], "fixed_order_ms": [round(x * 1e3, 2) for x in fx],
                  "speedup_mean": round(statistics.mean(sp), 4), "speedup_min": round(min(sp), 4),
                  "outputs_bitwise_identical": len(outs) == 1,
                  "simulated_speedup_unit_profile": sim["speedup"]["mean"]}))
