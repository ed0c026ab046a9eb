"""Config 3 structure: tensor-parallel LLaMA prefill memgraph over `tp`
memgraph devices (mapped to the visible GPUs, d % ngpu), transfers = NVLink
peer copies (or D2D when devices share a GPU). Reports step time, bytes moved
per link type and the step roofline."""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_2405_16283_b200 import workloads as W
from paper_2405_16283_b200.executor import Executor

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="65b")
ap.add_argument("--seq", type=int, default=8192)
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--tp", type=int, default=8)
ap.add_argument("--cap-gib", type=float, default=8)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--residency", default="device")
a = ap.parse_args()
cfg = W.LLAMA_65B if a.model == "65b" else W.LLAMA_7B
t0 = time.time()
g = W.llama_prefill_tp(cfg, a.seq, a.tp, layers=a.layers)
mg, st = W.plan(g, [int(a.cap_gib * (1 << 30))] * a.tp, alloc_horizon="lazy")
plan_s = time.time() - t0
ngpu = torch.cuda.device_count()
inputs = {}
for t in g.inputs():  # generate each input on its GPU
    inputs.update(bench.device_inputs_one(t, 0, torch.device("cuda", t.device % ngpu)))
ex = Executor(mg, g.to_json(), {"input_residency": a.residency, "devices": [d % ngpu for d in range(a.tp)]})
for k, v in inputs.items():
    ex.set_input(k, v)
del inputs
ts = []
for s in range(a.steps):
    tr = json.loads(ex.run())
    ts.append(tr["makespan"])
stt = ex.stats()
print(json.dumps({"workload": f"llama_{a.model}_tp{a.tp}_seq{a.seq}_layers{a.layers}_cap{a.cap_gib}GiB",
                  "gpus": ngpu, "memgraph_vertices": len(json.loads(mg)["vertices"]), "plan": st, "plan_s": round(plan_s, 2),
                  "step_s": [round(x, 4) for x in ts], "tokens_per_s": round(a.seq / min(ts), 1),
                  "flops": stt["flops"], "tflops_per_gpu": round(stt["flops"] / min(ts) / 1e12 / ngpu, 1),
                  "p2p_bytes": stt["p2p_bytes"], "d2d_bytes": stt["d2d_bytes"], "h2d_bytes": stt["h2d_bytes"],
                  "kernel_launches": stt["kernel_launches"], "exposed_transfer_s": round(stt["exposed_transfer_s"], 4)}))
