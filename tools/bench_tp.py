"""Config 3: tensor-parallel LLaMA prefill memgraph over `tp` memgraph devices
(mapped to the visible GPUs, d % ngpu), transfers = NVLink peer copies (or
D2D when devices share a GPU). Weights cold in pinned host RAM by default
(--residency host), so every step streams them H2D under the per-device cap.
Reports step time, bytes moved per link type, exposed transfer time and the
step roofline max(FLOP / sustained bf16 peak per GPU, H2D bytes / PCIe per GPU).

Inputs are generated one at a time on the GPU and handed to the executor
(which copies them into its pinned pool), so the device never holds more than
the arenas plus one weight tensor."""
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
ap.add_argument("--residency", default="host")
ap.add_argument("--execution", default="events")
a = ap.parse_args()
cfg = W.LLAMA_65B if a.model == "65b" else W.LLAMA_7B
t0 = time.time()
g = W.llama_prefill_tp(cfg, a.seq, a.tp, layers=a.layers)
mg, st = W.plan(g, [int(a.cap_gib * (1 << 30))] * a.tp, alloc_horizon="lazy")
plan_s = time.time() - t0
ngpu = torch.cuda.device_count()
ex = Executor(mg, g.to_json(), {"input_residency": a.residency, "devices": [d % ngpu for d in range(a.tp)],
                                "execution": a.execution})
t1 = time.time()
in_bytes = 0
for t in g.inputs():  # generate each input on its GPU, hand it over, drop it
    for k, v in bench.device_inputs_one(t, 0, torch.device("cuda", t.device % ngpu)).items():
        ex.set_input(k, v)
        in_bytes += v.numel() * v.element_size()
        del v
torch.cuda.empty_cache()
load_s = time.time() - t1
ts = bench.untimed_steps(ex, a.steps)  # timing-free completion events
st_untimed = ex.stats()
tr = json.loads(ex.run())  # one traced step (per-vertex timestamps) for the breakdown
ids = {v["id"]: v for v in json.loads(g.to_json())["vertices"]}
by_op = {}
for r_ in tr["rows"]:
    v = ids.get(r_["vertex"])
    key = ((v.get("op") or {}).get("type") or v["kind"]) if v else "offload/reload"
    by_op[key] = by_op.get(key, 0.0) + r_["end"] - r_["start"]
stt = ex.stats()
pk = bench.peaks()
pcie = bench.measure_pcie(torch.device("cuda", 0))
step = min(ts)
compute_s = stt["flops"] / (pk["bf16_tflops_sustained"] * 1e12 * ngpu)
pcie_s = stt["h2d_bytes"] / (pcie * 1e9 * ngpu)
bound = max(compute_s, pcie_s)
print(json.dumps({"workload": f"llama_{a.model}_tp{a.tp}_seq{a.seq}_layers{a.layers}_cap{a.cap_gib}GiB_{a.residency}",
                  "gpus": ngpu, "memgraph_vertices": len(json.loads(mg)["vertices"]), "plan": st,
                  "plan_s": round(plan_s, 2), "input_load_s": round(load_s, 1), "input_bytes": in_bytes,
                  "step_s": [round(x, 4) for x in ts], "traced_step_makespan_s": round(tr["makespan"], 4),
                  "tokens_per_s": round(a.seq / step, 1),
                  "flops": stt["flops"], "tflops_per_gpu": round(stt["flops"] / step / 1e12 / ngpu, 1),
                  "p2p_bytes": stt["p2p_bytes"], "d2d_bytes": stt["d2d_bytes"], "h2d_bytes": stt["h2d_bytes"],
                  "d2h_bytes": stt["d2h_bytes"], "kernel_launches": stt["kernel_launches"],
                  "exposed_transfer_s": round(stt["exposed_transfer_s"], 4),
                  "exposed_transfer_gpu_s": round(stt["exposed_transfer_gpu_s"], 4), "pcie_h2d_gbs": round(pcie, 1),
                  "host_dispatch_s": round(stt["host_dispatch_s"], 4), "host_wait_s": round(stt["host_wait_s"], 4),
                  "untimed_host_dispatch_s": round(st_untimed["host_dispatch_s"], 4),
                  "untimed_host_dispatch_us_per_vertex": round(st_untimed["host_dispatch_s"] * 1e6 / len(json.loads(mg)["vertices"]), 2),
                  "execution": a.execution, "graph_nodes": st_untimed.get("graph_nodes", 0),
                  "roofline": {"compute_s": round(compute_s, 4), "pcie_h2d_s": round(pcie_s, 4),
                               "bound": "pcie" if pcie_s > compute_s else "tensor",
                               "frac": round(bound / step, 4)},
                  "device_time_by_op_s": {k: round(v, 4) for k, v in sorted(by_op.items(), key=lambda kv: -kv[1])}}))
