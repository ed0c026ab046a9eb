"""Config 4: LLaMA-7B LoRA fine-tuning step (fwd + bwd, seq 4096) with
activation offload under an HBM cap, one B200. Reports step time, host
traffic, the step roofline max(FLOP/peak, H2D/PCIe, D2H/PCIe) and the
event-driven vs fixed-order comparison on hardware."""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_2405_16283_b200 import workloads as W
from paper_2405_16283_b200.executor import Executor

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=4096)
ap.add_argument("--layers", type=int, default=None)
ap.add_argument("--cap-gib", type=float, default=16)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--residency", default="host")
ap.add_argument("--compare", action="store_true")
ap.add_argument("--exec-cfg", default="{}", help="extra executor config keys (JSON)")
ap.add_argument("--horizon", default="lazy")
ap.add_argument("--bwd-prefetch", type=int, default=0)
ap.add_argument("--fused-attention", type=int, default=None, help="1/0: override the builder default")
ap.add_argument("--no-recompute-norms", action="store_true")
ap.add_argument("--no-mn-major", action="store_true", help="explicit transpose vertices in the backward")
ap.add_argument("--dump", default="", help="write the memgraph + one traced step here (JSON)")
a = ap.parse_args()
t0 = time.time()
g = W.llama_lora_step(W.LLAMA_7B, a.seq, layers=a.layers, mn_major=not a.no_mn_major, bwd_prefetch=a.bwd_prefetch,
                      recompute_norms=not a.no_recompute_norms,
                      **({} if a.fused_attention is None else {"fused_attention": bool(a.fused_attention)}))
mg, st = W.plan(g, int(a.cap_gib * (1 << 30)), alloc_horizon=a.horizon)
m = json.loads(mg)
off = sum(v["size"] for v in m["vertices"] if v["op"] == "offload")
plan_s = time.time() - t0
dev = torch.device("cuda", 0)
inputs = bench.device_inputs(g, 0, dev)
ex = Executor(mg, g.to_json(), {"input_residency": a.residency, **json.loads(a.exec_cfg)})
for k, v in inputs.items():
    ex.set_input(k, v)
del inputs
pcie = bench.measure_pcie(dev)
pk = bench.peaks()
ts = bench.untimed_steps(ex, a.steps)  # timing-free completion events
trj = json.loads(ex.run("event-driven", None, 0))
traced = trj["makespan"]
if a.dump:
    with open(a.dump, "w") as f:
        json.dump({"memgraph": m, "trace": trj}, f)
ids = {v["id"]: v for v in json.loads(g.to_json())["vertices"]}
by_op = {}
for r_ in trj["rows"]:
    v = ids.get(r_["vertex"])
    key = ((v.get("op") or {}).get("type") or v["kind"]) if v else "offload/reload"
    if key == "gemm" and v:
        o_ = v["op"]
        key = "gemm_small" if min(o_["M"], o_["N"]) <= 128 else ("gemm_bmm" if o_.get("batch", 1) > 1 else "gemm")
    by_op[key] = by_op.get(key, 0.0) + r_["end"] - r_["start"]
stt = ex.stats()
loss_id = next(o for o in g.outputs() if g.tensors[o].name == "loss")
import struct
loss = struct.unpack("<f", ex.get_output(loss_id, 4))[0]
res = {"workload": f"llama7b_lora_step_seq{a.seq}_cap{a.cap_gib}GiB_{a.residency}_{a.horizon}" + ("_transposes" if a.no_mn_major else "") + (f"_bwdpf{a.bwd_prefetch}" if a.bwd_prefetch else "") + ("_savednorms" if a.no_recompute_norms else "") + ("" if a.fused_attention is None else f"_fusedattn{a.fused_attention}"), "exec_cfg": a.exec_cfg, "memgraph_vertices": len(m["vertices"]),
       "plan": st, "plan_s": round(plan_s, 2), "offload_gb": round(off / 1e9, 1), "step_s": [round(x, 4) for x in ts], "traced_step_makespan_s": round(traced, 4),
       "loss": loss, "tokens_per_s": round(a.seq / min(ts), 1), "flops": stt["flops"],
       "h2d_gb": round(stt["h2d_bytes"] / 1e9, 2), "d2h_gb": round(stt["d2h_bytes"] / 1e9, 2),
       "pcie_h2d_measured_gbs": round(pcie, 1), "kernel_busy_s": round(stt["kernel_busy_s"], 4),
       "exposed_transfer_s": round(stt["exposed_transfer_s"], 4),
       "device_time_by_op_s": {k: round(v, 4) for k, v in sorted(by_op.items(), key=lambda kv: -kv[1])}}
roof = max(stt["flops"] / (pk["bf16_tflops_sustained"] * 1e12), stt["h2d_bytes"] / (pcie * 1e9),
           stt["d2h_bytes"] / (pcie * 1e9))
res["roofline_s"] = round(roof, 4)
res["plan_ideal_s"] = round(bench.plan_ideal_s(mg, pcie), 4)
res["frac_of_roofline"] = round(roof / min(ts), 4)
if a.compare:
    fx = bench.untimed_steps(ex, a.steps, "fixed-order")
    res["fixed_order_step_s"] = [round(x, 4) for x in fx]
    res["event_driven_speedup"] = round((min(fx) - min(ts)) / min(fx), 4)
print(json.dumps(res), flush=True)
