"""Config 1: tiled fp32 matmul chain (4096², tile 1024, L=4) partitioned over
2 memgraph devices with a cap forcing offload/reload, executed on the GPU
(tf32 tcgen05 tiles, fixed-order k-combines, transfers) and on the CPU oracle
executor (the reference configuration "on the CPU reference executor");
reports both times and the tf32-vs-fp32 error."""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
from helpers import inputs_of, oracle_outputs, out_values, rel_err
from paper_2405_16283_b200 import workloads as W
from paper_2405_16283_b200.executor import Executor

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--tile", type=int, default=1024)
ap.add_argument("--chain", type=int, default=4)
ap.add_argument("--cap-floor", type=float, default=1.5,
                help="per-device cap as a multiple of the working-set floor (1.5 -> 128 offloads)")
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
g = W.matmul_chain(a.n, a.tile, a.chain, devices=2)
tot = [0, 0]
for v in g.vertices:
    tot[v["device"]] += v["output_size"]
floor = W.working_set_floor(g)
caps = [int(f * a.cap_floor) // 1024 * 1024 for f in floor]
mg, st = W.plan(g, caps, alloc_horizon="lazy")
inp = inputs_of(g, seed=0)
ngpu = torch.cuda.device_count()
ex = Executor(mg, g.to_json(), {"devices": [0, 1 % ngpu]})
for k, v in inp.items():
    ex.set_input(k, v)
import bench
ts = bench.untimed_steps(ex, a.steps)  # timing-free completion events
tr = json.loads(ex.run())  # one traced step for the stats
outs = {o: ex.get_output(o, g.tensors[o].nbytes) for o in g.outputs()}
stt = ex.stats()
t0 = time.perf_counter()
want = oracle_outputs(g, mg, inp)
cpu_s = time.perf_counter() - t0
err = max(rel_err(out_values(g, o, outs[o]), out_values(g, o, want[o])) for o in g.outputs())
flops = 2.0 * a.n ** 3 * a.chain
print(json.dumps({"workload": f"matmul_chain_{a.n}_tile{a.tile}_L{a.chain}_2dev_cap{a.cap_floor}xfloor",
                  "plan": st, "caps": caps, "gpu_step_s": [round(x, 5) for x in ts], "gpu_tflops": round(flops / min(ts) / 1e12, 1),
                  "cpu_oracle_s": round(cpu_s, 2), "cpu_cores": os.cpu_count(), "speedup_vs_cpu": round(cpu_s / min(ts), 1),
                  "tf32_rel_err_vs_fp32_oracle": err, "h2d_bytes": stt["h2d_bytes"], "d2h_bytes": stt["d2h_bytes"],
                  "d2d_or_p2p_bytes": stt["d2d_bytes"] + stt["p2p_bytes"],
                  "exposed_transfer_s": round(stt["exposed_transfer_s"], 5)}))
