"""Config 1: tiled fp32 matmul chain (4096², tile 1024, L=4) partitioned over
2 memgraph devices with a cap forcing offload/reload, executed on the GPU
(tcgen05 tiles, fixed-order k-combines, transfers) at both GEMM precisions —
3xTF32 (fp32-accurate, the default) and plain tf32 — and on the CPU oracle
executor (the reference configuration "on the CPU reference executor").
Reports step times, the GEMM-only rate of each precision (kernel device time
of the gemm vertices in a traced step) and the error vs the fp32 oracle.

Step roofline: max(FLOP / GEMM rate, H2D / PCIe, D2H / PCIe) — the step is
PCIe-bound (inputs and reloads over the host link)."""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
from helpers import inputs_of, oracle_outputs, out_values, rel_err
from paper_2405_16283_b200 import workloads as W
from paper_2405_16283_b200.executor import Executor
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--tile", type=int, default=1024)
ap.add_argument("--chain", type=int, default=4)
ap.add_argument("--cap-floor", type=float, default=1.5,
                help="per-device cap as a multiple of the working-set floor (1.5 -> 128 offloads)")
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
ngpu = torch.cuda.device_count()
flops = 2.0 * a.n ** 3 * a.chain
res = {"workload": f"matmul_chain_{a.n}_tile{a.tile}_L{a.chain}_2dev_cap{a.cap_floor}xfloor", "gpus": ngpu,
       "flops": flops}
want = None
for prec in ("3xtf32", "tf32"):
    g = W.matmul_chain(a.n, a.tile, a.chain, devices=2, precision=prec)
    floor = W.working_set_floor(g)
    caps = [int(f * a.cap_floor) // 1024 * 1024 for f in floor]
    mg, st = W.plan(g, caps, alloc_horizon="lazy")
    inp = inputs_of(g, seed=0)
    with Executor(mg, g.to_json(), {"devices": [0, 1 % ngpu]}) as ex:
        for k, v in inp.items():
            ex.set_input(k, v)
        ts = bench.untimed_steps(ex, a.steps)
        tr = json.loads(ex.run())
        outs = {o: ex.get_output(o, g.tensors[o].nbytes) for o in g.outputs()}
        stt = ex.stats()
    ids = {v["id"]: v for v in g.vertices}
    gemm_s = sum(r["end"] - r["start"] for r in tr["rows"]
                 if r["vertex"] in ids and (ids[r["vertex"]].get("op") or {}).get("type") == "gemm")
    if want is None:
        t0 = time.perf_counter()
        want = oracle_outputs(g, mg, inp)
        res["cpu_oracle_s"] = round(time.perf_counter() - t0, 2)
        res["cpu_cores"] = os.cpu_count()
        res["plan"] = st
    err = max(rel_err(out_values(g, o, outs[o]), out_values(g, o, want[o])) for o in g.outputs())
    pcie = bench.measure_pcie(torch.device("cuda", 0))
    roof = max(stt["h2d_bytes"], stt["d2h_bytes"]) / (pcie * 1e9)
    res[prec] = {"gpu_step_s": [round(x, 5) for x in ts], "gemm_device_s_per_step": round(gemm_s, 5),
                 "gemm_tflops": round(flops / gemm_s / 1e12, 1), "rel_err_vs_fp32_oracle": err,
                 "h2d_bytes": stt["h2d_bytes"], "d2h_bytes": stt["d2h_bytes"],
                 "d2d_or_p2p_bytes": stt["d2d_bytes"] + stt["p2p_bytes"],
                 "exposed_transfer_s": round(stt["exposed_transfer_s"], 5), "pcie_bound_s": round(roof, 5),
                 "frac_of_pcie_roofline": round(roof / min(ts), 4),
                 "speedup_vs_cpu_oracle": round(res["cpu_oracle_s"] / min(ts), 1)}
print(json.dumps(res))
