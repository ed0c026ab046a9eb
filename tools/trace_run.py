"""Runs the config-2 memgraph once (inputs resident) and dumps graph + trace
for offline analysis (gpurun_out/trace_*.json)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import torch  # noqa: E402

from paper_2405_16283_b200 import workloads as W  # noqa: E402
from paper_2405_16283_b200.executor import Executor  # noqa: E402


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--residency", default="device")
    ap.add_argument("--cfg", default="{}")
    ap.add_argument("--tag", default="a")
    ap.add_argument("--runs", type=int, default=3)
    ap.add_argument("--longctx", default="", help="seq,heads,tile,lag,cap_gib for a config-5 graph")
    a = ap.parse_args()
    if a.longctx:
        seq, heads, tile, lag, cap = (float(x) for x in a.longctx.split(","))
        g = W.blockwise_attention(int(seq), int(heads), 128, int(tile), lag=int(lag))
        mg, st = W.plan(g, int(cap * (1 << 30)), alloc_horizon="lazy")
    else:
        g = W.llama_prefill(W.LLAMA_7B, 4096)
        mg, st = W.plan(g, 16 << 30)
    inputs = bench.device_inputs(g, 0, torch.device("cuda", 0))
    cfg = {"devices": [0], "input_residency": a.residency, **json.loads(a.cfg)}
    ex = Executor(mg, g.to_json(), cfg)
    for k, v in inputs.items():
        ex.set_input(k, v)
    for _ in range(a.runs):
        tr = ex.run()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump({"graph": json.loads(g.to_json()), "trace": json.loads(tr), "stats": ex.stats(), "cfg": cfg, "memgraph": json.loads(mg)},
              open(f"gpurun_out/trace_{a.tag}.json", "w"))
    print(json.dumps(ex.stats()))


if __name__ == "__main__":
    main()
