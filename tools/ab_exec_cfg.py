"""Paired A/B of executor configs on the 7B prefill step (same process, same
box, alternating blocks of untimed steps), e.g.

    python tools/ab_exec_cfg.py '{"lookahead": 1}' '{"lookahead": 2}' '{"lookahead": 4}'

AB_RESIDENCY=host runs the weights-cold (e2e) configuration; AB_REPS / AB_STEPS
set the number of alternating blocks and steps per block.
"""
import json
import statistics
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import torch  # noqa: E402

from paper_2405_16283_b200 import workloads as W  # noqa: E402
from paper_2405_16283_b200.executor import Executor  # noqa: E402


def main():
    cfgs = [json.loads(a) for a in sys.argv[1:]] or [{}]
    g = W.llama_prefill(W.LLAMA_7B, 4096)
    mg, _ = W.plan(g, 16 << 30)
    inputs = bench.device_inputs(g, 0, torch.device("cuda", 0))
    exs = []
    for c in cfgs:
        ex = Executor(mg, g.to_json(), {"devices": [0], "input_residency": os.environ.get("AB_RESIDENCY", "device"),
                                        **c})
        for k, v in inputs.items():
            ex.set_input(k, v)
        for _ in range(3):
            ex.run(trace=False)
        exs.append(ex)
    res = [[] for _ in cfgs]
    for rep in range(int(os.environ.get("AB_REPS", "6"))):
        order = range(len(cfgs)) if rep % 2 == 0 else reversed(range(len(cfgs)))
        for i in order:
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(int(os.environ.get("AB_STEPS", "10"))):
                exs[i].run(trace=False)
            e.record()
            torch.cuda.synchronize()
            res[i].append(s.elapsed_time(e) / int(os.environ.get("AB_STEPS", "10")))
    for c, r in zip(cfgs, res):
        print(json.dumps({"cfg": c, "median_ms": round(statistics.median(r), 3), "all": [round(x, 2) for x in r]}))


if __name__ == "__main__":
    main()
