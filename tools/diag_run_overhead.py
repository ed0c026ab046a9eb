import json, sys, time, statistics
sys.path.insert(0, '/root/repo')
import bench, torch
from paper_2405_16283_b200 import workloads as W
from paper_2405_16283_b200.executor import Executor
g = W.llama_prefill(W.LLAMA_7B, 4096)
mg, _ = W.plan(g, 16 << 30)
inputs = bench.device_inputs(g, 0, torch.device("cuda", 0))
for cfg in ({"input_residency": "device"}, {"input_residency": "device", "pdl": False}, {"input_residency": "device", "timestamps": "all"}):
    ex = Executor(mg, g.to_json(), {"devices": [0], **cfg})
    for k, v in inputs.items():
        ex.set_input(k, v)
    for _ in range(3):
        ex.run(trace=False)
    for trace in (False, True):
        ev = []
        ms = []
        walls = []
        for _ in range(8):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            s.record()
            r = ex.run(trace=trace)
            e.record()
            torch.cuda.synchronize()
            walls.append((time.perf_counter() - t0) * 1e3)
            ev.append(s.elapsed_time(e))
            if trace:
                ms.append(json.loads(r)["makespan"] * 1e3)
        st = ex.stats()
        print(json.dumps({"cfg": cfg, "trace": trace, "event_ms": round(statistics.median(ev), 2),
                          "host_wall_ms": round(statistics.median(walls), 2), "stats_wall_ms": round(st["wall_s"] * 1e3, 2),
                          "makespan_ms": round(statistics.median(ms), 2) if ms else None}))
    ex.close()
