"""Pinned H2D / D2H bandwidth with 1, 2 and 4 concurrent copy streams (1 GiB
total per direction, best of 5), to see whether splitting a large transfer
across copy engines beats one cudaMemcpyAsync."""
import json
import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
hd = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
res = {}
for direction in ("h2d", "d2h", "duplex"):
    for k in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(k)]
        best = 0.0
        for _ in range(5):
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for i, st in enumerate(streams):
                st.wait_event(s)
                with torch.cuda.stream(st):
                    sl = slice(i * n // k, (i + 1) * n // k)
                    if direction in ("h2d", "duplex"):
                        d[sl].copy_(h[sl], non_blocking=True)
                    if direction in ("d2h", "duplex"):
                        hd[sl].copy_(d2[sl], non_blocking=True)
            for st in streams:
                e.wait(st) if hasattr(e, "wait") else None
                torch.cuda.current_stream().wait_stream(st)
            e.record()
            e.synchronize()
            gb = n * (2 if direction == "duplex" else 1) / 1e9
            best = max(best, gb / (s.elapsed_time(e) * 1e-3))
        res[f"{direction}_x{k}"] = round(best, 1)
print(json.dumps(res))
