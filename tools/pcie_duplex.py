"""PCIe H2D / D2H / concurrent-duplex bandwidth of this GPU (pinned, 1 GiB)."""
import json, torch
n = 1 << 30
h1 = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(fn):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); 
    for s in (s1, s2): torch.cuda.current_stream().wait_stream(s)
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) * 1e-3
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
res = {}
for name, fn, byts in (("h2d", h2d, n), ("d2h", d2h, n), ("duplex", both, 2 * n)):
    best = min(timed(fn) for _ in range(4))
    res[name + "_gbs"] = round(byts / best / 1e9, 1)
print(json.dumps(res))
