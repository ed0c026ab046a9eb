"""Per-GEMM-class device time / TFLOP/s of one traced 7B step (trace_*.json)."""
import collections, json, sys
d = json.load(open(sys.argv[1]))
V = {v["id"]: v for v in d["graph"]["vertices"]}
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in d["trace"]["rows"]:
    v = V.get(r["vertex"])
    if not v or v["kind"] != "kernel":
        continue
    op = v["op"]
    name = op["type"] + ("/" + op["epilogue"] if op.get("epilogue") else "")
    if op["type"] == "gemm":
        f = 2 * op["M"] * op["N"] * op["K"] * op.get("batch", 1) * (0.5 if op.get("causal") else 1)
        name += f" {op['M']}x{op['N']}x{op['K']}"
    elif op["type"] == "attention":
        f = 4.0 * op["heads"] * op["seq"] ** 2 * op["hd"] * 0.5
    else:
        f = 0
    a = agg[name]
    a[0] += 1
    a[1] += r["end"] - r["start"]
    a[2] += f
tot = sum(a[1] for a in agg.values())
for k, (n, t, f) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:40s} n={n:3d} {t * 1e3:8.2f} ms {100 * t / tot:5.1f}%  avg {t / n * 1e6:8.1f} us" +
          (f"  {f / t / 1e12:7.1f} TF/s" if f else ""))
print("makespan %.2f ms, kernel sum %.2f ms" % (d["trace"]["makespan"] * 1e3, tot * 1e3))
