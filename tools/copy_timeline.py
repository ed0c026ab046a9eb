"""Copy-link timeline of a traced executor step (bench_longctx.py --dump):
busy time per direction (union of offload / reload+input intervals), time
both directions are busy, and the gaps in each direction."""
import json
import sys


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def total(iv):
    return sum(b - a for a, b in iv)


def inter(x, y):
    i = j = 0
    s = 0.0
    while i < len(x) and j < len(y):
        a, b = max(x[i][0], y[j][0]), min(x[i][1], y[j][1])
        if a < b:
            s += b - a
        if x[i][1] < y[j][1]:
            i += 1
        else:
            j += 1
    return s


d = json.load(open(sys.argv[1]))
m, t = d["memgraph"], d["trace"]
op = {v["id"]: v["op"] for v in m["vertices"]}
rows = t["rows"]
d2h = union([[r["start"], r["end"]] for r in rows if op[r["vertex"]] == "offload" and r["end"] > r["start"]])
h2d = union([[r["start"], r["end"]] for r in rows if op[r["vertex"]] in ("reload", "input") and r["end"] > r["start"]])
ker = union([[r["start"], r["end"]] for r in rows if op[r["vertex"]] == "kernel" and r["end"] > r["start"]])
mk = t["makespan"]
print(json.dumps({"makespan": mk, "d2h_busy": total(d2h), "h2d_busy": total(h2d), "both_busy": inter(d2h, h2d),
                  "kernel_busy": total(ker), "d2h_intervals": len(d2h), "h2d_intervals": len(h2d),
                  "neither_busy": mk - total(union(d2h + h2d))}))
# gap histogram per direction
for name, iv in (("d2h", d2h), ("h2d", h2d)):
    gaps = sorted(b[0] - a[1] for a, b in zip(iv, iv[1:]))
    if gaps:
        print(name, "gaps: n", len(gaps), "sum %.4f" % sum(gaps), "median %.1f us" % (gaps[len(gaps) // 2] * 1e6),
              "p90 %.1f us" % (gaps[int(0.9 * len(gaps))] * 1e6), "max %.1f us" % (gaps[-1] * 1e6))
