import json, sys
d = json.load(open(sys.argv[1]))
g, t = d["graph"], d["trace"]
V = {v["id"]: v for v in g["vertices"]}
rows = t["rows"]
kern = sorted([r for r in rows if V.get(r["vertex"], {}).get("kind") == "kernel"], key=lambda r: r["start"])
gaps = [b["start"] - a["end"] for a, b in zip(kern, kern[1:])]
import statistics as S
print("kernels", len(kern), "sum dur %.4f" % sum(r["end"]-r["start"] for r in kern), "sum gaps %.4f" % sum(max(0,x) for x in gaps),
      "median gap %.1f us" % (S.median(gaps)*1e6), "p90 %.1f us" % (sorted(gaps)[int(.9*len(gaps))]*1e6))
# for big gaps: what was the next kernel waiting for?
pred = {}
for e in g["edges"]: pass
print("makespan", t["makespan"])
ins = sorted([r for r in rows if V.get(r["vertex"], {}).get("kind") == "input"], key=lambda r: r["start"])
print("inputs", len(ins), "sum dur %.4f" % sum(r["end"]-r["start"] for r in ins), "first start %.4f last end %.4f" % (ins[0]["start"], ins[-1]["end"]))
big = sorted(zip(gaps, kern[1:]), key=lambda x: -x[0])[:8]
for gp, r in big:
    v = V[r["vertex"]]; print("gap %.1f us before %s" % (gp*1e6, v.get("op",{}).get("type")), r["vertex"])
