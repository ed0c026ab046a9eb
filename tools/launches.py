"""Summarises an ncu --metrics gpu__time_duration.sum launch list (CSV).

    python tools/launches.py launches.csv [--last N] [--dump out.csv]
--last N keeps only the last N tn:: launches (e.g. one step), --first I --count N
a window (bench.py runs value steps, then arena-copy steps, then e2e steps); --dump writes
those rows (tn:: kernels only) as a compact CSV for profiles/."""
import argparse, collections, csv, re

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--last", type=int, default=0)
ap.add_argument("--first", type=int, default=-1, help="start index (tn:: launches) of the window, instead of --last")
ap.add_argument("--count", type=int, default=0)
ap.add_argument("--dump", default=None)
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        hdr, start = r, i + 1
        break
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
ours = [r for r in rows[start:] if len(r) > vi and r[ki].startswith(("tn::", "void tn::"))]
if a.first >= 0:
    ours = ours[a.first:a.first + a.count]
elif a.last:
    ours = ours[-a.last:]  # torch kernels of the input generator run before the step
if a.dump:
    with open(a.dump, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(hdr)
        w.writerows(ours)
agg = collections.defaultdict(lambda: [0, 0.0])
for r in ours:
    name = re.sub(r"\(anonymous namespace\)::", "", r[ki].replace("void ", ""))
    name = re.sub(r"\(.*$", "", name)
    v = float(r[vi].replace(",", ""))
    v = {"ns": v / 1e3, "nsecond": v / 1e3, "ms": v * 1e3, "msecond": v * 1e3}.get(r[ui], v)  # -> microseconds
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(x[1] for x in agg.values())
print(f"{'kernel':45s} {'launches':>8s} {'total ms':>9s} {'share':>6s} {'avg us':>9s}")
for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:45s} {n:8d} {us / 1e3:9.2f} {100 * us / tot:5.1f}% {us / n:9.1f}")
print(f"{'total':45s} {sum(x[0] for x in agg.values()):8d} {tot / 1e3:9.2f}")
