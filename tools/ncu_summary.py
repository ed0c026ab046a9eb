"""Summarises an `ncu --set full` report (.ncu-rep) per launch: duration,
clock, DRAM bytes, L2 sector traffic, tensor-pipe utilisation, issue activity.

    python tools/ncu_summary.py REPORT.ncu-rep [--labels a,b,c] [--json out.json]

The JSON is what bench.py reads for roofline.traffic (profiles/)."""
import argparse
import csv
import io
import json
import subprocess

M = {
    "us": "gpu__time_duration.sum",
    "sm_ghz": "sm__cycles_elapsed.avg.per_second",
    "dram_read_mb": "dram__bytes_read.sum",
    "dram_write_mb": "dram__bytes_write.sum",
    "l2_sectors": "lts__t_sectors.sum",
    "l2_sectors_per_slice_cycle": "lts__t_sectors.avg.per_cycle_elapsed",
    "tensor_bf16_pct_of_peak": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "dram_pct_of_peak": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
}


def rows(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    r = list(csv.reader(io.StringIO(out.stdout)))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")].split("(")[0].replace("(anonymous namespace)::", "")}
        for k, m in M.items():
            if m not in hdr:
                continue
            v = row[hdr.index(m)].replace(",", "")
            u = units[hdr.index(m)]
            try:
                x = float(v)
            except ValueError:
                continue
            if k.endswith("_mb"):
                x *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
            if k == "us":
                x *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
            d[k] = round(x, 3)
        if "dram_read_mb" in d and "dram_write_mb" in d:
            d["dram_bytes"] = int(round((d["dram_read_mb"] + d["dram_write_mb"]) * 1e6))
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--labels", default="")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    rs = rows(a.report)
    labels = a.labels.split(",") if a.labels else []
    for i, r in enumerate(rs):
        if i < len(labels):
            r["label"] = labels[i]
        print(json.dumps(r))
    if a.json:
        json.dump({"report": a.report.split("/")[-1], "launches": rs}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
