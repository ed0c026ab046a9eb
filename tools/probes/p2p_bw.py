"""Link bandwidths the multi-GPU step roofline is built from:

  * peer copy GPU a -> GPU b (the executor's Transfer vertices are
    cudaMemcpyPeerAsync), every ordered pair, one at a time;
  * all pairs of a ring concurrently (every GPU sends to its neighbour,
    the pattern of a TP reduce-scatter step) — per-GPU GB/s;
  * pinned host -> device on every GPU at once (the e2e step streams each
    GPU's weight shard over its own PCIe link) — per-GPU and aggregate GB/s.

    python tools/probes/p2p_bw.py [--mib 1024] [--reps 3]
Prints one JSON line. With one visible GPU only the H2D figures are
reported."""
import argparse
import json

import torch


def timed(fn, devs):
    for d in devs:
        torch.cuda.synchronize(d)
    starts = {d: torch.cuda.Event(enable_timing=True) for d in devs}
    ends = {d: torch.cuda.Event(enable_timing=True) for d in devs}
    for d in devs:
        with torch.cuda.device(d):
            starts[d].record()
    fn()
    for d in devs:
        with torch.cuda.device(d):
            ends[d].record()
    for d in devs:
        torch.cuda.synchronize(d)
    return max(starts[d].elapsed_time(ends[d]) for d in devs) * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    n = a.mib << 20
    G = torch.cuda.device_count()
    devs = list(range(G))
    src = {d: torch.empty(n, dtype=torch.uint8, device=f"cuda:{d}") for d in devs}
    dst = {d: torch.empty(n, dtype=torch.uint8, device=f"cuda:{d}") for d in devs}
    host = {d: torch.empty(n, dtype=torch.uint8, pin_memory=True) for d in devs}
    out = {"gpus": G, "bytes": n, "peer_access": {}, "p2p_gbs": {}}
    for a_ in devs:
        for b in devs:
            if a_ != b:
                out["peer_access"][f"{a_}->{b}"] = torch.cuda.can_device_access_peer(a_, b)

    def best(fn, ds, bytes_moved):
        return round(max(bytes_moved / timed(fn, ds) / 1e9 for _ in range(a.reps)), 1)

    for a_ in devs:
        for b in devs:
            if a_ == b:
                continue

            def one(a_=a_, b=b):
                with torch.cuda.device(b):
                    dst[b].copy_(src[a_], non_blocking=True)
            out["p2p_gbs"][f"{a_}->{b}"] = best(one, [a_, b], n)
    if G > 1:
        def ring():
            for d in devs:
                with torch.cuda.device((d + 1) % G):
                    dst[(d + 1) % G].copy_(src[d], non_blocking=True)
        out["ring_concurrent_gbs_per_gpu"] = round(best(ring, devs, n * G) / G, 1)

    def h2d_all():
        for d in devs:
            with torch.cuda.device(d):
                dst[d].copy_(host[d], non_blocking=True)
    agg = best(h2d_all, devs, n * G)
    out["h2d_all_gpus_concurrent_gbs"] = {"aggregate": agg, "per_gpu": round(agg / G, 1)}

    def h2d_one():
        with torch.cuda.device(0):
            dst[0].copy_(host[0], non_blocking=True)
    out["h2d_single_gpu_gbs"] = best(h2d_one, [0], n)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
