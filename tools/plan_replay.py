"""Replays a memgraph on a model of one B200 to compare generator / planner
variants on the CPU before spending GPU time: kernels serialise on one
compute engine with durations measured in a traced step (`bench_lora.py
--dump`, keyed by taskgraph tensor name), Input / Reload copies share one H2D
engine and Offloads one D2H engine at the measured PCIe rates. Ready vertices
are taken in the memgraph's total order (the executor's "plan-order" tie break; "fifo" takes them by ready time)."""
import heapq
import json


def replay(mg: dict, dur_of, h2d_gbs=55.6, d2h_gbs=57.3, host_inputs=True, tie_break="plan-order"):
    """mg: memgraph JSON dict; dur_of(vertex) -> kernel seconds; tie_break
    "plan-order" (total order) or "fifo" (ready time). Returns (makespan,
    {vertex id: (start, end)})."""
    vs = {v["id"]: v for v in mg["vertices"]}
    pos = {vid: i for i, vid in enumerate(mg["total_order"])}
    preds = {vid: 0 for vid in vs}
    succ = {vid: [] for vid in vs}
    for e in mg["edges"]:
        preds[e["to"]] += 1
        succ[e["from"]].append(e["to"])

    def engine(v):
        op = v["op"]
        if op == "input":
            return "h2d" if host_inputs else None
        if op == "reload":
            return "h2d"
        if op == "offload":
            return "d2h"
        if op in ("kernel", "compute"):
            return "sm"
        return None

    def duration(v):
        op = v["op"]
        if op == "input":
            return v["size"] / (h2d_gbs * 1e9) if host_inputs else 0.0
        if op == "reload":
            return v["size"] / (h2d_gbs * 1e9)
        if op == "offload":
            return v["size"] / (d2h_gbs * 1e9)
        if op in ("kernel", "compute"):
            return dur_of(v)
        return 0.0

    ready = {"h2d": [], "d2h": [], "sm": []}
    busy = {"h2d": False, "d2h": False, "sm": False}
    events = []  # (time, seq, vid)
    seq = 0
    t = 0.0
    span = {}

    def make_ready(vid, now):
        nonlocal seq
        eng = engine(vs[vid])
        if eng is None:
            span[vid] = (now, now)
            seq += 1
            heapq.heappush(events, (now, seq, vid))
        else:
            key = pos[vid] if tie_break == "plan-order" else seq
            seq += 1
            heapq.heappush(ready[eng], (key, vid))

    for vid in vs:
        if preds[vid] == 0:
            make_ready(vid, 0.0)

    def start_engines(now):
        nonlocal seq
        for eng, q in ready.items():
            if not busy[eng] and q:
                _, vid = heapq.heappop(q)
                d = duration(vs[vid])
                span[vid] = (now, now + d)
                busy[eng] = vid
                seq += 1
                heapq.heappush(events, (now + d, seq, vid))

    start_engines(0.0)
    while events:
        t, _, vid = heapq.heappop(events)
        eng = engine(vs[vid])
        if eng is not None and busy[eng] == vid:
            busy[eng] = False
        for s in succ[vid]:
            preds[s] -= 1
            if preds[s] == 0:
                make_ready(s, t)
        start_engines(t)
    assert len(span) == len(vs), "replay did not complete every vertex"
    return t, span


def replay_duplex(mg: dict, dur_of, h2d_gbs=55.6, d2h_gbs=57.3, duplex_gbs=99.4, host_inputs=True):
    """Like replay(), with the PCIe link shared: a copy runs at its solo rate
    while the other direction is idle and at duplex_gbs / 2 while both
    directions move data (fluid model, rates re-evaluated at every event).
    Returns the makespan."""
    vs = {v["id"]: v for v in mg["vertices"]}
    pos = {vid: i for i, vid in enumerate(mg["total_order"])}
    preds = {vid: 0 for vid in vs}
    succ = {vid: [] for vid in vs}
    for e in mg["edges"]:
        preds[e["to"]] += 1
        succ[e["from"]].append(e["to"])

    def engine(v):
        op = v["op"]
        if op in ("reload",) or (op == "input" and host_inputs):
            return "h2d"
        if op == "offload":
            return "d2h"
        if op in ("kernel", "compute"):
            return "sm"
        return None

    ready = {"h2d": [], "d2h": [], "sm": []}
    cur = {"h2d": None, "d2h": None, "sm": None}  # [vid, remaining bytes or end time]
    t, done = 0.0, 0
    instant = []

    def make_ready(vid):
        eng = engine(vs[vid])
        if eng is None:
            instant.append(vid)
        else:
            heapq.heappush(ready[eng], (pos[vid], vid))

    def finish(vid):
        nonlocal done
        done += 1
        for s in succ[vid]:
            preds[s] -= 1
            if preds[s] == 0:
                make_ready(s)

    for vid in vs:
        if preds[vid] == 0:
            make_ready(vid)
    while True:
        while instant:
            finish(instant.pop())
        for eng, q in ready.items():
            if cur[eng] is None and q:
                _, vid = heapq.heappop(q)
                cur[eng] = [vid, t + dur_of(vs[vid]) if eng == "sm" else float(vs[vid]["size"])]
        if instant:
            continue
        if all(c is None for c in cur.values()):
            break
        both = cur["h2d"] is not None and cur["d2h"] is not None
        rate = {"h2d": (duplex_gbs / 2 if both else h2d_gbs) * 1e9, "d2h": (duplex_gbs / 2 if both else d2h_gbs) * 1e9}
        cand = []
        if cur["sm"] is not None:
            cand.append(cur["sm"][1])
        for eng in ("h2d", "d2h"):
            if cur[eng] is not None:
                cand.append(t + cur[eng][1] / rate[eng])
        tn = min(cand)
        dt = tn - t
        for eng in ("h2d", "d2h"):
            if cur[eng] is not None:
                cur[eng][1] -= rate[eng] * dt
        t = tn
        for eng in ("sm", "h2d", "d2h"):
            c = cur[eng]
            if c is None:
                continue
            if (eng == "sm" and c[1] <= t + 1e-15) or (eng != "sm" and c[1] <= 1e-3):
                cur[eng] = None
                finish(c[0])
    assert done == len(vs), "replay did not complete every vertex"
    return t
