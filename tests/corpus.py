"""Deterministic planner corpus shared by the golden generator and the tests.

Follows the reference acceptance corpus recipe (proj/tests/acceptance_main.cpp:107-164:
random DAGs / layered / blocked matmul, a capacity ladder from plenty to the
working-set floor) and additionally sweeps order policy, victim policy,
horizon, memory mode and keep_superfluous, with capacities below the floor
to pin the reference's error behaviour too.
"""
import json

OP = ["as-listed", "depth-first", "min-memory-greedy"]
VP = ["farthest-next-use", "last-allocated", "seeded-random"]


def _floor(gj, mode):
    D = gj["device_count"]
    unit = (lambda v: 1) if mode == "slot" else (lambda v: v.get("output_size", 1))
    byid = {v["id"]: v for v in gj["vertices"]}
    cons = {v["id"]: 0 for v in gj["vertices"]}
    prods = {v["id"]: [] for v in gj["vertices"]}
    for p, c in gj["edges"]:
        cons[p] += 1
        prods[c].append(p)
    outs, fl = [0] * D, [0] * D
    for v in gj["vertices"]:
        if cons[v["id"]] == 0:
            outs[v["device"]] += unit(v)
        ws = unit(v) + sum(unit(byid[p]) for p in prods[v["id"]] if byid[p]["device"] == v["device"])
        fl[v["device"]] = max(fl[v["device"]], ws)
    res = []
    for d in range(D):
        f = fl[d] + outs[d]
        if mode == "byte":
            f = f * 3 // 2 + 4
        res.append(max(f, 1))
    return res


def _total(gj, mode):
    t = [0] * gj["device_count"]
    for v in gj["vertices"]:
        t[v["device"]] += 1 if mode == "slot" else v.get("output_size", 1)
    return [max(x, 1) for x in t]


def gen_args(seed):
    k = seed % 3
    if k == 0:
        return "gen_random_dag", [8 + seed % 29, 0.25 + 0.1 * (seed % 4), 1 + seed % 3, seed]
    if k == 1:
        return "gen_layered", [1 + seed % 4, 1 + seed % 3, 1 + seed % 3, seed]
    return "gen_matmul", [1 + seed % 5]


_GRAPHS = None


def taskgraph(name, args):
    """A toy taskgraph emitted by the reference generator `name(*args)`
    (tests/golden/taskgraphs.json, written by make_taskgraphs.py from oracle/_ref)."""
    global _GRAPHS
    if _GRAPHS is None:
        import os
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "taskgraphs.json")) as f:
            _GRAPHS = json.load(f)["graphs"]
    return _GRAPHS[f"{name}{json.dumps(list(args))}"]


def corpus_cases(n_seeds=90):
    """Yields build cases over the reference-generated toy taskgraphs."""
    for seed in range(n_seeds):
        name, args = gen_args(seed)
        gj = json.loads(taskgraph(name, args))
        for mode in ("slot", "byte"):
            fl, tot = _floor(gj, mode), _total(gj, mode)
            for rung in range(4):
                caps = [tot[d] if rung == 0 else (fl[d] + tot[d]) // 2 if rung == 1 else fl[d] if rung == 2
                        else max(1, fl[d] * 2 // 3) for d in range(len(fl))]
                kw = dict(mode=mode, order_policy=OP[(seed + rung) % 3],
                          victim_policy=VP[(seed + rung + (mode == "byte")) % 3], seed=seed,
                          alloc_horizon="lazy" if (seed + rung) % 4 == 0 else "greedy",
                          keep_superfluous=(seed + rung) % 5 != 0)
                case = {"gen": name, "gen_args": args, "caps": caps, "kw": kw}
                if rung in (1, 2) and seed % 2 == 0:
                    case["simulate"] = [
                        ["event-driven", "fifo", ""],
                        ["fixed-order", "lowest-id", ""],
                        ["event-driven", "seeded-random",
                         json.dumps({"noise": {"kind": "lognormal", "param": 0.3}, "host_link_bandwidth": 2.0,
                                     "streams_per_device": 1 + seed % 5})],
                    ]
                yield case
