"""Virtual-time dispatcher parity with the reference simulator
(proj/tests/test_simulator.cpp restated through the memplan-compatible API)."""
import json

from corpus import taskgraph
from paper_2405_16283_b200 import memplan


def chain(n):
    vs = [{"id": 0, "kind": "input", "device": 0}] + [{"id": i, "kind": "kernel", "device": 0} for i in range(1, n + 1)]
    return json.dumps({"device_count": 1, "vertices": vs, "edges": [[i - 1, i] for i in range(1, n + 1)]})


def invariants(mg, trace):
    m, t = json.loads(mg), json.loads(trace)
    row = {r["vertex"]: r for r in t["rows"]}
    assert len(row) == len(m["vertices"])
    for e in m["edges"]:
        assert row[e["from"]]["end"] <= row[e["to"]]["start"] + 1e-9
    rows = t["rows"]
    for i in range(len(rows)):
        for j in range(i + 1, len(rows)):
            a, b = rows[i], rows[j]
            if a["device"] != b["device"] or a["stream"] != b["stream"] or a["stream"] < 0:
                continue
            assert not (a["start"] < b["end"] - 1e-9 and b["start"] < a["end"] - 1e-9)


def test_chain_makespan():
    mg, _ = memplan.build_memgraph(chain(3), [4])
    t = memplan.simulate(mg)
    assert json.loads(t)["makespan"] == 3.0
    invariants(mg, t)


def test_overlap_on_two_devices():
    def build(devs):
        second = 1 if devs > 1 else 0
        g = json.dumps({"device_count": devs, "vertices": [
            {"id": 0, "kind": "input", "device": 0}, {"id": 1, "kind": "kernel", "device": 0},
            {"id": 2, "kind": "input", "device": second}, {"id": 3, "kind": "kernel", "device": second}],
            "edges": [[0, 1], [2, 3]]})
        return memplan.build_memgraph(g, [4] * devs)[0]

    assert json.loads(memplan.simulate(build(1)))["makespan"] == 2.0
    assert json.loads(memplan.simulate(build(2)))["makespan"] == 1.0


def test_fixed_order_never_faster_without_noise():
    for seed in range(12):
        g = taskgraph("gen_random_dag", [14, 0.3, 2, seed])
        try:
            mg, _ = memplan.build_memgraph(g, [6, 6])
        except memplan.MemplanError:
            continue
        e = json.loads(memplan.simulate(mg, seed=seed))["makespan"]
        f = json.loads(memplan.simulate(mg, policy="fixed-order", seed=seed))["makespan"]
        assert e <= f + 1e-9


def test_compare_policies_chain_zero():
    mg, _ = memplan.build_memgraph(chain(4), [5])
    s = json.loads(memplan.compare_policies(mg, trials=10, seed=7))
    assert s["speedup"]["mean"] == 0.0 and s["trials"] == 10


def test_fixed_order_chains_each_device():
    mg, _ = memplan.build_memgraph(taskgraph("gen_matmul", [1]), [4])
    fixed = json.loads(memplan.make_fixed_order(mg))
    m = json.loads(mg)
    op = {v["id"]: v["op"] for v in m["vertices"]}
    ops = [i for i in m["total_order"] if op[i] != "input"]
    edges = {(e["from"], e["to"]) for e in fixed["edges"]}
    assert all((a, b) in edges for a, b in zip(ops, ops[1:]))


def test_noisy_traces_deterministic_and_csv():
    g = taskgraph("gen_layered", [2, 2, 2, 3])
    mg, _ = memplan.build_memgraph(g, [6, 6])
    prof = json.dumps({"noise": {"kind": "uniform", "param": 0.2}})
    a = memplan.simulate(mg, prof, tie_break="seeded-random", seed=99)
    assert a == memplan.simulate(mg, prof, tie_break="seeded-random", seed=99)
    csv = memplan.simulate(mg, prof, tie_break="seeded-random", seed=99, format="csv")
    assert csv.splitlines()[0] == "vertex,start,end,device,stream"
    invariants(mg, a)


def test_deadlock_and_bad_profile_raise():
    import pytest
    mg, _ = memplan.build_memgraph(chain(2), [4])
    with pytest.raises(memplan.MemplanError):
        memplan.simulate(mg, json.dumps({"streams_per_device": 0}))
    with pytest.raises(memplan.MemplanError):
        memplan.simulate(mg, policy="nope")


def test_plan_order_tie_break():
    """"plan-order" (an extension): ready vertices go in the memgraph's total
    order, not in the order they became ready. One stream; kernel 2 is ready
    at t=0 but planned last, kernel 3 becomes ready at t=1 (after kernel 1)."""
    vs = [{"id": 0, "kind": "input", "device": 0}] + [{"id": i, "kind": "kernel", "device": 0} for i in range(1, 4)]
    g = json.dumps({"device_count": 1, "vertices": vs, "edges": [[0, 1], [0, 2], [1, 3]]})
    mg, _ = memplan.build_memgraph(g, [8], order=[0, 1, 3, 2])
    prof = json.dumps({"streams_per_device": 1})

    def ran(tb):
        t = json.loads(memplan.simulate(mg, prof, tie_break=tb))
        invariants(mg, json.dumps(t))
        return [r["vertex"] for r in sorted(t["rows"], key=lambda r: r["start"]) if r["vertex"] != 0]

    assert ran("plan-order") == [1, 3, 2]
    assert ran("fifo") == [1, 2, 3]
    for seed in range(6):
        g = taskgraph("gen_random_dag", [14, 0.3, 2, seed])
        try:
            mg, _ = memplan.build_memgraph(g, [6, 6])
        except memplan.MemplanError:
            continue
        invariants(mg, memplan.simulate(mg, tie_break="plan-order"))
