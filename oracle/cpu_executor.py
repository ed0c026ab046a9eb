"""CPU oracle executor for memgraphs (numpy, fp32 op math).

TEST INFRASTRUCTURE ONLY — the checker, never the product: only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg may import this.

Restates the reference's model of a correct execution,
`TokenMachine::run` (/root/reference/proj/src/verifier.cpp:316-349), with real
bytes instead of tokens: per memgraph device a byte arena of exactly
`capacities[d]` bytes; walking any linear extension of the memgraph, every
vertex writes its placement (inputs: their host bytes; kernels: their op,
oracle/ops_ref.py; transfers: a copy of the single data predecessor,
taskgraph.cpp:159-175; reloads: the host slot of the evicted root) and every
offload copies its data predecessor's region to the host slot of its root
(compiler.cpp:334-359, :430-441). A placement bug shows up as a wrong number,
and a result that changes with the schedule is a race.

Memgraph construction parity is pinned separately (oracle/_ref = the
unmodified reference build, tests/golden/); tensor values are "parity
unpinned" because the reference has no tensor math.
"""
from __future__ import annotations

import json
import random
from dataclasses import dataclass

import numpy as np

from . import ops_ref


@dataclass
class _V:
    id: int
    op: str
    device: int
    ref: int
    size: int


def linear_extension(memgraph: dict, kind: str = "total_order", seed: int = 0) -> list[int]:
    """A schedule: the build's total order, or a seeded random / max-id-first
    linear extension (like verifier.cpp:431-447's sampled schedules)."""
    if kind == "total_order":
        return list(memgraph["total_order"])
    ids = [v["id"] for v in memgraph["vertices"]]
    indeg = {i: 0 for i in ids}
    succ: dict[int, list[int]] = {i: [] for i in ids}
    for e in memgraph["edges"]:
        indeg[e["to"]] += 1
        succ[e["from"]].append(e["to"])
    ready = sorted(i for i in ids if indeg[i] == 0)
    rng = random.Random(seed)
    out = []
    while ready:
        if kind == "random":
            k = rng.randrange(len(ready))
        elif kind == "max_id":
            k = max(range(len(ready)), key=lambda j: ready[j])
        else:
            raise ValueError(kind)
        u = ready.pop(k)
        out.append(u)
        for w in succ[u]:
            indeg[w] -= 1
            if indeg[w] == 0:
                ready.append(w)
    if len(out) != len(ids):
        raise ValueError("memgraph has a cycle")
    return out


class CpuExecutor:
    def __init__(self, memgraph_json: str, taskgraph_json: str):
        self.mg = json.loads(memgraph_json)
        tg = json.loads(taskgraph_json)
        if self.mg.get("mode") != "byte":
            raise ValueError("the oracle executes byte-mode memgraphs")
        self.ops = {v["id"]: v["op"] for v in tg["vertices"] if v.get("op")}
        self.verts = {
            v["id"]: _V(v["id"], v["op"], v["device"], v["origin"]["ref"], v["size"]) for v in self.mg["vertices"]
        }
        self.place = {int(k): (p["device"], p["offset"], p["size"]) for k, p in self.mg["placement"].items()}
        self.data_in: dict[int, list[int]] = {}
        for e in self.mg["edges"]:
            if e["kind"] == "data":
                self.data_in.setdefault(e["to"], []).append(e["from"])
        self.caps = self.mg["capacities"]
        self.inputs: dict[int, np.ndarray] = {}

    def set_input(self, vid: int, data) -> None:
        self.inputs[vid] = np.frombuffer(bytes(data) if not isinstance(data, np.ndarray) else data.tobytes(),
                                         dtype=np.uint8)

    def region(self, arenas, mid):
        d, off, sz = self.place[mid]
        return arenas[d][off:off + sz]

    def run(self, schedule: list[int] | None = None, outputs: list[int] | None = None,
            record_reads: bool = False) -> dict[int, bytes]:
        """Executes `schedule` (default: the build's total order). With
        `record_reads`, self.reads[(reader, producer)] = digest of the bytes the
        reader found in the producer's region when it ran: the byte-level
        counterpart of TokenMachine's "reads region of P but finds ..."
        check (verifier.cpp:316-349)."""
        import hashlib

        arenas = [np.zeros(c, dtype=np.uint8) for c in self.caps]
        host: dict[int, np.ndarray] = {}
        self.reads = {}
        for vid in schedule or self.mg["total_order"]:
            if record_reads:
                for src in self.data_in.get(vid, []):
                    if src in self.place:
                        self.reads[(vid, src)] = hashlib.sha1(self.region(arenas, src).tobytes()).hexdigest()
            v = self.verts[vid]
            if v.op == "input":
                r = self.region(arenas, vid)
                src = self.inputs.get(v.ref)
                if src is None:
                    raise KeyError(f"input {v.ref} not set")
                n = min(r.size, src.size)
                r[:n] = src[:n]
            elif v.op == "offload":
                (src,) = self.data_in[vid]
                host[v.ref] = self.region(arenas, src).copy()
            elif v.op == "reload":
                r = self.region(arenas, vid)
                h = host[v.ref]
                r[: min(r.size, h.size)] = h[: r.size]
            elif v.op == "transfer":
                (src,) = self.data_in[vid]
                s, r = self.region(arenas, src), self.region(arenas, vid)
                n = min(s.size, r.size)
                r[:n] = s[:n]
            else:
                op = self.ops[v.ref]
                srcs = {self.verts[s].ref: s for s in self.data_in.get(vid, [])}
                args = [self.region(arenas, srcs[a]) for a in op["args"]]
                ops_ref.OPS[op["type"]](op, args, self.region(arenas, vid))
        res = {}
        for o in outputs or []:
            res[o] = self.region(arenas, o).tobytes()
        return res
