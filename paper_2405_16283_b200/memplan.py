"""Drop-in mirror of the reference `memplan` Python API
(proj/python/memplan/__init__.py, proj/python/bindings.cpp:36-124).

Same function names, argument names/defaults, JSON-string formats and error
type (`MemplanError`), served by libturnip_b200.so through the C ABI in
include/turnip.h. `build_memgraph` is byte-identical to the reference;
`simulate`/`compare_policies` are the virtual-time dispatcher (byte-identical
traces); `execute` is the new real-hardware path (see executor.py).
"""
from __future__ import annotations

import json

from ._lib import MemplanError, call, enc, i64_array

__all__ = [
    "MemplanError",
    "build_memgraph",
    "compare_policies",
    "make_fixed_order",
    "memgraph_to_dot",
    "simulate",
    "taskgraph_to_dot",
    "topological_order",
    "validate_taskgraph",
    "verify",
    "check_capacity",
]


def validate_taskgraph(graph_json: str) -> list[str]:
    """bindings.cpp:39-45."""
    return json.loads(call("tn_validate_taskgraph", enc(graph_json)))


def topological_order(graph_json: str, policy: str = "as-listed", seed: int = 0) -> list[int]:
    """bindings.cpp:47-51."""
    return json.loads(call("tn_topological_order", enc(graph_json), enc(policy), seed))


def build_memgraph(
    graph_json: str,
    capacities,
    mode: str = "slot",
    order=(),
    order_policy: str = "as-listed",
    victim_policy: str = "farthest-next-use",
    seed: int = 0,
    alloc_horizon: str = "greedy",
    keep_superfluous: bool = True,
    host_capacity: int | None = None,
):
    """bindings.cpp:61-85: returns (memgraph_json, stats dict).

    `host_capacity` exposes BuildOptions::host_capacity (compiler.hpp:37),
    which the reference keeps C++-only."""
    caps, ncaps = i64_array(capacities)
    order_arr, norder = i64_array(order)
    mg, stats = call(
        "tn_build_memgraph",
        enc(graph_json),
        caps,
        ncaps,
        enc(mode),
        order_arr,
        norder,
        enc(order_policy),
        enc(victim_policy),
        seed,
        enc(alloc_horizon),
        1 if keep_superfluous else 0,
        -1 if host_capacity is None else int(host_capacity),
        nout=2,
    )
    return mg, json.loads(stats)


def verify(graph_json: str, memgraph_json: str, schedule_limit: int = 0) -> str:
    """bindings.cpp:87-93: every verifier check; returns the report as JSON."""
    return call("tn_verify", enc(graph_json), enc(memgraph_json), int(schedule_limit))


def check_capacity(memgraph_json: str, order) -> dict:
    """verifier.hpp:47-48 (C++-only in the reference): replays `order`."""
    arr, n = i64_array(order)
    return json.loads(call("tn_check_capacity", enc(memgraph_json), arr, n))


def simulate(memgraph_json: str, profile_json: str = "", policy: str = "event-driven",
             tie_break: str = "fifo", seed: int = 0, format: str = "json") -> str:
    """bindings.cpp:95-107 (plus the CLI's --format csv)."""
    return call("tn_simulate", enc(memgraph_json), enc(profile_json), enc(policy), enc(tie_break), seed,
                enc(format))


def compare_policies(memgraph_json: str, profile_json: str = "", trials: int = 20, seed: int = 0) -> str:
    """bindings.cpp:109-116."""
    return call("tn_compare_policies", enc(memgraph_json), enc(profile_json), trials, seed)


def make_fixed_order(memgraph_json: str) -> str:
    """simulator.hpp:72-73 (C++-only in the reference)."""
    return call("tn_make_fixed_order", enc(memgraph_json))


def taskgraph_to_dot(graph_json: str) -> str:
    return call("tn_taskgraph_to_dot", enc(graph_json))


def memgraph_to_dot(memgraph_json: str) -> str:
    return call("tn_memgraph_to_dot", enc(memgraph_json))
