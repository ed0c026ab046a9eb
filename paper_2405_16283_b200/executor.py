"""Real execution of memgraphs on B200 GPUs (the slot of the reference
`simulate`, proj/include/memplan/simulator.hpp:67-68), through the C ABI
`tn_exec_*` in include/turnip.h.

    ex = Executor(memgraph_json, taskgraph_json, {"streams_per_device": 5})
    ex.set_input(vid, numpy_array_or_cuda_tensor)
    trace_json = ex.run(policy="event-driven", tie_break="fifo", seed=0)
    out = ex.get_output(vid, nbytes)

There is no CPU fallback: without the CUDA library (or a GPU) this raises.
"""
from __future__ import annotations

import ctypes
import json
from ctypes import byref, c_void_p

from ._lib import MemplanError, Out, check, enc, lib


class Executor:
    def __init__(self, memgraph_json: str, taskgraph_json: str, config: dict | str | None = None):
        cfg = config if isinstance(config, str) else json.dumps(config or {})
        h = c_void_p()
        err = Out()
        check(lib().tn_exec_create(enc(memgraph_json), enc(taskgraph_json), enc(cfg), byref(h), err.ref), err)
        self._h = h

    def _ptr(self):
        if not self._h:
            raise MemplanError("executor is closed")
        return self._h

    def set_input(self, vid: int, data) -> None:
        """`data`: numpy array / bytes (host) or a torch tensor (CUDA or CPU)."""
        err = Out()
        mod = type(data).__module__
        if mod.startswith("torch"):
            t = data.contiguous()
            nbytes = t.numel() * t.element_size()
            if t.is_cuda:
                rc = lib().tn_exec_set_input_device(self._ptr(), vid, c_void_p(t.data_ptr()), nbytes, err.ref)
            else:
                rc = lib().tn_exec_set_input(self._ptr(), vid, c_void_p(t.data_ptr()), nbytes, err.ref)
            check(rc, err)
            return
        if hasattr(data, "ctypes"):
            import numpy as np

            a = np.ascontiguousarray(data)
            rc = lib().tn_exec_set_input(self._ptr(), vid, a.ctypes.data_as(c_void_p), a.nbytes, err.ref)
        else:
            b = bytes(data)
            buf = ctypes.create_string_buffer(b, len(b))
            rc = lib().tn_exec_set_input(self._ptr(), vid, ctypes.cast(buf, c_void_p), len(b), err.ref)
        check(rc, err)

    def run(self, policy: str = "event-driven", tie_break: str | None = None, seed: int = 0,
            trace: bool = True) -> str | None:
        """tie_break None: the config's "tie_break" (default "plan-order")."""
        out, err = Out(), Out()
        rc = lib().tn_exec_run(self._ptr(), enc(policy), enc(tie_break or ""), seed, out.ref if trace else None,
                               err.ref)
        check(rc, err)
        return out.take()

    def last_trace(self) -> str:
        """Trace of the most recent run (useful after runs with trace=False)."""
        out, err = Out(), Out()
        check(lib().tn_exec_last_trace(self._ptr(), out.ref, err.ref), err)
        return out.take()

    def get_output(self, vid: int, nbytes: int) -> bytes:
        buf = ctypes.create_string_buffer(nbytes)
        err = Out()
        check(lib().tn_exec_get_output(self._ptr(), vid, ctypes.cast(buf, c_void_p), nbytes, err.ref), err)
        return buf.raw

    def placement_ptr(self, vid: int) -> int:
        p, err = c_void_p(), Out()
        check(lib().tn_exec_placement_ptr(self._ptr(), vid, byref(p), err.ref), err)
        return p.value or 0

    def stats(self) -> dict:
        out, err = Out(), Out()
        check(lib().tn_exec_stats(self._ptr(), out.ref, err.ref), err)
        return json.loads(out.take())

    def compare_policies(self, trials: int = 10, seed: int = 0) -> str:
        """Hardware counterpart of memplan.compare_policies (bindings.cpp:109-116):
        paired event-driven / fixed-order runs of this memgraph with
        device-timed makespans; the reference's summary JSON schema."""
        out, err = Out(), Out()
        check(lib().tn_exec_compare_policies(self._ptr(), trials, seed, out.ref, err.ref), err)
        return out.take()

    def close(self) -> None:
        if self._h:
            lib().tn_exec_destroy(self._h)
            self._h = c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def execute(memgraph_json: str, taskgraph_json: str, inputs: dict, outputs=(), config=None,
            policy: str = "event-driven", tie_break: str | None = None, seed: int = 0):
    """One-shot: returns (trace_json, {vid: bytes}) — the real-hardware
    counterpart of `memplan.simulate(memgraph_json, ...)`. tie_break None: the
    config's (default "plan-order"; simulate's default is the reference's "fifo")."""
    mg = json.loads(memgraph_json)
    sizes = {int(k): p["size"] for k, p in mg["placement"].items()}
    with Executor(memgraph_json, taskgraph_json, config) as ex:
        for vid, data in inputs.items():
            ex.set_input(vid, data)
        trace = ex.run(policy, tie_break, seed)
        outs = {vid: ex.get_output(vid, sizes[vid]) for vid in outputs}
    return trace, outs
