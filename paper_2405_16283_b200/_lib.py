"""ctypes binding of the C ABI in include/turnip.h (libturnip_b200.so).

This is the reference-side binding a maintainer would write: plain pointers,
sizes and JSON strings; no torch types cross the boundary.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, byref, c_char_p, c_double, c_int, c_int64, c_size_t, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libturnip_b200.so")


class MemplanError(RuntimeError):
    """Mirror of the reference's `_memplan.MemplanError` (bindings.cpp:34).

    `code` is the C-ABI return code (1 check/deadlock, 2 usage/parse/plan,
    3 CUDA)."""

    def __init__(self, msg: str, code: int = 2):
        super().__init__(msg)
        self.code = code


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        L = ctypes.CDLL(LIB_PATH)
        P = POINTER(c_char_p)
        sig = {
            "tn_version": (c_char_p, []),
            "tn_free": (None, [c_void_p]),
            "tn_validate_taskgraph": (c_int, [c_char_p, P, P]),
            "tn_topological_order": (c_int, [c_char_p, c_char_p, c_uint64, P, P]),
            "tn_taskgraph_to_dot": (c_int, [c_char_p, P, P]),
            "tn_memgraph_to_dot": (c_int, [c_char_p, P, P]),
            "tn_build_memgraph": (
                c_int,
                [c_char_p, POINTER(c_int64), c_size_t, c_char_p, POINTER(c_int64), c_size_t, c_char_p,
                 c_char_p, c_uint64, c_char_p, c_int, c_int64, P, P, P],
            ),
            "tn_simulate": (c_int, [c_char_p, c_char_p, c_char_p, c_char_p, c_uint64, c_char_p, P, P]),
            "tn_compare_policies": (c_int, [c_char_p, c_char_p, c_int64, c_uint64, P, P]),
            "tn_make_fixed_order": (c_int, [c_char_p, P, P]),
            "tn_verify": (c_int, [c_char_p, c_char_p, c_int64, P, P]),
            "tn_check_capacity": (c_int, [c_char_p, POINTER(c_int64), c_size_t, P, P]),
        }
        exec_sig = {
            "tn_exec_create": (c_int, [c_char_p, c_char_p, c_char_p, POINTER(c_void_p), P]),
            "tn_exec_set_input": (c_int, [c_void_p, c_int64, c_void_p, c_size_t, P]),
            "tn_exec_set_input_device": (c_int, [c_void_p, c_int64, c_void_p, c_size_t, P]),
            "tn_exec_run": (c_int, [c_void_p, c_char_p, c_char_p, c_uint64, P, P]),
            "tn_exec_get_output": (c_int, [c_void_p, c_int64, c_void_p, c_size_t, P]),
            "tn_exec_last_trace": (c_int, [c_void_p, P, P]),
            "tn_exec_placement_ptr": (c_int, [c_void_p, c_int64, POINTER(c_void_p), P]),
            "tn_exec_stats": (c_int, [c_void_p, P, P]),
            "tn_exec_compare_policies": (c_int, [c_void_p, c_int64, c_uint64, P, P]),
            "tn_exec_destroy": (None, [c_void_p]),
        }
        for name, (res, args) in {**sig, **exec_sig}.items():
            fn = getattr(L, name)  # AttributeError: the library lacks a declared symbol
            fn.restype = res
            fn.argtypes = args
        # char** outputs must be freed with tn_free, so read them as raw pointers.
        for name in list(sig) + list(exec_sig):
            fn = getattr(L, name)
            fn.argtypes = [c_void_p if a is P else a for a in fn.argtypes]
        _lib = L
    return _lib


class Out:
    """A char* out-parameter that is released with tn_free."""

    def __init__(self):
        self.p = c_char_p()

    @property
    def ref(self):
        return ctypes.cast(byref(self.p), c_void_p)

    def take(self) -> str | None:
        if not self.p:
            return None
        v = ctypes.string_at(self.p).decode()
        lib().tn_free(self.p)
        self.p = c_char_p()
        return v


def enc(s):
    return None if s is None else s.encode()


def check(rc: int, err: Out):
    if rc != 0:
        raise MemplanError(err.take() or f"error code {rc}", rc)


def call(name: str, *args, nout: int = 1):
    """Calls tn_<name>(*args, out_1..out_n, err) and returns the outputs."""
    outs = [Out() for _ in range(nout)]
    err = Out()
    rc = getattr(lib(), name)(*args, *[o.ref for o in outs], err.ref)
    check(rc, err)
    vals = [o.take() for o in outs]
    return vals[0] if nout == 1 else tuple(vals)


def i64_array(vals):
    vals = list(vals)
    arr = (c_int64 * max(len(vals), 1))(*vals)
    return arr, len(vals)
