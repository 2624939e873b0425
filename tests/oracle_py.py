"""Test-side access to the oracle (TEST INFRASTRUCTURE ONLY).

Binds oracle/liboracle_conv.so (plain-C fp64 restatement of
reference_conv.hpp) and, when built here, oracle/_ref/ref_conv.so (the
reference's own conv compiled from /root/reference). Used only by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg, as the checker.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle_conv.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "ref_conv.so")

_oracle = None
_ref = None


def oracle():
    global _oracle
    if _oracle is None:
        l = C.CDLL(ORACLE_SO)
        dp = C.POINTER(C.c_double)
        lp = C.POINTER(C.c_longlong)
        for n in ("oracle_conv_forward", "oracle_conv_backward_data", "oracle_conv_backward_filter_acc"):
            getattr(l, n).argtypes = [lp, dp, dp, dp]
            getattr(l, n).restype = None
        l.oracle_execute_plan.argtypes = [C.c_int, lp, lp, C.c_int, dp, dp, dp]
        l.oracle_execute_plan.restype = C.c_int
        l.oracle_set_threads.argtypes = [C.c_int]
        _oracle = l
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        l = C.CDLL(REF_SO)
        dp = C.POINTER(C.c_double)
        lp = C.POINTER(C.c_longlong)
        l.ref_execute_plan.argtypes = [C.c_int, lp, lp, C.c_int, dp, dp, dp]
        l.ref_execute_plan.restype = C.c_int
        l.ref_conv_threads.argtypes = [C.c_int, lp, dp, dp, dp, C.c_int]
        l.ref_conv_threads.restype = C.c_int
        _ref = l
    return _ref


def _shape(s):
    return (C.c_longlong * 11)(s.N, s.C, s.H, s.W, s.K, s.R, s.S, s.ph, s.pw, s.sh, s.sw)


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def out_shape(op, s):
    return [(s.N, s.K, s.OH, s.OW), (s.N, s.C, s.H, s.W), (s.K, s.C, s.R, s.S)][op]


def conv_ref(op, s, a, b, micro=None, use_reference=False):
    """fp64 result of op 0 (x,w->y), 1 (dy,w->dx), 2 (x,dy->dw) under the
    micro-batch plan `micro` (list of sizes; default undivided)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.zeros(out_shape(op, s), dtype=np.float64)
    micro = list(micro) if micro else [s.N]
    m = (C.c_longlong * len(micro))(*micro)
    lib = ref() if use_reference else oracle()
    fn = lib.ref_execute_plan if use_reference else lib.oracle_execute_plan
    rc = fn(op, _shape(s), m, len(micro), _dp(a), _dp(b), _dp(out))
    assert rc == 0, "oracle rejected the plan"
    return out


def ref_conv_threads(op, s, a, b, threads):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    out = np.zeros(out_shape(op, s), dtype=np.float64)
    assert ref().ref_conv_threads(op, _shape(s), _dp(a), _dp(b), _dp(out), threads) == 0
    return out


def rand_int(rng, shape, lo=-3, hi=3):
    """Integer tensors in [lo, hi] (reference test_util.hpp:72-78 style): exact in TF32."""
    return rng.integers(lo, hi + 1, size=shape).astype(np.float64)


def inputs_for(op, s, rng, integer=True):
    gen = (lambda sh: rand_int(rng, sh)) if integer else (lambda sh: rng.standard_normal(sh))
    x = gen((s.N, s.C, s.H, s.W))
    w = gen((s.K, s.C, s.R, s.S))
    dy = gen((s.N, s.K, s.OH, s.OW))
    return [(x, w), (dy, w), (x, dy)][op]
