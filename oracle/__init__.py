"""ORACLE — test infrastructure only (see sg_oracle.c header).

Python ctypes wrapper around ``liboracle_sg.so`` (plain C, __float128, OpenMP).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may
import this package.  It never imports the CUDA product package and shares no code with it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sg_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_sg.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, OpenMP, libquadmath).  No fast-math: quad is soft-float."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=gnu11", _SRC,
               "-o", _LIB + ".tmp", "-lquadmath", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        lib.sgo_node_count.argtypes = [ctypes.c_int, ctypes.c_int]
        lib.sgo_node_count.restype = ctypes.c_int
        lib.sgo_rule.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp]
        lib.sgo_rule.restype = ctypes.c_int
        lib.sgo_integrate.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, ctypes.c_double,
            ctypes.c_longlong, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int,
            dp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_longlong), dp]
        lib.sgo_integrate.restype = ctypes.c_int
        lib.sgo_eval_point.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp, ctypes.c_double, dp,
                                       dp, dp]
        lib.sgo_eval_point.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def node_count(rule: int, level: int) -> int:
    return _load().sgo_node_count(rule, level)


def rule(rule_id: int, level: int):
    """(nodes, weights) of the 1-D rule at ``level`` on [0,1], float64."""
    n = node_count(rule_id, level)
    if n < 0:
        raise ValueError("unsupported level")
    x = np.zeros(n)
    w = np.zeros(n)
    if _load().sgo_rule(rule_id, level, _ptr(x), _ptr(w)) < 0:
        raise ValueError("unsupported level")
    return x, w


@dataclass
class OracleResult:
    hi: float
    lo: float
    text: str          # quad value, 37 significant digits
    npoints: int
    seconds: float

    @property
    def value(self) -> float:
        return self.hi


def integrate(d: int, L: int, rule_id: int, kind: int, c, w=None, u: float = 0.0,
              lo: int = 0, hi: int = -1, include_root: bool = True, eval_mode: int = 0,
              nthreads: int = 0) -> OracleResult:
    """Eq 2.6 with q = d + L on [0,1]^d, in __float128.

    ``lo``/``hi`` restrict to points whose first active coordinate triple (k1, l1, j1) has depth-1
    lexicographic rank in [lo, hi) (shard semantics); ``include_root`` adds
    the all-midpoint point.  ``eval_mode`` 0 = plain O(d) integrand, 1 = active-coordinate form.
    """
    c = np.ascontiguousarray(c, dtype=np.float64)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    out = np.zeros(2)
    buf = ctypes.create_string_buffer(64)
    npts = ctypes.c_longlong(0)
    secs = ctypes.c_double(0)
    rc = _load().sgo_integrate(d, L, rule_id, kind, _ptr(c), _ptr(w), float(u), int(lo), int(hi),
                               int(bool(include_root)), int(eval_mode), int(nthreads), _ptr(out),
                               buf, ctypes.byref(npts), ctypes.byref(secs))
    if rc != 0:
        raise ValueError("oracle rejected arguments")
    return OracleResult(float(out[0]), float(out[1]), buf.value.decode(), int(npts.value),
                        float(secs.value))


def integrate_problem(p, **kw) -> OracleResult:
    return integrate(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u, **kw)


def eval_point(kind: int, c, w, u: float, x):
    """f at one full point, (plain, active) forms, each as a (hi, lo) pair of doubles."""
    c = np.ascontiguousarray(c, dtype=np.float64)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    a = np.zeros(2)
    b = np.zeros(2)
    _load().sgo_eval_point(len(c), kind, _ptr(c), _ptr(w), float(u), _ptr(x), _ptr(a), _ptr(b))
    return (a[0], a[1]), (b[0], b[1])
