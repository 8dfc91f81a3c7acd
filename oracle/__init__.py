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


_LIB64 = os.path.join(_HERE, "liboracle_sg_fp64.so")
_lib64 = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, OpenMP, libquadmath).  No fast-math: quad is soft-float.
    Also builds the FP64 instantiation of the same source (-DSGO_FP64: sums and integrand in double,
    a CPU speed baseline that is NOT parity-grade)."""
    for lib_path, extra in ((_LIB, []), (_LIB64, ["-DSGO_FP64", "-ffp-contract=off"])):
        if force or not os.path.exists(lib_path) or os.path.getmtime(lib_path) < os.path.getmtime(_SRC):
            cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=gnu11", *extra, _SRC,
                   "-o", lib_path + ".tmp", "-lquadmath", "-lm"]
            subprocess.check_call(cmd)
            os.replace(lib_path + ".tmp", lib_path)
    return _LIB


def _load(fp64: bool = False):
    global _lib, _lib64
    if fp64:
        if _lib64 is None:
            build()
            _lib64 = _bind(ctypes.CDLL(_LIB64))
        return _lib64
    if _lib is None:
        build()
        _lib = _bind(ctypes.CDLL(_LIB))
    return _lib


def _bind(lib):
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
    lib.sgo_integrate_ex.argtypes = [
        ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, dp, dp, ctypes.c_double,
        ctypes.c_longlong, ctypes.c_longlong, ctypes.c_longlong, ctypes.c_int, ctypes.c_int,
        ctypes.c_int, ctypes.c_int, dp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_longlong), dp]
    lib.sgo_integrate_ex.restype = ctypes.c_int
    return lib


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
              nthreads: int = 0, stride: int = 1, count_only: bool = False,
              fp64: bool = False) -> OracleResult:
    """Eq 2.6 with q = d + L on [0,1]^d, in __float128.

    ``lo``/``hi`` restrict to points whose first active coordinate triple (k1, l1, j1) has depth-1
    lexicographic rank in [lo, hi) (shard semantics); ``include_root`` adds
    the all-midpoint point.  ``eval_mode`` 0 = plain O(d) integrand, 1 = active-coordinate form.
    ``stride`` > 1 keeps only every stride-th depth-2 multi-index subtree of each top-level item (an
    evenly spread sample of the tree, for CPU timing); ``count_only`` counts the selected points without evaluating them;
    ``fp64`` runs the FP64 instantiation of the same program (speed baseline, not parity-grade).
    """
    c = np.ascontiguousarray(c, dtype=np.float64)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    out = np.zeros(2)
    buf = ctypes.create_string_buffer(64)
    npts = ctypes.c_longlong(0)
    secs = ctypes.c_double(0)
    rc = _load(fp64).sgo_integrate_ex(d, L, rule_id, kind, _ptr(c), _ptr(w), float(u), int(lo),
                                      int(hi), int(stride), int(bool(include_root)), int(eval_mode),
                                      int(nthreads), int(bool(count_only)), _ptr(out), buf,
                                      ctypes.byref(npts), ctypes.byref(secs))
    if rc != 0:
        raise ValueError("oracle rejected arguments")
    return OracleResult(float(out[0]), float(out[1]), buf.value.decode(), int(npts.value),
                        float(secs.value))


def integrate_problem(p, **kw) -> OracleResult:
    return integrate(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u, **kw)


def count_points(p, **kw) -> int:
    """Smolyak points of the (restricted / sampled) point set, counted by the oracle's own
    multi-index walk (no evaluation)."""
    return integrate_problem(p, count_only=True, **kw).npoints


def depth1_count(p) -> int:
    """Number of depth-1 prefixes (k1, l1, j1): d * sum_{l=2}^{L+1} n_l."""
    return p.d * sum(node_count(p.rule, l) for l in range(2, p.L + 2))


def n_points(p) -> int:
    """n_d^q for q = d + L: the sum over the band e = max(0, L-d+1) .. L of the
    multi-index products n_{l_1} ... n_{l_d}, i.e. [z^e] (sum_{l=1}^{L+1} n_l z^{l-1})^d, written
    out as a truncated polynomial power in exact integers."""
    g = [node_count(p.rule, l) for l in range(1, p.L + 2)]
    acc = [1] + [0] * p.L
    for _ in range(p.d):
        acc = [sum(acc[i] * g[e - i] for i in range(e + 1)) for e in range(p.L + 1)]
    return sum(acc[e] for e in range(max(0, p.L - p.d + 1), p.L + 1))


def timing_sample(p, target_points: int, nthreads: int = 0, fp64: bool = False, eval_mode: int = 1):
    """A bounded CPU timing sample of problem p: every s-th depth-2 multi-index subtree of the whole
    tree (sgo_integrate_ex stride), s calibrated with the oracle's point count so the sample holds
    about target_points points, evaluated by the oracle as it stands.
    Returns (OracleResult, stride, n_d^q)."""
    import math
    total = n_points(p)
    stride = max(1, round(total / max(1, target_points)))
    best = None
    for _ in range(8):   # sample sizes are heavy-tailed in the subtree sizes: calibrate on counts
        if stride == 1:
            best = (0.0, 1)
            break
        n = count_points(p, stride=stride, include_root=False, nthreads=nthreads)
        dev = abs(math.log(max(n, 1) / target_points))
        if best is None or dev < best[0]:
            best = (dev, stride)
        if dev < math.log(1.25):
            break
        stride = max(1, round(stride * max(n, 1) / target_points))
    stride = best[1]
    r = integrate_problem(p, stride=stride, include_root=False, eval_mode=eval_mode,
                          nthreads=nthreads, fp64=fp64)
    return r, stride, total


def eval_point(kind: int, c, w, u: float, x):
    """f at one full point, (plain, active) forms, each as a (hi, lo) pair of doubles."""
    c = np.ascontiguousarray(c, dtype=np.float64)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    a = np.zeros(2)
    b = np.zeros(2)
    _load().sgo_eval_point(len(c), kind, _ptr(c), _ptr(w), float(u), _ptr(x), _ptr(a), _ptr(b))
    return (a[0], a[1]), (b[0], b[1])
