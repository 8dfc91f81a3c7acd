"""ctypes binding of include/sg_b200.h (argument marshalling only; all compute is in the .so).

Fails loudly if ``libsg_b200.so`` is missing: there is no CPU fallback on the product path.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SG_B200_LIB") or os.path.join(_HERE, "libsg_b200.so")

SG_OK = 0
SG_EINVAL = -1
SG_EUNSUPPORTED = -2
SG_EOVERFLOW = -3
SG_ENOMEM = -4
SG_ECUDA = -5
SG_ENONFINITE = -6
SG_ENOWORKSPACE = -7

# exported symbols (checked by tests/test_abi.py against include/sg_b200.h)
SYMBOLS = ["sg_plan", "sg_workspace_size", "sg_set_workspace", "sg_update_integrand",
           "sg_integrate", "sg_finalize", "sg_integrate_host", "sg_status_word", "sg_plan_points",
           "sg_plan_range", "sg_plan_passes", "sg_plan_leaf_work", "sg_debug_tables", "sg_plan_query",
           "sg_rule_table", "sg_profile_enable", "sg_profile_read", "sg_unrank", "sg_eval_points",
           "sg_destroy", "sg_strerror"]


class SGError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        msg = lib().sg_strerror(code).decode() if _lib is not None else str(code)
        super().__init__(f"{where}: {msg} (status {code})")


class sg_integrand_desc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("d", ctypes.c_int),
                ("c", ctypes.POINTER(ctypes.c_double)), ("w", ctypes.POINTER(ctypes.c_double)),
                ("u", ctypes.c_double)]


class sg_options(ctypes.Structure):
    _fields_ = [("form", ctypes.c_int), ("arith", ctypes.c_int), ("rank", ctypes.c_int),
                ("world", ctypes.c_int), ("range_lo", ctypes.c_longlong),
                ("range_hi", ctypes.c_longlong), ("merge", ctypes.c_int), ("method", ctypes.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not built: run `python -m paper_2210_14313_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        dp = ctypes.POINTER(ctypes.c_double)
        ull = ctypes.POINTER(ctypes.c_ulonglong)
        ll = ctypes.POINTER(ctypes.c_longlong)
        L.sg_plan.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                              ctypes.POINTER(sg_integrand_desc), ctypes.POINTER(sg_options),
                              ctypes.POINTER(vp)]
        L.sg_workspace_size.argtypes = [vp, ctypes.POINTER(ctypes.c_size_t)]
        L.sg_set_workspace.argtypes = [vp, vp, ctypes.c_size_t]
        L.sg_update_integrand.argtypes = [vp, vp, ctypes.POINTER(sg_integrand_desc)]
        L.sg_integrate.argtypes = [vp, vp, vp]
        L.sg_finalize.argtypes = [vp, vp, vp, ctypes.c_int, vp]
        L.sg_integrate_host.argtypes = [vp, vp, dp]
        L.sg_status_word.argtypes = [vp, ctypes.POINTER(ctypes.c_int)]
        L.sg_plan_points.argtypes = [vp, ull, ull]
        L.sg_plan_range.argtypes = [vp, ll, ll, ll]
        L.sg_plan_passes.argtypes = [vp, ctypes.POINTER(ctypes.c_int), ull, ull]
        L.sg_plan_leaf_work.argtypes = [vp, dp, dp]
        L.sg_debug_tables.argtypes = [vp, dp, ctypes.c_size_t, dp]
        L.sg_plan_query.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(sg_options), ull, ull, ll, ll,
                                    ctypes.POINTER(ctypes.c_int)]
        L.sg_rule_table.argtypes = [ctypes.c_int, ctypes.c_int, dp, dp]
        L.sg_profile_enable.argtypes = [vp, ctypes.c_int]
        L.sg_profile_read.argtypes = [vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_int)]
        ip = ctypes.POINTER(ctypes.c_int)
        L.sg_unrank.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                ctypes.POINTER(sg_options), ctypes.c_ulonglong, ip, ip, ip, ip, dp]
        L.sg_eval_points.argtypes = [vp, vp, vp, ctypes.c_longlong, vp, vp]
        L.sg_destroy.argtypes = [vp]
        L.sg_strerror.argtypes = [ctypes.c_int]
        L.sg_strerror.restype = ctypes.c_char_p
        for name in SYMBOLS:
            if name != "sg_strerror":
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def check(code: int, where: str) -> None:
    if code != SG_OK:
        raise SGError(code, where)
