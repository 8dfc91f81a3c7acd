"""Thin Python API over the C ABI (include/sg_b200.h).  Same names as the ABI; PyTorch only provides
device memory (workspace, outputs), the CUDA stream and torch.distributed process groups.

    plan = sg_plan(d, q, rule, kind, c, w, u)          # -> Plan (owns the C plan + workspace)
    out = plan.sg_integrate()                           # device tensor [hi, lo], async
    res = plan.sg_finalize(out)                         # device tensor [value, residual]
    value = plan.integrate_host()                       # synchronous float
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, lib, sg_integrand_desc, sg_options

RULE_CC = 2
RULE_GL = 4
KIND_EXP, KIND_OSC, KIND_PEAK, KIND_GAUSS, KIND_CORNER = 0, 1, 2, 3, 4
FORM_COMBINATION, FORM_DELTA = 0, 1
ARITH_FACTOR_DD, ARITH_SFORM_FP64, ARITH_SFORM_DD = 0, 1, 2   # s-forms: per-point outer function
                                                            # (FP64 ablation / dd, parity-grade)
MERGE_NONE, MERGE_MIDPOINT = 0, 1          # midpoint-merged evaluation (sg_merge)
METHOD_TREE, METHOD_COLLAPSE, METHOD_PLAIN = 0, 1, 2   # sg_method: prefix tree / separable collapse /
                                                      # plain per-point SG baseline (ablation)


def _stream_handle(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dptr(t: torch.Tensor) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr())


@dataclass
class PassInfo:
    terms: int       # tree nodes (Smolyak point terms) evaluated by the pass
    written: int     # frontier nodes written for the next pass


class Plan:
    """One sg_plan_t plus its torch-allocated workspace."""

    def __init__(self, d: int, q: int, rule: int, kind: int, c, w=None, u: float = 0.0,
                 form: int = FORM_COMBINATION, rank: int = 0, world: int = 1,
                 range_lo: int = 0, range_hi: int = -1, device=None,
                 arith: int = ARITH_FACTOR_DD, merge: int = MERGE_NONE, method: int = METHOD_TREE):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2210_14313_b200 needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device if device is not None else "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.d, self.q, self.rule, self.kind = int(d), int(q), int(rule), int(kind)
        self._c = np.ascontiguousarray(c, dtype=np.float64)
        self._w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
        self.u = float(u)
        desc = self._desc(self._c, self._w, self.u)
        opts = sg_options(int(form), int(arith), int(rank), int(world), int(range_lo), int(range_hi),
                          int(merge), int(method))
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            check(lib().sg_plan(self.d, self.q, self.rule, ctypes.byref(desc), ctypes.byref(opts),
                                ctypes.byref(h)), "sg_plan")
            self._h = h
            nbytes = ctypes.c_size_t()
            check(lib().sg_workspace_size(h, ctypes.byref(nbytes)), "sg_workspace_size")
            self.workspace_bytes = int(nbytes.value)
            self._ws = torch.empty(max(self.workspace_bytes, 256), dtype=torch.uint8,
                                   device=self.device)
            check(lib().sg_set_workspace(h, _dptr(self._ws), self._ws.numel()), "sg_set_workspace")
            self._out = torch.zeros(2, dtype=torch.float64, device=self.device)
            self._res = torch.zeros(2, dtype=torch.float64, device=self.device)

    def _desc(self, c, w, u):
        dp = ctypes.POINTER(ctypes.c_double)
        return sg_integrand_desc(self.kind, self.d, c.ctypes.data_as(dp),
                                 None if w is None else w.ctypes.data_as(dp), float(u))

    # -- C ABI wrappers ------------------------------------------------------------------------
    def sg_integrate(self, stream=None, out: torch.Tensor | None = None) -> torch.Tensor:
        out = self._out if out is None else out
        check(lib().sg_integrate(self._h, _stream_handle(stream), _dptr(out)), "sg_integrate")
        return out

    def sg_finalize(self, gathered: torch.Tensor, world: int = 1, stream=None,
                    result: torch.Tensor | None = None) -> torch.Tensor:
        result = self._res if result is None else result
        check(lib().sg_finalize(self._h, _stream_handle(stream), _dptr(gathered), int(world),
                                _dptr(result)), "sg_finalize")
        return result

    def sg_update_integrand(self, c, w=None, u: float | None = None, stream=None):
        """Async parameter refresh.  c/w: numpy (host) or torch tensors (pinned host or device).

        Tensors must be float64, contiguous, with d elements, on the CPU or on this plan's device
        (else ValueError: the C side reads exactly 8 d bytes from each pointer).  Host arrays are
        staged by the CUDA runtime before the call returns (pageable memory) or read by the copy
        engine in stream order (pinned tensors: keep them alive until the stream reaches the copy)."""
        dp = ctypes.POINTER(ctypes.c_double)
        keep = []

        def ptr(a):
            if a is None:
                return None
            if isinstance(a, torch.Tensor):
                if a.dtype != torch.float64 or not a.is_contiguous() or a.numel() != self.d:
                    raise ValueError("parameters must be contiguous float64 tensors of d elements")
                if a.device.type != "cpu" and a.device != self.device:
                    raise ValueError(f"parameter tensor on {a.device}, plan on {self.device}")
                return ctypes.cast(ctypes.c_void_p(a.data_ptr()), dp)
            a = np.ascontiguousarray(a, dtype=np.float64)
            if a.size != self.d:
                raise ValueError("parameters must have d elements")
            keep.append(a)   # alive until sg_update_integrand returns (pageable: staged by then)
            return a.ctypes.data_as(dp)

        desc = sg_integrand_desc(self.kind, self.d, ptr(c), ptr(w), float(self.u if u is None else u))
        check(lib().sg_update_integrand(self._h, _stream_handle(stream), ctypes.byref(desc)),
              "sg_update_integrand")
        if u is not None:
            self.u = float(u)

    def integrate_host(self, stream=None) -> tuple[float, float]:
        res = (ctypes.c_double * 2)()
        rc = lib().sg_integrate_host(self._h, _stream_handle(stream), res)
        check(rc, "sg_integrate_host")
        return float(res[0]), float(res[1])

    def status_word(self) -> int:
        v = ctypes.c_int()
        check(lib().sg_status_word(self._h, ctypes.byref(v)), "sg_status_word")
        return v.value

    def points(self) -> tuple[int, int]:
        a, b = ctypes.c_ulonglong(), ctypes.c_ulonglong()
        check(lib().sg_plan_points(self._h, ctypes.byref(a), ctypes.byref(b)), "sg_plan_points")
        return int(a.value), int(b.value)

    def range(self) -> tuple[int, int, int]:
        a, b, n = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_longlong()
        check(lib().sg_plan_range(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)),
              "sg_plan_range")
        return int(a.value), int(b.value), int(n.value)

    def passes(self) -> list[PassInfo]:
        n = ctypes.c_int(0)
        check(lib().sg_plan_passes(self._h, ctypes.byref(n), None, None), "sg_plan_passes")
        t = (ctypes.c_ulonglong * n.value)()
        w = (ctypes.c_ulonglong * n.value)()
        check(lib().sg_plan_passes(self._h, ctypes.byref(n), t, w), "sg_plan_passes")
        return [PassInfo(int(t[i]), int(w[i])) for i in range(n.value)]

    def leaf_work(self) -> tuple[float, float]:
        """(DFMA, DADD) FP64 thread-instructions per point of the dominant leaf kernel variant."""
        f, a = ctypes.c_double(), ctypes.c_double()
        check(lib().sg_plan_leaf_work(self._h, ctypes.byref(f), ctypes.byref(a)), "sg_plan_leaf_work")
        return float(f.value), float(a.value)

    def debug_tables(self):
        ncplx = 4 if self.kind == KIND_OSC else 2
        lo, hi, nd1 = self.range()
        buf = np.zeros(nd1 * ncplx)
        base = np.zeros(4)
        dp = ctypes.POINTER(ctypes.c_double)
        check(lib().sg_debug_tables(self._h, buf.ctypes.data_as(dp), buf.size,
                                    base.ctypes.data_as(dp)), "sg_debug_tables")
        return buf.reshape(nd1, ncplx), base

    def eval_points(self, index, stream=None):
        """Device K1 + per-point terms (sg_eval_points): index = int64-compatible tensor/array of
        flat point indices of this plan's shard.  Returns (points [n, 1 + 3L] int32 on device,
        terms [n, 2] float64 on device: (hi, lo) of coefficient * Re(point value))."""
        idx = torch.as_tensor(np.asarray(index, dtype=np.uint64).astype(np.int64), device=self.device)
        n = int(idx.numel())
        L = self.q - self.d
        pts = torch.empty((max(n, 1), 1 + 3 * L), dtype=torch.int32, device=self.device)
        terms = torch.empty((max(n, 1), 2), dtype=torch.float64, device=self.device)
        check(lib().sg_eval_points(self._h, _stream_handle(stream), _dptr(idx), n, _dptr(pts),
                                   _dptr(terms)), "sg_eval_points")
        return pts[:n], terms[:n]

    def capture_graph(self, finalize: bool = True, profile: bool = False):
        """Capture one step (sg_integrate, + sg_finalize(world=1) if `finalize`) into a CUDA graph.

        Returns the torch.cuda.CUDAGraph; ``graph.replay()`` re-runs the step with ~one launch of
        CPU overhead (the small configs are launch-latency bound).  The partial lands in the
        plan's default output (``sg_integrate()``'s tensor), the value in ``result()``.  With
        `profile`, the per-launch events are captured as graph event-record nodes and
        ``profile_read()`` returns the last replay's launch times."""
        self.profile_enable(profile)
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):
            out = self.sg_integrate(side)
            if finalize:
                self.sg_finalize(out, 1, side)
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            out = self.sg_integrate()
            if finalize:
                self.sg_finalize(out, 1)
        return g

    def result(self) -> torch.Tensor:
        """Device tensor [value, residual] written by sg_finalize (default output buffer)."""
        return self._res

    def profile_enable(self, on=True):
        """0/False off, 1/True every launch, 2 the dominant pass only (sg_profile_enable)."""
        mode = on if isinstance(on, int) and not isinstance(on, bool) else int(bool(on))
        check(lib().sg_profile_enable(self._h, mode), "sg_profile_enable")

    def profile_read(self) -> list[float]:
        """Device ms of each launch of the last sg_integrate:
        [K0 factor, K0 base, root pass, pass 1..nfront, final reduce]."""
        n = ctypes.c_int(0)
        check(lib().sg_profile_read(self._h, None, ctypes.byref(n)), "sg_profile_read")
        buf = (ctypes.c_float * n.value)()
        check(lib().sg_profile_read(self._h, buf, ctypes.byref(n)), "sg_profile_read")
        return [float(x) for x in buf]

    def close(self):
        if getattr(self, "_h", None):
            torch.cuda.synchronize(self.device)
            lib().sg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sg_unrank(d, q, rule, kind, index, form=FORM_COMBINATION, rank=0, world=1, range_lo=0,
              range_hi=-1, merge=MERGE_NONE):
    """Host-only K1 unranker: (coefficient, [(k, l, j), ...]) of the index-th Smolyak point of the
    shard in canonical (root, then depth-1 subtrees in preorder) order.  No GPU needed."""
    L = q - d
    n = max(L, 1)
    t = ctypes.c_int()
    k, l, j = (ctypes.c_int * n)(), (ctypes.c_int * n)(), (ctypes.c_int * n)()
    cf = ctypes.c_double()
    o = sg_options(int(form), 0, int(rank), int(world), int(range_lo), int(range_hi), int(merge), 0)
    check(lib().sg_unrank(d, q, rule, kind, ctypes.byref(o), int(index), ctypes.byref(t), k, l, j,
                          ctypes.byref(cf)), "sg_unrank")
    return cf.value, [(k[m], l[m], j[m]) for m in range(t.value)]


def sg_plan(d, q, rule, kind, c, w=None, u=0.0, **kw) -> Plan:
    return Plan(d, q, rule, kind, c, w, u, **kw)


def integrate(d, L, rule, kind, c, w=None, u=0.0, form=FORM_COMBINATION, **kw) -> tuple[float, float]:
    """One-shot A(d+L, d) f on the current CUDA device -> (value, residual) double-double."""
    p = Plan(d, d + L, rule, kind, c, w, u, form=form, **kw)
    try:
        return p.integrate_host()
    finally:
        p.close()


def integrate_distributed(d, L, rule, kind, c, w=None, u=0.0, form=FORM_COMBINATION,
                          group=None) -> tuple[float, float]:
    """Shard the depth-1 subtrees over the ranks of ``group`` (one GPU per rank), one
    all_gather_into_tensor of the 2-double partials (NCCL over NVLink), fixed rank-order dd sum."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    p = Plan(d, d + L, rule, kind, c, w, u, form=form, rank=rank, world=world)
    try:
        part = p.sg_integrate()
        gathered = torch.empty(2 * world, dtype=torch.float64, device=p.device)
        dist.all_gather_into_tensor(gathered, part, group=group)
        res = p.sg_finalize(gathered, world)
        r = res.cpu()
        return float(r[0]), float(r[1])
    finally:
        p.close()
