"""bench.py — Smolyak points/s and time-to-integral (FP64) of the B200 hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N ...      (one rank per GPU, NCCL)

Workload (default): BASELINE.json configs[4] — d=300, q=d+4, Clenshaw-Curtis, oscillatory Genz
integrand (seed 4), 27,521,113,876 Smolyak points: the configuration BASELINE.json ties to the
1/2/4/8-GPU scaling run; it fits one GPU.  A step = the whole hot path:
K0 factor tables, root pass, all prefix-tree passes, deterministic reduction, the cross-rank
all-gather + fixed-order finalize.  Rank r evaluates its shard of depth-1 subtrees (strong scaling:
the integral is fixed, the work is split).  Inputs (integrand parameters) are device-resident at
the start of the timed region; L2 is flushed (256 MiB write) between timed steps, outside the
events.  Times: CUDA events on the launching stream, barrier + synchronize on both sides, max over
ranks.  The "e2e" leg times the same step through the C ABI with HOST buffers: pinned H2D of the
parameters (sg_update_integrand), the step, and the D2H read of the 16-byte result.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import sg_configs as S  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
# Algorithmic FP64 work per Smolyak point of the dominant leaf kernel comes from the library
# (sg_plan_leaf_work: DFMA and DADD thread-instructions per point of the variant the plan runs;
# DESIGN.md §6): flops = 2 DFMA + DADD, pipe slots = DFMA + DADD.
# FP64 peak derived from the unit count and clock: 148 SMs x 64 FP64 FMA/clk x 2 flops
# x 1.965 GHz (MEASURED_PEAKS.json sm_max_mhz) = 37.2 TFLOP/s.
SM_COUNT = 148
FP64_FMA_PER_SM_CLK = 64


def peak_fp64_tflops():
    mhz = 1965.0
    try:
        mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
    except Exception:
        pass
    return SM_COUNT * FP64_FMA_PER_SM_CLK * 2 * mhz * 1e6 / 1e12, mhz


# ----------------------------------------------------------------------------------------------
# clocks sampled during the timed region (pynvml)
# ----------------------------------------------------------------------------------------------
class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz, self.power = [], set(), None, []
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                try:
                    self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                except Exception:
                    pass
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "power_w": statistics.median(self.power) if self.power else None}


# ----------------------------------------------------------------------------------------------
# CPU oracle sample (cpu_baseline and --impl reference)
# ----------------------------------------------------------------------------------------------
def oracle_sample_range(p: S.Problem, target_points: int):
    """Depth-1 range [lo, nd1) of the workload whose subtrees hold about target_points points
    (host-only library query; the range is the sample the oracle times)."""
    from paper_2210_14313_b200._lib import lib, sg_options
    L = lib()

    def pts(lo, hi):
        o = sg_options(0, 0, 0, 1, lo, hi)
        sp = ctypes.c_ulonglong()
        rc = L.sg_plan_query(p.d, p.q, p.rule, p.kind, ctypes.byref(o), ctypes.byref(sp), None,
                             None, None, None)
        assert rc == 0
        return sp.value

    o = sg_options(0, 0, 0, 1, 0, -1)
    nd1 = ctypes.c_longlong()
    hi_ = ctypes.c_longlong()
    L.sg_plan_query(p.d, p.q, p.rule, p.kind, ctypes.byref(o), None, None, None,
                    ctypes.byref(hi_), None)
    nd1 = hi_.value
    a, b = 1, nd1
    while a < b:   # smallest lo such that points(lo, nd1) <= target
        m = (a + b) // 2
        if pts(m, nd1) > target_points:
            a = m + 1
        else:
            b = m
    return a, nd1, pts(a, nd1)


def run_oracle_sample(p, lo, hi):
    import oracle
    # all host cores, explicitly: torchrun sets OMP_NUM_THREADS=1 for its ranks
    r = oracle.integrate_problem(p, lo=lo, hi=hi, include_root=False, eval_mode=1,
                                 nthreads=os.cpu_count())
    return r


def cpu_baseline(p, target_points=int(1.2e8)):
    lo, hi, npts = oracle_sample_range(p, target_points)
    r = run_oracle_sample(p, lo, hi)
    cores = os.cpu_count()
    return {"value": r.npoints / r.seconds, "unit": "points/s", "cores": cores, "kind": "oracle",
            "sample": f"{p.name} depth-1 subtrees [{lo},{hi}) = {r.npoints} of "
                      f"{S_total_points(p)} Smolyak points, __float128 oracle (eval_mode=1), "
                      f"OpenMP {cores} threads, {r.seconds:.2f} s",
            "seconds": r.seconds, "points": r.npoints}


def S_total_points(p):
    from paper_2210_14313_b200._lib import lib, sg_options
    o = sg_options(0, 0, 0, 1, 0, -1)
    tp = ctypes.c_ulonglong()
    lib().sg_plan_query(p.d, p.q, p.rule, p.kind, ctypes.byref(o), None, ctypes.byref(tp), None,
                        None, None)
    return tp.value


def config_block(p, extra=None):
    c = {"workload": f"BASELINE.json configs[{int(p.name[1:]) - 1}] ({p.name}): d={p.d}, "
                     f"q=d+{p.L}, {S.RULE_NAMES[p.rule]}, {S.KIND_NAMES[p.kind]} integrand",
         "d": p.d, "q": p.q, "L": p.L, "rule": S.RULE_NAMES[p.rule],
         "integrand": S.KIND_NAMES[p.kind], "points": S_total_points(p),
         "form": "combination (Eq 2.6)", "arith": "factor-form double-double",
         "l2": "flushed between timed steps (256 MiB write, outside the events)"}
    if extra:
        c.update(extra)
    return c


# ----------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-merged", action="store_true", help="skip the SG_MERGE_MIDPOINT leg")
    ap.add_argument("--no-graph", action="store_true",
                    help="time the stream-launched step instead of its CUDA-graph replay")
    ap.add_argument("--no-collapse", action="store_true", help="skip the SG_METHOD_COLLAPSE leg")
    ap.add_argument("--no-frontier", action="store_true",
                    help="skip the stored-frontier (unfused) leg that measures the HBM-bound frontier kernel")
    ap.add_argument("--no-plain", action="store_true",
                    help="skip the plain per-point SG ablation leg (SG_METHOD_PLAIN)")
    ap.add_argument("--no-corner", action="store_true",
                    help="skip the non-separable corner-peak leg (SG_ARITH_SFORM_DD)")
    # testing aids for the multi-rank path on a 1-GPU box: gloo carries the 16-byte collective
    # through host memory and every rank may share one device (ranks never wait on each other
    # inside a kernel, so sharing is safe); the product configuration is nccl + one GPU per rank
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--device-index", type=int, default=None)
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    p = S.baseline_config(args.config)

    if args.impl == "reference":
        if rank != 0:
            return
        return bench_reference(p, args, world)

    import torch
    import torch.distributed as dist
    from paper_2210_14313_b200 import api
    from paper_2210_14313_b200 import build as B

    if rank == 0 or world == 1:
        B.build()
    local = local if args.device_index is None else args.device_index
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        dist.barrier()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)

    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=rank, world=world, device=dev)
    plan.profile_enable(True)
    shard_pts, total_pts = plan.points()
    passes = plan.passes()
    dominant = max(range(1, len(passes)), key=lambda i: passes[i].terms) if len(passes) > 1 else 0
    gathered = torch.zeros(2 * world, dtype=torch.float64, device=dev)
    result = torch.zeros(2, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step(plan=plan):
        part = plan.sg_integrate(stream)
        if world > 1:
            if args.dist_backend == "nccl":
                dist.all_gather_into_tensor(gathered, part)
            else:
                g = torch.zeros(2 * world, dtype=torch.float64)
                dist.all_gather_into_tensor(g, part.cpu())
                gathered.copy_(g)
            plan.sg_finalize(gathered, world, stream, result)
        else:
            plan.sg_finalize(part, 1, stream, result)

    def graph_step(plan):
        """The step as one CUDA-graph replay (sg_integrate, + sg_finalize at world 1; the launch
        events are graph event-record nodes, so profile_read still times each launch); at world > 1
        the all-gather and sg_finalize follow the replay as in step()."""
        if args.no_graph:
            return lambda: step(plan)
        plan.profile_enable(True)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            part = plan.sg_integrate()
            if world == 1:
                plan.sg_finalize(part, 1, None, result)

        def fn():
            g.replay()
            if world > 1:
                if args.dist_backend == "nccl":
                    dist.all_gather_into_tensor(gathered, part)
                else:
                    gl = torch.zeros(2 * world, dtype=torch.float64)
                    dist.all_gather_into_tensor(gl, part.cpu())
                    gathered.copy_(gl)
                plan.sg_finalize(gathered, world, stream, result)
        fn.graph = g
        return fn

    def timed(fn, k, plan=plan, dominant=dominant):
        times, dom = [], []
        for _ in range(k):
            flush.fill_(1.0)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ms = e0.elapsed_time(e1)
            if world > 1:
                t = torch.tensor([ms], dtype=torch.float64,
                                 device=dev if args.dist_backend == "nccl" else "cpu")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                ms = float(t.item())
            times.append(ms)
            prof = plan.profile_read()
            dom.append(prof[3 + dominant - 1] if dominant > 0 else prof[2])
        return times, dom

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    gstep = graph_step(plan)
    for _ in range(args.warmup):
        gstep()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        times, dom = timed(gstep, args.steps)
    ms = statistics.mean(times)

    # e2e: host buffers through the C ABI (pinned H2D of c/w, step, D2H of the result)
    c_host = torch.from_numpy(p.c.copy()).pin_memory()
    w_host = torch.from_numpy(p.w.copy()).pin_memory() if p.w is not None else None
    res_host = torch.zeros(2, dtype=torch.float64).pin_memory()

    def e2e_step():
        plan.sg_update_integrand(c_host, w_host, p.u, stream)
        step()
        res_host.copy_(result, non_blocking=True)

    for _ in range(2):
        e2e_step()
    e2e_times, _ = timed(e2e_step, args.steps)
    e2e_ms = statistics.mean(e2e_times)
    h2d = 8 * p.d * (2 if p.w is not None else 1) + 8
    value_res = result.cpu().numpy()

    # merged leg (SG_MERGE_MIDPOINT): the same integral with the midpoint copies of
    # every point summed into merged coefficients, each remaining point evaluated once
    merged = None
    if not args.no_merged:
        mplan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=rank, world=world,
                         device=dev, merge=api.MERGE_MIDPOINT)
        mplan.profile_enable(True)
        m_shard, m_total = mplan.points()
        mpasses = mplan.passes()
        mdom = max(range(1, len(mpasses)), key=lambda i: mpasses[i].terms) if len(mpasses) > 1 else 0
        for _ in range(args.warmup):
            step(mplan)
        torch.cuda.synchronize(dev)
        mstep = graph_step(mplan)
        mstep()
        m_times, m_dom = timed(mstep, args.steps, mplan, mdom)
        m_res = result.cpu().numpy()
        m_ms = statistics.mean(m_times)
        mf, ma = mplan.leaf_work()
        m_dom_ms = statistics.mean(m_dom)
        peak_, mhz_ = peak_fp64_tflops()
        m_ach = mpasses[mdom].terms * (2 * mf + ma) / (m_dom_ms * 1e-3) / 1e12
        merged = {
            "time_to_integral_ms": m_ms, "points": m_total,
            "value": m_total / (m_ms * 1e-3), "unit": "points/s",
            "eq26_points_per_s": total_pts / (m_ms * 1e-3),
            "speedup_vs_combination": ms / m_ms,
            "result": float(m_res[0]),
            "rel_diff_vs_combination": abs((float(m_res[0]) + float(m_res[1]))
                                           - (float(value_res[0]) + float(value_res[1])))
                                       / abs(float(value_res[0])),
            "roofline": {"bound": "alu", "achieved": m_ach, "peak": peak_, "unit": "TFLOP/s",
                         "frac": m_ach / peak_, "kernel": f"pass {mdom} ({mpasses[mdom].terms} points)",
                         "kernel_ms": m_dom_ms, "fp64_inst_per_point": mf + ma,
                         "pipe_frac": mpasses[mdom].terms * (mf + ma) / (m_dom_ms * 1e-3)
                                      / (SM_COUNT * FP64_FMA_PER_SM_CLK * mhz_ * 1e6)},
            "step_ms_all": [round(t, 4) for t in m_times],
        }
        mplan.close()

    # collapse leg (SG_METHOD_COLLAPSE): the same integral as a per-coordinate
    # polynomial product in the level budget, O(d L^2) dd work and no points (not sharded: rank 0
    # emits the value, the other ranks a zero partial; the all-gather + finalize are unchanged)
    collapse = None
    if not args.no_collapse:
        cplan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=rank, world=world,
                         device=dev, method=api.METHOD_COLLAPSE)
        for _ in range(args.warmup):
            step(cplan)
        torch.cuda.synchronize(dev)
        c_times = []
        for _ in range(args.steps):
            flush.fill_(1.0)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step(cplan)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            c_ms_i = e0.elapsed_time(e1)
            if world > 1:
                t = torch.tensor([c_ms_i], dtype=torch.float64,
                                 device=dev if args.dist_backend == "nccl" else "cpu")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                c_ms_i = float(t.item())
            c_times.append(c_ms_i)
        c_res = result.cpu().numpy()
        c_ms = statistics.mean(c_times)
        collapse = {
            "time_to_integral_ms": c_ms, "eq26_points_per_s": total_pts / (c_ms * 1e-3),
            "speedup_vs_combination": ms / c_ms, "result": float(c_res[0]),
            "rel_diff_vs_combination": abs((float(c_res[0]) + float(c_res[1]))
                                           - (float(value_res[0]) + float(value_res[1])))
                                       / abs(float(value_res[0])),
            "work": f"d*(L+1) = {p.d * (p.L + 1)} level sums + d truncated polynomial products "
                    f"of degree {p.L} (dd); launch-latency bound",
            "step_ms_all": [round(t, 4) for t in c_times],
        }
        cplan.close()

    # frontier leg: the same workload with the last two levels NOT fused (SG_B200_NOFUSE=1), so the
    # frontier kernel k_pass<., WRITE> materialises the deepest frontier (config 5: 119 M records,
    # 4.3 GB) — the HBM-bound step of the level-synchronous design that the default fused path
    # avoids.  Reports that launch's HBM bytes / time against MEASURED_PEAKS.json hbm_gbs.
    frontier = None
    if not args.no_frontier:
        os.environ["SG_B200_NOFUSE"] = "1"
        try:
            fplan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=rank, world=world,
                             device=dev)
        finally:
            del os.environ["SG_B200_NOFUSE"]
        fplan.profile_enable(True)
        fpasses = fplan.passes()
        # the pass writing the largest frontier
        wpass = max(range(1, len(fpasses)), key=lambda i: fpasses[i].written) if len(fpasses) > 1 else 0
        for _ in range(min(args.warmup, 2)):
            step(fplan)
        torch.cuda.synchronize(dev)
        f_times, f_kern = timed(lambda: step(fplan), min(args.steps, 3), fplan, wpass)
        rec = (32 if p.kind == S.KIND_OSC else 16) + 4
        wbytes = fpasses[wpass].written * rec
        rbytes = fpasses[wpass - 1].written * rec if wpass >= 1 else 0
        k_ms = statistics.mean(f_kern)
        hbm = None
        try:
            hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        except Exception:
            pass
        gbs = (wbytes + rbytes) / (k_ms * 1e-3) / 1e9
        tfile = os.path.join(ROOT, "profiles", "traffic.json")
        ftraffic = json.load(open(tfile)).get(f"c{args.config}_frontier") if os.path.exists(tfile) else None
        frontier = {"what": f"unfused step; pass {wpass} (k_pass WRITE) writes {fpasses[wpass].written} "
                            f"frontier records of {rec} B and evaluates {fpasses[wpass].terms} points",
                    "step_ms": statistics.mean(f_times), "kernel_ms": k_ms,
                    "algorithmic_bytes": wbytes + rbytes, "achieved_gbs": gbs,
                    "peak_gbs": hbm, "frac": (gbs / hbm) if hbm else None, "traffic": ftraffic}
        fplan.close()

    # plain-SG ablation leg (SG_METHOD_PLAIN): the same integral with every point unranked and
    # evaluated on its own (no dimension iteration) — what the MDI prefix reuse saves on this GPU
    plain = None
    if not args.no_plain:
        pplan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=rank, world=world, device=dev,
                         method=api.METHOD_PLAIN)
        pplan.profile_enable(True)
        step(pplan)
        torch.cuda.synchronize(dev)
        p_times, _ = timed(lambda: step(pplan), 1, pplan, 0)
        p_res = result.cpu().numpy()
        plain = {"what": "every point unranked on the device and its term formed from its t factors "
                         "(the paper's plain SG method), dd accumulation; 1 timed step",
                 "time_to_integral_ms": p_times[0], "value": total_pts / (p_times[0] * 1e-3),
                 "unit": "points/s", "mdi_speedup": p_times[0] / ms,
                 "rel_diff_vs_tree": abs((float(p_res[0]) + float(p_res[1]))
                                         - (float(value_res[0]) + float(value_res[1])))
                                     / abs(float(value_res[0]))}
        pplan.close()

    # corner-peak leg (SG_ARITH_SFORM_DD): the non-separable Genz corner peak on its own workload
    # (sg_configs.corner_config: d=100, L=4, CC), partial sums carried in dd, dd outer function per
    # point; sharded like the headline tree
    corner = None
    if not args.no_corner:
        pc = S.corner_config()
        kplan = api.Plan(pc.d, pc.q, pc.rule, pc.kind, pc.c, pc.w, pc.u, rank=rank, world=world,
                         device=dev, arith=api.ARITH_SFORM_DD)
        kplan.profile_enable(True)
        k_shard, k_total = kplan.points()
        for _ in range(args.warmup):
            step(kplan)
        torch.cuda.synchronize(dev)
        kstep = graph_step(kplan)
        kstep()
        k_times, _ = timed(kstep, args.steps, kplan, 0)
        k_res = result.cpu().numpy()
        k_ms = statistics.mean(k_times)
        corner = {"workload": f"{pc.name}: Genz corner peak (1 + sum c_k x_k)^-(d+1), d={pc.d}, "
                              f"q=d+{pc.L}, {S.RULE_NAMES[pc.rule]}, c~U(0,1) seed 5, sum c = 1",
                  "arith": "s-form double-double (dd partial sums, dd power per point)",
                  "points": k_total, "time_to_integral_ms": k_ms,
                  "value": k_total / (k_ms * 1e-3), "unit": "points/s",
                  "result": float(k_res[0]), "step_ms_all": [round(t, 4) for t in k_times]}
        gfile = os.path.join(ROOT, "tests", "golden", "oracle_full.json")
        if os.path.exists(gfile):
            vals = json.load(open(gfile))["values"]
            if pc.name in vals:
                ref = float(vals[pc.name]["hi"]) + float(vals[pc.name]["lo"])
                corner["rel_err_vs_oracle"] = abs(float(k_res[0]) + float(k_res[1]) - ref) / abs(ref)
        kplan.close()

    # rank-0 report
    if rank == 0:
        peak, mhz = peak_fp64_tflops()
        dom_ms = statistics.mean(dom)
        dom_terms = passes[dominant].terms
        fma_pp, add_pp = plan.leaf_work()
        fpp, ipp = 2 * fma_pp + add_pp, fma_pp + add_pp
        achieved = dom_terms * fpp / (dom_ms * 1e-3) / 1e12
        traffic = None
        tfile = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tfile):
            traffic = json.load(open(tfile)).get(f"c{args.config}")
        parity = parity_block(p, value_res)
        fp64_meas = measure_fp64_peak()
        line = {
            "metric": METRIC, "value": total_pts / (ms * 1e-3), "unit": "points/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "time_to_integral_ms": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(p, {"parallelism": f"dp{world} (depth-1 subtree shards)",
                                       "shard_points_rank0": shard_pts,
                                       "launch": "stream launches" if args.no_graph else
                                       "CUDA-graph replay of sg_integrate (+ sg_finalize)"}),
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": f"pass {dominant} leaf kernel ({dom_terms} points)",
                         "kernel_ms": dom_ms, "flops_per_point": round(fpp, 4),
                         "fp64_inst_per_point": round(ipp, 4),
                         "pipe_frac": dom_terms * ipp / (dom_ms * 1e-3)
                                      / (SM_COUNT * FP64_FMA_PER_SM_CLK * mhz * 1e6),
                         "max_flop_frac_of_mix": fpp / (2 * ipp),
                         "peak_note": f"FP64 peak derived: {SM_COUNT} SMs x {FP64_FMA_PER_SM_CLK} "
                                      f"DFMA/clk x 2 x {mhz:.0f} MHz; measured DFMA burst "
                                      f"{fp64_meas} TFLOP/s"},
            "e2e": {"value": total_pts / (e2e_ms * 1e-3), "unit": "points/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 16, "ms_per_step": e2e_ms},
            # per step: k_factor_base, k_suffix_abs, k_root, one kernel per pass >= 1,
            # k_reduce_fused, k_finalize
            "gpu_launches": (len(passes) - 1 + 5) * args.steps,
            "clocks": clk.summary(),
            "parity": parity,
            "step_ms_all": [round(t, 4) for t in times],
        }
        if merged is not None:
            line["merged"] = merged
        if collapse is not None:
            line["collapse"] = collapse
        if corner is not None:
            line["corner_peak"] = corner
        if frontier is not None:
            line["frontier_kernel"] = frontier
        if plain is not None:
            line["plain_sg"] = plain
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(p)
        print(json.dumps(line), flush=True)
    plan.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def closed_form(p):
    """Exact integral over [0,1]^d of the BASELINE integrands (the closed forms BASELINE.json states),
    40 digits; the Smolyak quadrature error A(q,d)f - I_d f is reported against it."""
    import mpmath as mp
    with mp.workdps(40):
        c = [mp.mpf(float(x)) for x in p.c]
        if p.kind == S.KIND_EXP:
            return mp.fprod([(mp.exp(ck) - 1) / ck if ck != 0 else mp.mpf(1) for ck in c])
        if p.kind == S.KIND_OSC:
            r = mp.expj(2 * mp.pi * mp.mpf(p.u)) * mp.fprod([(mp.expj(ck) - 1) / (1j * ck) for ck in c])
            return mp.re(r)
        w = [mp.mpf(float(x)) for x in p.w]
        if p.kind == S.KIND_PEAK:
            return mp.fprod([ck * (mp.atan(ck * (1 - wk)) + mp.atan(ck * wk)) for ck, wk in zip(c, w)])
        if p.kind == S.KIND_GAUSS:
            return mp.fprod([mp.sqrt(mp.pi) / (2 * ck) * (mp.erf(ck * (1 - wk)) + mp.erf(ck * wk))
                             for ck, wk in zip(c, w)])
    return None


def parity_block(p, res):
    """GPU value against the stored full-size oracle value (tests/golden, written by oracle/ only)
    in 40-digit arithmetic, and the absolute / relative quadrature error against the closed form."""
    import mpmath as mp
    out = {"value": float(res[0])}
    with mp.workdps(40):
        got = mp.mpf(float(res[0])) + mp.mpf(float(res[1]))
        gfile = os.path.join(ROOT, "tests", "golden", "oracle_full.json")
        if os.path.exists(gfile):
            vals = json.load(open(gfile))["values"]
            if p.name in vals:
                ref = mp.mpf(vals[p.name]["text"])
                out.update({"oracle": vals[p.name]["text"],
                            "rel_err_vs_oracle": float(abs((got - ref) / ref)),
                            "gate": 1e-12})
        cf = closed_form(p)
        if cf is not None:
            out.update({"closed_form": mp.nstr(cf, 20), "abs_err_vs_closed_form": float(abs(got - cf)),
                        "rel_err_vs_closed_form": float(abs((got - cf) / cf))})
    return out


def measure_fp64_peak():
    lib_path = os.path.join(ROOT, "tools", "libfp64peak.so")
    try:
        if not os.path.exists(lib_path):
            import subprocess
            subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode",
                                   "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                                   "-Xcompiler", "-fPIC", os.path.join(ROOT, "tools", "fp64_peak.cu"),
                                   "-o", lib_path])
        L = ctypes.CDLL(lib_path)
        L.fp64_peak_tflops.restype = ctypes.c_double
        L.fp64_peak_tflops.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_double)]
        ms = ctypes.c_double()
        return round(L.fp64_peak_tflops(SM_COUNT, 10, 2000, ctypes.byref(ms)), 2)
    except Exception as e:  # report, do not fail the bench
        return f"unavailable: {e}"


def bench_reference(p, args, world):
    """--impl reference: the CPU oracle (oracle/, __float128, OpenMP) as it stands, each step a
    bounded sample of the workload (a fixed depth-1 subtree range)."""
    target = int(4e7)
    lo, hi, npts = oracle_sample_range(p, target)
    for _ in range(args.warmup):
        run_oracle_sample(p, lo, hi)
    secs, pts = [], 0
    for _ in range(args.steps):
        r = run_oracle_sample(p, lo, hi)
        secs.append(r.seconds)
        pts = r.npoints
    ms = statistics.mean(secs) * 1e3
    value = pts / (ms * 1e-3)
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "points/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f128",
        "data": "synthetic",
        "config": config_block(p, {"sample_points_per_step": pts, "sample_range": [lo, hi],
                                   "arith": "__float128, plain Eq 2.6/2.7 point enumeration (oracle/)"}),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "kind": "oracle",
                         "sample": f"{p.name} depth-1 subtrees [{lo},{hi}) = {pts} points per step"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
