"""bench.py — Smolyak points/s and time-to-integral (FP64) of the B200 hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N ...      (one rank per GPU, NCCL)

Workload (headline): BASELINE.json configs[4] — d=300, q=d+4, Clenshaw-Curtis, oscillatory Genz
integrand (seed 4), 27,521,113,876 Smolyak points: the configuration BASELINE.json ties to the
1/2/4/8-GPU scaling run; it fits one GPU.  A step = the whole hot path:
K0 factor tables, root pass, all prefix-tree passes, deterministic reduction, the cross-rank
all-gather + fixed-order finalize.  Rank r evaluates its shard of depth-1 subtrees (strong scaling:
the integral is fixed, the work is split).  Inputs (integrand parameters) are device-resident at
the start of the timed region; L2 is flushed (256 MiB write) between timed steps, outside the
events.  Times: CUDA events on the launching stream, barrier + synchronize on both sides, max over
ranks.  The "e2e" leg times the same step through the C ABI with HOST buffers: pinned H2D of the
parameters (sg_update_integrand), the step, and the D2H read of the 16-byte result.

The "configs" block repeats the measurement for every BASELINE config c1-c5 (Eq 2.6 over each config,
PAPER.md:65-75): sg_plan time, time-to-integral best / median / mean, points/s, relative error against
the stored __float128 oracle value (tests/golden, written by oracle/ only) and, for c3-c5, the FP64
fraction of the dominant leaf kernel.  FP64 work per point comes from the ncu counters committed in
profiles/ (sm__sass_thread_inst_executed_op_{dfma,dadd,dmul}_pred_on of that launch).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import sg_configs as S  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
# FP64 peak derived from the unit count and clock: 148 SMs x 64 FP64 FMA/clk x 2 flops
# x 1.965 GHz (MEASURED_PEAKS.json sm_max_mhz) = 37.2 TFLOP/s.  MEASURED_PEAKS.json has no FP64 figure;
# the DFMA burst measured in this run (tools/fp64_peak.cu) is reported beside it.
SM_COUNT = 148
FP64_FMA_PER_SM_CLK = 64
COUNTERS = os.path.join(ROOT, "profiles", "fp64_counters.json")   # written by tools/fp64_counters.py
GOLDEN = os.path.join(ROOT, "tests", "golden", "oracle_full.json")


def peak_fp64_tflops():
    mhz = 1965.0
    try:
        mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
    except Exception:
        pass
    return SM_COUNT * FP64_FMA_PER_SM_CLK * 2 * mhz * 1e6 / 1e12, mhz


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or platform.machine()


def stats(times):
    return {"best": min(times), "median": statistics.median(times), "mean": statistics.mean(times)}


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
# CPU oracle (cpu_baseline and --impl reference): oracle/ only, never the product library
# ----------------------------------------------------------------------------------------------
def oracle_sample(p, target_points, fp64=False):
    import oracle
    # all host cores, explicitly: torchrun sets OMP_NUM_THREADS=1 for its ranks
    return oracle.timing_sample(p, int(target_points), nthreads=os.cpu_count(), fp64=fp64)


def sample_text(p, r, stride, total, what):
    return (f"{p.name}: every {stride}-th depth-2 multi-index subtree of the whole tree (lexicographic, "
            f"oracle.timing_sample) = {r.npoints} of {total} Smolyak points, {what}, eval_mode=1 "
            f"(active-coordinate form), OpenMP {os.cpu_count()} threads, {r.seconds:.2f} s")


def cpu_baseline(p, target_points=int(6e7)):
    r, stride, total = oracle_sample(p, target_points)
    return {"value": r.npoints / r.seconds, "unit": "points/s", "cores": os.cpu_count(),
            "cpu": cpu_model(), "kind": "oracle",
            "sample": sample_text(p, r, stride, total, "__float128 oracle"),
            "seconds": r.seconds, "points": r.npoints}


def cpu_baseline_fp64(full_configs=(1, 2, 3, 4), sample_config=5, target_points=int(1e9)):
    """The FP64 instantiation of the same plain oracle (oracle/sg_oracle.c -DSGO_FP64): a CPU speed
    baseline that is not parity-grade; its error against the stored quad value shows the
    conditioning of Eq 2.6.  Full size for c1-c4, a sample for c5 (its full-size
    error is committed in profiles/ by tools/oracle_fp64.py)."""
    import mpmath as mp
    import oracle
    gold = json.load(open(GOLDEN))["values"] if os.path.exists(GOLDEN) else {}
    rows = {}
    with mp.workdps(40):
        for i in full_configs:
            p = S.baseline_config(i)
            r = oracle.integrate_problem(p, eval_mode=1, nthreads=os.cpu_count(), fp64=True)
            row = {"points": r.npoints, "seconds": r.seconds, "points_per_s": r.npoints / max(r.seconds, 1e-9)}
            if p.name in gold:
                ref = mp.mpf(gold[p.name]["text"])
                row["rel_err_vs_quad_oracle"] = float(abs((mp.mpf(r.hi) + mp.mpf(r.lo) - ref) / ref))
            rows[p.name] = row
    p = S.baseline_config(sample_config)
    r, stride, total = oracle_sample(p, target_points, fp64=True)
    rows[p.name] = {"points": r.npoints, "seconds": r.seconds, "points_per_s": r.npoints / r.seconds,
                    "sample": sample_text(p, r, stride, total, "FP64 oracle")}
    committed = os.path.join(ROOT, "profiles", "r02_oracle_fp64_container.json")
    if os.path.exists(committed):
        c = json.load(open(committed))["configs"].get(p.name)
        if c:
            rows[p.name]["full_size_rel_err_vs_quad_oracle"] = c["rel_err_vs_quad_oracle"]
            rows[p.name]["full_size_note"] = "profiles/r02_oracle_fp64_container.json (tools/oracle_fp64.py)"
    return {"kind": "oracle (FP64 instantiation, not parity-grade)", "cores": os.cpu_count(),
            "cpu": cpu_model(), "configs": rows}


# ----------------------------------------------------------------------------------------------
def fp64_counters(cfg, variant="tree"):
    """Committed ncu FP64 counters of config `cfg`'s dominant leaf launch (tools/fp64_counters.py)."""
    if not os.path.exists(COUNTERS):
        return None
    return json.load(open(COUNTERS)).get("launches", {}).get(f"c{cfg}_{variant}")


def roofline_from(points, kernel_ms, ctr, plan, peak, mhz, burst):
    """achieved FP64 FLOP/s of the dominant launch: points x (flops per point from the committed ncu
    counters of that launch; the plan's inner-loop count if none) / its live CUDA-event time."""
    if ctr is not None and ctr.get("points") == points:
        fpp, ipp = ctr["flops_per_point"], ctr["fp64_inst_per_point"]
        src = f"ncu counters {ctr['source']}"
    else:
        fma, add = plan.leaf_work()
        fpp, ipp = 2 * fma + add, fma + add
        src = "sg_plan_leaf_work (inner loop only; no committed ncu counters for this launch)"
    ach = points * fpp / (kernel_ms * 1e-3) / 1e12
    out = {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
           "flops_per_point": round(fpp, 4), "fp64_inst_per_point": round(ipp, 4),
           "work_source": src, "kernel_ms": kernel_ms,
           "pipe_frac": points * ipp / (kernel_ms * 1e-3) / (SM_COUNT * FP64_FMA_PER_SM_CLK * mhz * 1e6)}
    if isinstance(burst, (int, float)) and burst > 0:
        out["frac_of_measured_dfma_burst"] = ach / burst
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config block (c1-c5)")
    ap.add_argument("--no-merged", action="store_true", help="skip the SG_MERGE_MIDPOINT leg")
    ap.add_argument("--no-graph", action="store_true",
                    help="time the stream-launched step instead of its CUDA-graph replay")
    ap.add_argument("--no-collapse", action="store_true", help="skip the SG_METHOD_COLLAPSE leg")
    ap.add_argument("--no-frontier", action="store_true",
                    help="skip the stored-frontier (unfused) leg that measures the HBM-bound frontier kernel")
    ap.add_argument("--plain-ablation", action="store_true",
                    help="also run the plain per-point SG ablation leg (SG_METHOD_PLAIN: the paper's "
                         "comparison system, out of the hot-path scope; off by default)")
    ap.add_argument("--no-corner", action="store_true",
                    help="skip the non-separable corner-peak leg (SG_ARITH_SFORM_DD)")
    # testing aids for the multi-rank path on a 1-GPU box: gloo carries the 16-byte collective
    # through host memory and every rank may share one device (ranks never wait on each other
    # inside a kernel, so sharing is safe); the product configuration is nccl + one GPU per rank
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--device-index", type=int, default=None)
    ap.add_argument("--force-dist", action="store_true",
                    help="initialise the process group and run the all-gather even at world 1 "
                         "(exercises the NCCL branch on a 1-GPU box)")
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
    dist_on = world > 1 or args.force_dist
    if dist_on:
        if args.dist_backend == "nccl":
            # NCCL's init lines (nRanks, NVLS / ring setup) on stderr, so a multi-GPU record can confirm
            # the communicator; the JSON line stays the only stdout line of rank 0
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        dist.barrier()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    gathered = torch.zeros(2 * world, dtype=torch.float64, device=dev)
    result = torch.zeros(2, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def make_plan(q, **kw):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        pl = api.Plan(q.d, q.q, q.rule, q.kind, q.c, q.w, q.u, rank=rank, world=world, device=dev, **kw)
        torch.cuda.synchronize(dev)
        return pl, (time.perf_counter() - t0) * 1e3

    def gather_finalize(plan, part):
        if args.dist_backend == "nccl":
            dist.all_gather_into_tensor(gathered, part)
        else:
            g = torch.zeros(2 * world, dtype=torch.float64)
            dist.all_gather_into_tensor(g, part.cpu())
            gathered.copy_(g)
        plan.sg_finalize(gathered, world, stream, result)

    def step(plan):
        part = plan.sg_integrate(stream)
        if dist_on:
            gather_finalize(plan, part)
        else:
            plan.sg_finalize(part, 1, stream, result)

    def graph_step(plan, prof=2):
        """The step as one CUDA-graph replay (sg_integrate, + sg_finalize at world 1); with prof = 2
        the dominant pass's launch is bracketed by two graph event-record nodes (profile_read times it
        on every replay), with 0 the step has no event nodes; with a process group the all-gather and
        sg_finalize follow the replay as in step()."""
        if args.no_graph:
            return lambda: step(plan)
        plan.profile_enable(prof)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            part = plan.sg_integrate()
            if not dist_on:
                plan.sg_finalize(part, 1, None, result)

        def fn():
            g.replay()
            if dist_on:
                gather_finalize(plan, part)
        fn.graph = g
        return fn

    def maxrank(ms):
        if not dist_on:
            return ms
        t = torch.tensor([ms], dtype=torch.float64, device=dev if args.dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, k, plan=None, dominant=None):
        times, dom = [], []
        for _ in range(k):
            flush.fill_(1.0)
            if dist_on:
                dist.barrier()
            torch.cuda.synchronize(dev)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            times.append(maxrank(e0.elapsed_time(e1)))
            if plan is not None and dominant is not None:
                prof = plan.profile_read()
                dom.append(prof[3 + dominant - 1] if dominant > 0 else prof[2])
        return times, dom

    def dominant_pass(plan):
        passes = plan.passes()
        return (max(range(1, len(passes)), key=lambda i: passes[i].terms) if len(passes) > 1 else 0), passes

    def measure(q, k, w, prof=2, **kw):
        """plan + warm-up + k timed graph replays of problem q (prof = 2: the dominant pass timed
        inside the replays; 0: no event nodes, and no kernel time)."""
        plan, plan_ms = make_plan(q, **kw)
        plan.profile_enable(prof)
        dom, passes = dominant_pass(plan)
        for _ in range(w):
            step(plan)
        torch.cuda.synchronize(dev)
        g = graph_step(plan, prof)
        for _ in range(w):
            g()
        torch.cuda.synchronize(dev)
        times, dom_ms = timed(g, k, plan, dom if prof else None)
        res = result.cpu().numpy().copy()
        return plan, plan_ms, dom, passes, times, dom_ms, res, g

    peak, mhz = peak_fp64_tflops()

    # ---- headline config -------------------------------------------------------------------------
    plan, plan_ms, dominant, passes, _, _, _, gstep = measure(p, 0, args.warmup)
    shard_pts, total_pts = plan.points()
    with ClockSampler(local) as clk:
        times, dom = timed(gstep, args.steps, plan, dominant)
    st = stats(times)
    ms = st["mean"]
    value_res = result.cpu().numpy().copy()

    # e2e: host buffers through the C ABI (pinned H2D of c/w, step, D2H of the result)
    c_host = torch.from_numpy(p.c.copy()).pin_memory()
    w_host = torch.from_numpy(p.w.copy()).pin_memory() if p.w is not None else None
    res_host = torch.zeros(2, dtype=torch.float64).pin_memory()

    def e2e_step():
        plan.sg_update_integrand(c_host, w_host, p.u, stream)
        step(plan)
        res_host.copy_(result, non_blocking=True)

    for _ in range(2):
        e2e_step()
    e2e_times, _ = timed(e2e_step, args.steps)
    e2e_ms = statistics.mean(e2e_times)
    h2d = 8 * p.d * (2 if p.w is not None else 1) + 8

    # ---- every BASELINE config (c1-c5) -----------------------------------------------------------
    configs = None
    if not args.no_configs:
        configs = {}
        for i in range(1, 6):
            q = S.baseline_config(i)
            if i == args.config:
                cplan, c_plan_ms, cdom, cpasses, ctimes, cdom_ms, cres = (plan, plan_ms, dominant, passes,
                                                                          times, dom, value_res)
            else:
                cplan, c_plan_ms, cdom, cpasses, ctimes, cdom_ms, cres, _ = measure(q, args.steps, args.warmup,
                                                                                prof=2 if i >= 3 else 0)
            cst = stats(ctimes)
            npts = cplan.points()[1]
            row = {"d": q.d, "q": q.q, "rule": S.RULE_NAMES[q.rule], "integrand": S.KIND_NAMES[q.kind],
                   "points": npts, "plan_ms": c_plan_ms, "time_to_integral_ms": cst,
                   "points_per_s": npts / (cst["mean"] * 1e-3), "points_per_s_best": npts / (cst["best"] * 1e-3),
                   "parity": parity_block(q, cres, brief=True)}
            if i >= 3 and cdom > 0:
                row["dominant_kernel"] = roofline_from(cpasses[cdom].terms, statistics.mean(cdom_ms),
                                                       fp64_counters(i), cplan, peak, mhz, None)
                row["dominant_kernel"]["points"] = cpasses[cdom].terms
            configs[q.name] = row
            if cplan is not plan:
                cplan.close()

    # merged leg (SG_MERGE_MIDPOINT): the same integral with the midpoint copies of
    # every point summed into merged coefficients, each remaining point evaluated once
    merged = None
    if not args.no_merged:
        mplan, _, mdom, mpasses, m_times, m_dom, m_res, _ = measure(p, args.steps, args.warmup,
                                                                    merge=api.MERGE_MIDPOINT)
        m_total = mplan.points()[1]
        mst = stats(m_times)
        merged = {
            "time_to_integral_ms": mst["mean"], "time_to_integral_stats_ms": mst, "points": m_total,
            "value": m_total / (mst["mean"] * 1e-3), "unit": "points/s",
            "eq26_points_per_s": total_pts / (mst["mean"] * 1e-3),
            "speedup_vs_combination": ms / mst["mean"], "result": float(m_res[0]),
            "rel_diff_vs_combination": abs((float(m_res[0]) + float(m_res[1]))
                                           - (float(value_res[0]) + float(value_res[1])))
                                       / abs(float(value_res[0])),
            "roofline": roofline_from(mpasses[mdom].terms, statistics.mean(m_dom),
                                      fp64_counters(args.config, "merged"), mplan, peak, mhz, None),
            "step_ms_all": [round(t, 4) for t in m_times],
        }
        mplan.close()

    # collapse leg (SG_METHOD_COLLAPSE): the same integral as a per-coordinate
    # polynomial product in the level budget, O(d L^2) dd work and no points (not sharded: rank 0
    # emits the value, the other ranks a zero partial; the all-gather + finalize are unchanged)
    collapse = None
    if not args.no_collapse:
        cplan, _ = make_plan(p, method=api.METHOD_COLLAPSE)
        for _ in range(args.warmup):
            step(cplan)
        torch.cuda.synchronize(dev)
        c_times, _ = timed(lambda: step(cplan), args.steps)
        c_res = result.cpu().numpy()
        c_ms = statistics.mean(c_times)
        collapse = {
            "time_to_integral_ms": c_ms, "time_to_integral_stats_ms": stats(c_times),
            "eq26_points_per_s": total_pts / (c_ms * 1e-3),
            "speedup_vs_combination": ms / c_ms, "result": float(c_res[0]),
            "rel_diff_vs_combination": abs((float(c_res[0]) + float(c_res[1]))
                                           - (float(value_res[0]) + float(value_res[1])))
                                       / abs(float(value_res[0])),
            "work": f"d*(L+1) = {p.d * (p.L + 1)} level sums + d truncated polynomial products "
                    f"of degree {p.L} (dd); launch-latency bound",
        }
        cplan.close()

    # frontier leg: the same workload with the last two levels NOT fused (SG_B200_NOFUSE=1), so the
    # frontier kernel k_pass<., WRITE> materialises the deepest frontier (config 5: 119 M records,
    # 4.3 GB) — the HBM-bound step of the level-synchronous design that the default fused path
    # avoids.  Reports that launch's HBM bytes / time against MEASURED_PEAKS.json hbm_gbs.
    frontier = None
    if not args.no_frontier:
        # the deepest frontier pass is split (sg_kernels.cu): k_front stores the 4.3 GB of records
        # (HBM-bound, its own interval here: the serial split order) and k_leaf evaluates the other
        # children after it
        os.environ["SG_B200_NOFUSE"] = "1"
        os.environ["SG_B200_SPLIT_SERIAL"] = "1"
        try:
            fplan, _ = make_plan(p)
        finally:
            del os.environ["SG_B200_NOFUSE"]
            del os.environ["SG_B200_SPLIT_SERIAL"]
        fplan.profile_enable(True)
        fpasses = fplan.passes()
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
        frontier = {"what": f"unfused step; pass {wpass}'s write-only frontier kernel k_front writes "
                            f"{fpasses[wpass].written} frontier records of {rec} B (and accumulates their "
                            f"terms; the pass's other children, {fpasses[wpass].terms} points in all, "
                            f"follow in the leaf-only k_leaf)",
                    "step_ms": statistics.mean(f_times), "kernel_ms": k_ms,
                    "algorithmic_bytes": wbytes + rbytes, "achieved_gbs": gbs,
                    "peak_gbs": hbm, "frac": (gbs / hbm) if hbm else None, "traffic": ftraffic}
        fplan.close()

    # plain-SG ablation leg (opt-in; SG_METHOD_PLAIN): the paper's comparison system on the GPU
    plain = None
    if args.plain_ablation:
        pplan, _ = make_plan(p, method=api.METHOD_PLAIN)
        step(pplan)
        torch.cuda.synchronize(dev)
        p_times, _ = timed(lambda: step(pplan), 1)
        p_res = result.cpu().numpy()
        plain = {"what": "opt-in ablation (comparison system, out of the hot-path scope): every point "
                         "unranked on the device and its term formed from its t factors, dd "
                         "accumulation; 1 timed step",
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
        kplan, _, _, _, k_times, _, k_res, _ = measure(pc, args.steps, args.warmup, arith=api.ARITH_SFORM_DD)
        k_total = kplan.points()[1]
        kst = stats(k_times)
        corner = {"workload": f"{pc.name}: Genz corner peak (1 + sum c_k x_k)^-(d+1), d={pc.d}, "
                              f"q=d+{pc.L}, {S.RULE_NAMES[pc.rule]}, c~U(0,1) seed 5, sum c = 1",
                  "arith": "s-form double-double (dd partial sums, dd power per point)",
                  "points": k_total, "time_to_integral_ms": kst["mean"], "time_to_integral_stats_ms": kst,
                  "value": k_total / (kst["mean"] * 1e-3), "unit": "points/s",
                  "result": float(k_res[0])}
        if os.path.exists(GOLDEN):
            vals = json.load(open(GOLDEN))["values"]
            if pc.name in vals:
                ref = float(vals[pc.name]["hi"]) + float(vals[pc.name]["lo"])
                corner["rel_err_vs_oracle"] = abs(float(k_res[0]) + float(k_res[1]) - ref) / abs(ref)
        kplan.close()

    # rank-0 report
    if rank == 0:
        with ClockSampler(local) as bclk:
            fp64_meas = measure_fp64_peak()
        dom_ms = statistics.mean(dom)
        dom_terms = passes[dominant].terms
        roof = roofline_from(dom_terms, dom_ms, fp64_counters(args.config), plan, peak, mhz,
                             fp64_meas if isinstance(fp64_meas, float) else None)
        traffic = None
        tfile = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tfile):
            traffic = json.load(open(tfile)).get(f"c{args.config}")
        roof.update({"traffic": traffic, "kernel": f"pass {dominant} leaf kernel ({dom_terms} points)",
                     "max_flop_frac_of_mix": roof["flops_per_point"] / (2 * roof["fp64_inst_per_point"]),
                     "peak_note": f"FP64 peak derived: {SM_COUNT} SMs x {FP64_FMA_PER_SM_CLK} DFMA/clk x 2 x "
                                  f"{mhz:.0f} MHz (MEASURED_PEAKS.json has no FP64 entry); measured DFMA "
                                  f"burst {fp64_meas} TFLOP/s (tools/fp64_peak.cu, clocks in "
                                  f"roofline.burst_clocks)",
                     "burst_tflops": fp64_meas, "burst_clocks": bclk.summary(),
                     "flops_note": "flops per point = (2 DFMA + DADD + DMUL) thread-instructions of this "
                                   "launch / its points (ncu counters, profiles/fp64_counters.json); "
                                   "DESIGN.md §6 explains why SURVEY.md §8d's textbook-dd 68 flops per "
                                   "point are not this kernel's work"})
        line = {
            "metric": METRIC, "value": total_pts / (ms * 1e-3), "unit": "points/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "time_to_integral_ms": ms, "time_to_integral_stats_ms": st,
            "points_per_s_best": total_pts / (st["best"] * 1e-3),
            "plan_ms": plan_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_block(p, total_pts, {
                "parallelism": f"dp{world} (depth-1 subtree shards)", "shard_points_rank0": shard_pts,
                "collective": ("nccl all_gather_into_tensor" if dist_on and args.dist_backend == "nccl"
                               else "gloo (test aid)" if dist_on else "none (world 1)"),
                "process_group": ({"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                                   "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))
                                   if args.dist_backend == "nccl" else None} if dist_on else None),
                "launch": "stream launches" if args.no_graph else
                          "CUDA-graph replay of sg_integrate (+ sg_finalize)"}),
            "roofline": roof,
            "e2e": {"value": total_pts / (e2e_ms * 1e-3), "unit": "points/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 16, "ms_per_step": e2e_ms},
            # per step: k_head (d <= 2048; else k_factor_base, k_suffix_abs, k_root), one kernel per
            # pass >= 1, k_reduce_fused, k_finalize
            "gpu_launches": ((1 if p.d <= 2048 else 3) + (len(passes) - 1) + 2) * args.steps,
            "clocks": clk.summary(),
            "parity": parity_block(p, value_res),
            "step_ms_all": [round(t, 4) for t in times],
        }
        if configs is not None:
            line["configs"] = configs
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
            line["cpu_baseline_fp64"] = cpu_baseline_fp64()
        print(json.dumps(line), flush=True)
    plan.close()
    if dist_on:
        dist.barrier()
        dist.destroy_process_group()


def config_block(p, total_points, extra=None):
    c = {"workload": f"BASELINE.json configs[{int(p.name[1:]) - 1}] ({p.name}): d={p.d}, "
                     f"q=d+{p.L}, {S.RULE_NAMES[p.rule]}, {S.KIND_NAMES[p.kind]} integrand",
         "d": p.d, "q": p.q, "L": p.L, "rule": S.RULE_NAMES[p.rule],
         "integrand": S.KIND_NAMES[p.kind], "points": total_points,
         "form": "combination (Eq 2.6)", "arith": "factor-form double-double",
         "l2": "flushed between timed steps (256 MiB write, outside the events)"}
    if extra:
        c.update(extra)
    return c


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


def parity_block(p, res, brief=False):
    """GPU value against the stored full-size oracle value (tests/golden, written by oracle/ only)
    in 40-digit arithmetic, and the absolute / relative quadrature error against the closed form."""
    import mpmath as mp
    out = {"value": float(res[0])}
    with mp.workdps(40):
        got = mp.mpf(float(res[0])) + mp.mpf(float(res[1]))
        if os.path.exists(GOLDEN):
            vals = json.load(open(GOLDEN))["values"]
            if p.name in vals:
                ref = mp.mpf(vals[p.name]["text"])
                if not brief:
                    out["oracle"] = vals[p.name]["text"]
                out.update({"rel_err_vs_oracle": float(abs((got - ref) / ref)), "gate": 1e-12})
        cf = closed_form(p)
        if cf is not None:
            if not brief:
                out["closed_form"] = mp.nstr(cf, 20)
            out.update({"abs_err_vs_closed_form": float(abs(got - cf)),
                        "rel_err_vs_closed_form": float(abs((got - cf) / cf))})
    return out


def measure_fp64_peak():
    lib_path = os.path.join(ROOT, "tools", "libfp64peak.so")
    try:
        if not os.path.exists(lib_path):
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
    """--impl reference: the CPU oracle (oracle/, __float128, OpenMP) as it stands on the box's host
    cores, each step the same bounded sample of the workload (every s-th depth-2 multi-index subtree
    of the whole tree, oracle.timing_sample).  Loads only oracle/ (never the product library)."""
    import oracle
    target = int(1e7)
    total = oracle.n_points(p)
    r0, stride, _ = oracle_sample(p, target)
    for _ in range(max(0, args.warmup - 1)):
        oracle.integrate_problem(p, stride=stride, include_root=False, eval_mode=1, nthreads=os.cpu_count())
    secs, pts = [], r0.npoints
    for _ in range(args.steps):
        r = oracle.integrate_problem(p, stride=stride, include_root=False, eval_mode=1, nthreads=os.cpu_count())
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
        "config": config_block(p, total, {"sample_points_per_step": pts, "sample_stride": stride,
                                          "arith": "__float128, plain Eq 2.6/2.7 point enumeration (oracle/)"}),
        "cpu_baseline": {"value": value, "unit": "points/s", "cores": cores, "cpu": cpu_model(),
                         "kind": "oracle", "sample": sample_text(p, r0, stride, total, "__float128 oracle")
                         + " per step"},
        "e2e": {"value": value, "unit": "points/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
