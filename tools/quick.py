"""Quick GPU sanity/timing run: per-config relative error vs oracle/DP and CUDA-event time."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import mpmath as mp  # noqa: E402
import torch  # noqa: E402

import pins  # noqa: E402
import sg_configs as S  # noqa: E402
from paper_2210_14313_b200 import api  # noqa: E402

mp.mp.dps = 50


def tp_small(plan):
    return plan.points()[1] < 10 ** 9


def main():
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else "1,2,3,4,5".split(",")
    for i in cfgs:
        # "cp" = the corner-peak workload (non-separable: dd s-form, no DP pin)
        p = S.corner_config() if i == "cp" else S.baseline_config(int(i))
        t0 = time.time()
        plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u,
                        merge=int(os.environ.get("QUICK_MERGE", "0")),
                        method=int(os.environ.get("QUICK_METHOD", "0")),
                        arith=int(os.environ.get("QUICK_ARITH", "0")))
        tplan = time.time() - t0
        hi, lo = plan.integrate_host()
        if p.kind == S.KIND_CORNER:
            err = mp.nan
        else:
            dp = pins.dp_value(p)
            err = abs((mp.mpf(hi) + mp.mpf(lo) - dp) / dp)
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        times = []
        plan.profile_enable(True)
        for _ in range(5):
            ev0.record()
            plan.sg_integrate()
            ev1.record()
            torch.cuda.synchronize()
            times.append(ev0.elapsed_time(ev1))
        prof = plan.profile_read()
        ms = min(times)
        if tp_small(plan):
            g = plan.capture_graph()
            gt = []
            for _ in range(10):
                ev0.record()
                g.replay()
                ev1.record()
                torch.cuda.synchronize()
                gt.append(ev0.elapsed_time(ev1))
            print(f"   cuda-graph step (integrate+finalize): min {min(gt):.4f} ms")
        print(f"   launches(ms): {[round(x, 4) for x in prof]}  all={[round(x, 3) for x in times]}")
        sp, tp = plan.points()
        print(f"{p.name}: value={hi!r} rel_err_vs_DP={float(err):.3e} plan={tplan*1e3:.1f}ms "
              f"integrate={ms:.3f}ms points={tp} -> {tp / (ms * 1e-3):.3e} pts/s "
              f"ws={plan.workspace_bytes/1e9:.3f}GB passes={[(x.terms, x.written) for x in plan.passes()]}",
              flush=True)
        plan.close()


if __name__ == "__main__":
    main()
