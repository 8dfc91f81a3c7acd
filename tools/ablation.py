"""Ablation: factor-form dd (product path) vs s-form FP64 (SG_ARITH_SFORM_FP64) on BASELINE configs.
Prints one JSON line per (config, arith): device ms per integrate (best of 5, CUDA events),
points/s and relative error vs the 50-digit generating-function value (tests/pins.py)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import mpmath as mp  # noqa: E402
import torch  # noqa: E402

import pins  # noqa: E402
import sg_configs as S  # noqa: E402
from paper_2210_14313_b200 import api  # noqa: E402

mp.mp.dps = 50


def run(i, arith):
    p = S.baseline_config(i)
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, arith=arith)
    hi, lo = plan.integrate_host()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        e0.record()
        plan.sg_integrate()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    sp, tp = plan.points()
    plan.close()
    dp = pins.dp_value(p)
    err = float(abs((mp.mpf(hi) + mp.mpf(lo) - dp) / dp))
    return {"config": p.name, "arith": ["factor_dd", "sform_fp64"][arith], "ms": best,
            "points_per_s": tp / (best * 1e-3), "rel_err": err}


def main():
    cfgs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,3,4,5").split(",")]
    for i in cfgs:
        for arith in (0, 1):
            if i == 3 and arith == 1:
                continue  # product-peak has no additive argument (s-form unsupported)
            print(json.dumps(run(i, arith)), flush=True)


if __name__ == "__main__":
    main()
