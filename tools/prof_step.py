"""Minimal driver for ncu: plan one BASELINE config and run `steps` hot-path steps.

    python tools/prof_step.py <config> [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import sg_configs as S  # noqa: E402
from paper_2210_14313_b200 import api  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "5"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    p = S.corner_config() if cfg == "cp" else S.baseline_config(int(cfg))
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u,
                    merge=int(os.environ.get("QUICK_MERGE", "0")),
                    method=int(os.environ.get("QUICK_METHOD", "0")),
                    arith=int(os.environ.get("QUICK_ARITH", "0")),
                    rank=int(os.environ.get("QUICK_RANK", "0")), world=int(os.environ.get("QUICK_WORLD", "1")))
    for _ in range(steps):
        out = plan.sg_integrate()
        plan.sg_finalize(out, 1)
    torch.cuda.synchronize()
    print(p.name, plan.sg_finalize(out, 1).cpu().numpy())
    plan.close()


if __name__ == "__main__":
    main()
