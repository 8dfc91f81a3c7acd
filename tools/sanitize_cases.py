"""Small problems for compute-sanitizer (memcheck / racecheck / synccheck / initcheck), each checked
against the __float128 oracle at the 1e-12 gate:

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py

Cases cover every kernel family of the hot path: K0 factor tables + suffix bounds, root, frontier
writer k_pass, generic k_leaf, fused k_leaf2 (real and oscillatory NJ = 3, NJ = 2 GL), k_leaf2_sym3
with source tasks (atomic task counters), the merged k_leaf2_pairs, the last-block-ticket reduction
k_reduce_fused, k_finalize, the collapse and the dd s-form, whole and sharded (world 3)."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import mpmath as mp  # noqa: E402

import oracle  # noqa: E402
import sg_configs as S  # noqa: E402


def main():
    from paper_2210_14313_b200 import api
    mp.mp.dps = 40
    cases = [
        (S.baseline_config(1), {}, "c1 tree"),
        (S.baseline_config(2), {}, "c2 tree (k_leaf2_sym3 + source tasks)"),
        (S.random_problem(61, 40, 3, S.RULE_CC, S.KIND_OSC), {}, "osc d=40 L=3 fused + source tasks"),
        (S.random_problem(62, 30, 4, S.RULE_CC, S.KIND_GAUSS), {}, "gauss d=30 L=4 fused k_leaf2 real"),
        (S.random_problem(63, 25, 4, S.RULE_GL, S.KIND_PEAK), {}, "peak d=25 L=4 GL (NJ=2)"),
        (S.random_problem(64, 12, 5, S.RULE_CC, S.KIND_EXP), {}, "exp d=12 L=5"),
        (S.random_problem(65, 20, 4, S.RULE_CC, S.KIND_OSC), {"merge": api.MERGE_MIDPOINT}, "merged osc"),
        (S.random_problem(66, 20, 4, S.RULE_CC, S.KIND_OSC), {"method": api.METHOD_COLLAPSE}, "collapse"),
        (S.random_problem(67, 8, 4, S.RULE_CC, S.KIND_CORNER), {"arith": api.ARITH_SFORM_DD}, "s-form dd"),
    ]
    if os.environ.get("SG_SANITIZE_NOFUSE") != "0":
        cases.append((S.random_problem(68, 30, 4, S.RULE_CC, S.KIND_OSC), {"_nofuse": True},
                      "unfused (k_pass WRITE + k_leaf1)"))
    worst = 0.0
    for p, kw, what in cases:
        ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
        worlds = [1, 3] if "method" not in kw and "arith" not in kw else [1]
        for world in worlds:
            kw2 = {k: v for k, v in kw.items() if not k.startswith("_")}
            if kw.get("_nofuse"):
                os.environ["SG_B200_NOFUSE"] = "1"
            try:
                acc = mp.mpf(0)
                for rank in range(world):
                    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=rank, world=world, **kw2)
                    hi, lo = plan.integrate_host()
                    plan.close()
                    acc += mp.mpf(hi) + mp.mpf(lo)
            finally:
                os.environ.pop("SG_B200_NOFUSE", None)
            err = float(abs((acc - ref) / ref))
            worst = max(worst, err)
            print(f"{what:45s} world={world}: rel_err={err:.3e}", flush=True)
            assert err <= 1e-12, (what, world, err)
    print(f"SANITIZE_CASES_OK worst={worst:.3e}")


if __name__ == "__main__":
    main()
