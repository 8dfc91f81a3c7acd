"""Seeded sweep of every evaluation path against the __float128 oracle (health bound 1e-15).

    python tools/fuzz_all.py [n] [seed]

Each case draws a rule, kind, d, L (point count bounded for the oracle), form, merge / method /
arithmetic, a shard world, and one of the plan-time path switches (split frontier passes, forced
k_leaf2 lane groups, unfused last levels, the generic leaf, the three-launch head); prints every case
and the worst relative error, exits non-zero if any case exceeds the bound.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import mpmath as mp  # noqa: E402

mp.mp.dps = 50
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import pins  # noqa: E402
import sg_configs as S  # noqa: E402
from paper_2210_14313_b200 import api  # noqa: E402

SWITCHES = [{}, {"SG_B200_FRONT_SPLIT": "1"}, {"SG_B200_LEAF2_GROUPS": "2"}, {"SG_B200_LEAF2_GROUPS": "4"},
            {"SG_B200_LEAF2_GROUPS": "8"}, {"SG_B200_NOFUSE": "1"}, {"SG_B200_GENERIC_LEAF": "1"},
            {"SG_B200_NOHEAD": "1"}, {"SG_B200_NOFUSE": "1", "SG_B200_FRONT_SPLIT": "1"}]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 11
    rng = np.random.default_rng(seed)
    worst, bad = 0.0, 0
    for i in range(n):
        rule = [S.RULE_CC, S.RULE_GL, S.RULE_TRAP, S.RULE_GP][int(rng.integers(0, 4))]
        kind = int(rng.integers(0, 4))
        L = int(rng.integers(0, 7))
        d = int(rng.integers(1, 160))
        while pins.n_points(rule, d, L) > 2_000_000 and d > 1:
            d = max(1, d * 2 // 3)
        p = S.random_problem(7000 + 97 * seed + i, d, L, rule, kind)
        form = int(rng.integers(0, 2))
        what = int(rng.integers(0, 5))
        kw = {"form": form}
        if what == 1:
            kw["merge"] = api.MERGE_MIDPOINT
        elif what == 2:
            kw["method"] = api.METHOD_COLLAPSE
        elif what == 3 and kind != S.KIND_PEAK:
            kw["arith"] = api.ARITH_SFORM_DD
        world = [1, 1, 2, 3, 8][int(rng.integers(0, 5))] if what != 2 else 1
        env = SWITCHES[int(rng.integers(0, len(SWITCHES)))]
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            tot = mp.mpf(0)
            for r in range(world):
                plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=r, world=world, **kw)
                hi, lo = plan.integrate_host()
                plan.close()
                tot += mp.mpf(hi) + mp.mpf(lo)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
        err = float(abs((tot - ref) / ref)) if ref != 0 else float(abs(tot))
        worst = max(worst, err)
        flag = "" if err <= 1e-15 else "  <-- FAIL"
        bad += err > 1e-15
        print(f"{i:4d} {p.name:28s} form={form} {kw} world={world} env={env} rel_err={err:.2e}{flag}", flush=True)
    print(f"FUZZ_ALL cases={n} worst={worst:.3e} failures={bad}")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
