"""Wider seeded sweep of the k_leaf2_sym3 source-task path against the __float128 oracle.

    python tools/fuzz_src.py [n] [seed]

Oscillatory problems with the symmetric {0, 1/2, 1} level-2 row (Clenshaw-Curtis / trapezoidal,
combination / delta form), random d, L, shard (rank, world) or explicit depth-1 range; prints the
worst relative error (health bound 1e-15).
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


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    worst = 0.0
    for i in range(n):
        rule = [S.RULE_CC, S.RULE_TRAP][int(rng.integers(0, 2))]
        L = int(rng.integers(3, 7))
        d = int(rng.integers(L, 90))
        while pins.n_points(rule, d, L) > 3_000_000 and d > L:
            d -= 7
        d = max(d, L)
        form = int(rng.integers(0, 2))
        p = S.random_problem(5000 + i, d, L, rule, S.KIND_OSC)
        kw = {"form": form}
        mode = int(rng.integers(0, 3)) if form == 0 else 0   # delta-form shards sum differently
        lo, hi = 0, -1
        if mode == 1:
            world = int(rng.integers(2, 9))
            kw.update(rank=int(rng.integers(0, world)), world=world)
            plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, **kw)
            lo, hi, _ = plan.range()
            plan.close()
        elif mode == 2:
            plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, form=form)
            _, _, nd1 = plan.range()
            plan.close()
            a = int(rng.integers(0, nd1))
            b = int(rng.integers(a + 1, min(nd1, a + 40) + 1))
            lo, hi = a, b
            kw.update(range_lo=lo, range_hi=hi)
        plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, **kw)
        v = plan.integrate_host()
        plan.close()
        ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1, lo=lo, hi=hi,
                                              include_root=lo == 0).text)
        got = mp.mpf(v[0]) + mp.mpf(v[1])
        r = float(abs((got - ref) / ref)) if ref != 0 else float(abs(got))
        worst = max(worst, r)
        flag = "" if r <= 1e-15 else "  <-- FAIL"
        print(f"{i:3d} d={d} L={L} rule={rule} form={form} mode={mode} lo={lo} hi={hi} rel={r:.2e}{flag}",
              flush=True)
    print(f"worst {worst:.3e} over {n}")


if __name__ == "__main__":
    main()
