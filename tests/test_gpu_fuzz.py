"""Seeded random sweep: every evaluation mode of the C ABI against the __float128 oracle.

60 small problems drawn from one seeded generator: dimension 1-40, level budget 0-7 (capped so the
oracle enumerates at most 2e5 points), all four rules, all five integrand kinds, and for each a
mode chosen among the every-point tree (combination and delta forms), the midpoint-merged tree,
the separable collapse and the double-double s-form (the corner peak only has the s-form).
Gate: 1e-15 relative (the health bound; the north-star gate is 1e-12).
"""
import mpmath as mp
import numpy as np
import pytest

import oracle
import pins
import sg_configs as S
from test_gpu_parity import HEALTH, rel

pytestmark = pytest.mark.gpu

RULES = [S.RULE_TRAP, S.RULE_CC, S.RULE_GP, S.RULE_GL]
KINDS = [S.KIND_EXP, S.KIND_OSC, S.KIND_PEAK, S.KIND_GAUSS, S.KIND_CORNER]
MODES = ["tree", "delta", "merged", "collapse", "sform_dd"]


def _cases(n=60, seed=2024):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        d = int(rng.integers(1, 41))
        L = int(rng.integers(0, 8))
        rule = RULES[int(rng.integers(0, 4))]
        kind = KINDS[int(rng.integers(0, 5))]
        if rule in (S.RULE_CC, S.RULE_TRAP) and L > 6:
            L = 6
        while L > 0 and pins.n_points(rule, d, L) > 200_000:
            L -= 1
        mode = MODES[int(rng.integers(0, 5))]
        if kind == S.KIND_CORNER:
            mode = "sform_dd" if mode != "delta" else "delta"
        if kind == S.KIND_PEAK and mode == "sform_dd":
            mode = "tree"
        out.append((1000 + len(out), d, L, rule, kind, mode))
    return out


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2210_14313_b200 import build as B
    B.build()
    from paper_2210_14313_b200 import api as A
    return A


@pytest.mark.parametrize("seed,d,L,rule,kind,mode", _cases(), ids=lambda v: str(v))
def test_fuzz_vs_oracle(api, seed, d, L, rule, kind, mode):
    p = S.random_problem(seed, d, L, rule, kind)
    kw = {"tree": {}, "delta": {"form": api.FORM_DELTA}, "merged": {"merge": api.MERGE_MIDPOINT},
          "collapse": {"method": api.METHOD_COLLAPSE}, "sform_dd": {"arith": api.ARITH_SFORM_DD}}[mode]
    hi, lo = api.integrate(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u, **kw)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    r = rel(mp.mpf(hi) + mp.mpf(lo), ref)
    assert r <= HEALTH, (p.name, mode, float(r))


def test_fuzz_all_paths_and_switches():
    """tools/fuzz_all.py: 40 seeded cases over every rule, kind, form, merge / collapse / dd s-form,
    shard world and plan switch (split frontier passes, lane groups, unfused, generic leaf, the
    three-launch head) against the oracle at 1e-15 (the 300-case sweep: profiles/r02F_fuzz_all_300.txt)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "fuzz_all.py"), "40", "3"], cwd=root,
                         capture_output=True, text=True, timeout=1200)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-2000:]
    assert "failures=0" in out.stdout
