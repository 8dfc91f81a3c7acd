"""GPU parity of the separable collapse (SG_METHOD_COLLAPSE) against the
__float128 oracle (plain Eq 2.6/2.7 point enumeration) on the same seeded inputs.

The collapse evaluates A(q,d)f = Re(B sum_e coef[e] [z^e] prod_k p_k(z)) in double-double without
visiting any point (the symbolic partial function carried per coordinate).
Same 1e-12 gate as the tree (BASELINE.json north_star) and the same 1e-15 health bound; it must also
agree with the tree path to dd rounding.
"""
import json
import os

import mpmath as mp
import numpy as np
import pytest

import oracle
import pins
import sg_configs as S
from test_gpu_parity import CASES, GATE, GOLDEN, HEALTH, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2210_14313_b200 import build as B
    B.build()
    from paper_2210_14313_b200 import api as A
    return A


def collapse_value(api, p, **kw):
    hi, lo = api.integrate(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u, method=api.METHOD_COLLAPSE, **kw)
    return mp.mpf(hi) + mp.mpf(lo)


@pytest.mark.parametrize("i", [1, 2])
def test_collapse_small_baseline_vs_oracle(api, i):
    p = S.baseline_config(i)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    r = rel(collapse_value(api, p), ref)
    assert r <= GATE and r <= HEALTH, float(r)


@pytest.mark.parametrize("i", [3, 4, 5])
def test_collapse_full_size_vs_oracle_golden(api, i):
    """Configs 3-5 at full size: the stored full-size oracle values (oracle/make_golden.py, computed
    by the __float128 oracle only) and the independent 50-digit DP pin."""
    p = S.baseline_config(i)
    v = collapse_value(api, p)
    assert rel(v, pins.dp_value(p)) <= HEALTH
    vals = json.load(open(GOLDEN))["values"]
    if p.name in vals:
        assert rel(v, mp.mpf(vals[p.name]["text"])) <= HEALTH


@pytest.mark.parametrize("seed,d,L,rule,kind", CASES)
def test_collapse_random_problems(api, seed, d, L, rule, kind):
    p = S.random_problem(seed, d, L, rule, kind)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    r = rel(collapse_value(api, p), ref)
    assert r <= HEALTH, (p.name, float(r))


@pytest.mark.parametrize("seed,d,L,rule,kind", CASES[1::3])
def test_collapse_delta_form(api, seed, d, L, rule, kind):
    p = S.random_problem(seed, d, L, rule, kind)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    assert rel(collapse_value(api, p, form=1), ref) <= HEALTH


@pytest.mark.parametrize("i", [2, 3, 4, 5])
def test_collapse_equals_tree(api, i):
    """Two different evaluation orders of the same Eq 2.6 sum agree to dd rounding: each is within
    ~1e-20 of the 50-digit value on config 5 (the tree's FP64 low accumulators, amplified by the
    combination sum's cancellation kappa <= 9.3e9; measured 5e-21), so 1e-19."""
    p = S.baseline_config(i)
    hi, lo = api.integrate(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u)
    tree = mp.mpf(hi) + mp.mpf(lo)
    assert rel(collapse_value(api, p), tree) <= 1e-19


@pytest.mark.parametrize("d,L,rule,kind", [
    (2, 19, S.RULE_GL, S.KIND_OSC),      # maximum level budget: largest shared-memory polynomials
    (3, 11, S.RULE_CC, S.KIND_EXP),      # maximum Clenshaw-Curtis level (n = 2049)
    (1, 0, S.RULE_CC, S.KIND_GAUSS),     # degenerate: one point
])
def test_collapse_extreme_levels_vs_oracle(api, d, L, rule, kind):
    p = S.random_problem(70 + L, d, L, rule, kind)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    assert rel(collapse_value(api, p), ref) <= HEALTH


def test_collapse_large_d_vs_dp(api):
    """d = 50,000 (many CTAs, ragged coordinate chunks) against the 50-digit DP pin."""
    p = S.random_problem(77, 50000, 2, S.RULE_GL, S.KIND_GAUSS)
    assert rel(collapse_value(api, p), pins.dp_value(p)) <= HEALTH


def test_collapse_ranks_and_determinism(api):
    import torch
    p = S.baseline_config(5)
    whole = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, method=api.METHOD_COLLAPSE)
    a = whole.integrate_host()
    assert whole.integrate_host() == a                     # bitwise reproducible
    assert whole.passes() == []                            # no tree pass runs
    parts = []
    for r in range(3):
        sp = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=r, world=3,
                      method=api.METHOD_COLLAPSE)
        parts.append(sp.sg_integrate().clone())
        torch.cuda.synchronize()
        if r:
            assert parts[-1].abs().sum().item() == 0.0     # only rank 0 emits the value
            assert sp.points()[0] == 0
        sp.close()
    res = whole.sg_finalize(torch.cat(parts), 3).cpu().numpy()
    assert (float(res[0]), float(res[1])) == a
    whole.close()


def test_collapse_option_errors(api):
    from paper_2210_14313_b200._lib import SGError
    p = S.baseline_config(1)
    with pytest.raises(SGError) as e:
        api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, method=api.METHOD_COLLAPSE,
                 merge=api.MERGE_MIDPOINT)
    assert e.value.code == -1
    with pytest.raises(SGError) as e:
        api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, method=api.METHOD_COLLAPSE,
                 arith=api.ARITH_SFORM_FP64)
    assert e.value.code == -2
    with pytest.raises(SGError):
        api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, method=7)
    # non-finite factor -> NaN result and NonFiniteIntegrand
    q = api.Plan(3, 6, S.RULE_CC, S.KIND_EXP, np.array([2000.0, 1.0, 1.0]), method=api.METHOD_COLLAPSE)
    with pytest.raises(SGError) as e:
        q.integrate_host()
    assert e.value.code == -6
    q.close()
