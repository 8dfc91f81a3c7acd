"""GPU parity at the size limits of the C ABI (include/sg_b200.h): maximum dimension d = 2^20 - 1
(20-bit coordinate fields of the frontier records), maximum level budget L = 19 (Gauss-Legendre)
and the maximum Clenshaw-Curtis level 12 (n = 2049 nodes per row), in the tree and merged modes.
"""
import mpmath as mp
import pytest

import oracle
import sg_configs as S
from test_gpu_parity import HEALTH, rel

pytestmark = pytest.mark.gpu

DMAX = (1 << 20) - 1


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2210_14313_b200 import build as B
    B.build()
    from paper_2210_14313_b200 import api as A
    return A


def gpu(api, p, **kw):
    hi, lo = api.integrate(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u, **kw)
    return mp.mpf(hi) + mp.mpf(lo)


def test_max_dimension_tail_subtrees_vs_oracle(api):
    """d = 2^20 - 1, L = 2: the depth-1 prefixes of the last 50 coordinates (their coordinate
    indices need all 20 bits) against the oracle's point-by-point enumeration."""
    p = S.random_problem(110, DMAX, 2, S.RULE_CC, S.KIND_OSC)
    nd1 = DMAX * (3 + 5)
    lo, hi = nd1 - 400, nd1
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1, lo=lo, hi=hi, include_root=False).text)
    assert rel(gpu(api, p, range_lo=lo, range_hi=hi), ref) <= HEALTH


def test_max_dimension_full_tree_equals_collapse(api):
    """The whole d = 2^20 - 1, L = 2 integral (2.2e12 Gauss-Legendre points) by the tree and by the
    separable collapse (two independent evaluation orders of Eq 2.6) agree to dd rounding times the
    cancellation of the combination sum: coefficients C(d-1, 2) = 5.5e11, -(d-1), 1 against class
    sums 1, ~d, ~d^2/2 leave an O(1) result, kappa ~ 1e12, so ~1e-32 * 1e12 = 1e-20."""
    p = S.random_problem(111, DMAX, 2, S.RULE_GL, S.KIND_EXP)
    p.c[:] = p.c * (1.0 / abs(p.c).sum())   # keep exp(sum c x) O(1) at this d
    tree = gpu(api, p)
    coll = gpu(api, p, method=api.METHOD_COLLAPSE)
    assert rel(tree, coll) <= 1e-18


@pytest.mark.parametrize("d,L,rule,kind,kw", [
    (2, 19, S.RULE_GL, S.KIND_OSC, {}),                      # maximum level budget
    (2, 19, S.RULE_GL, S.KIND_PEAK, {"form": 1}),            # ... in the delta form
    (3, 11, S.RULE_CC, S.KIND_EXP, {}),                      # maximum CC level: 2049-node rows
    (3, 11, S.RULE_CC, S.KIND_OSC, {"merge": 1}),            # ... midpoint-merged
    (2, 11, S.RULE_TRAP, S.KIND_GAUSS, {}),                  # maximum trapezoidal level
    (2, 19, S.RULE_GP, S.KIND_EXP, {}),                      # 31-point Patterson rows
])
def test_maximum_levels_vs_oracle(api, d, L, rule, kind, kw):
    p = S.random_problem(120 + L + rule, d, L, rule, kind)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    assert rel(gpu(api, p, **kw), ref) <= HEALTH


def test_limits_rejected(api):
    from paper_2210_14313_b200._lib import SGError
    import numpy as np
    for d, q, rule in [(2, 2 + 20, S.RULE_GL),            # L = 20 > 19
                       (3, 3 + 12, S.RULE_CC),            # CC level 13
                       (DMAX + 1, DMAX + 2, S.RULE_CC)]:  # d > 2^20 - 1
        with pytest.raises(SGError) as e:
            api.Plan(d, q, rule, S.KIND_EXP, np.full(d, 0.1))
        assert e.value.code == -2


@pytest.mark.parametrize("d,L,kind", [(1, 19, S.KIND_OSC), (2, 15, S.KIND_GAUSS), (3, 12, S.KIND_EXP)])
def test_trapezoid_up_to_level_20(api, d, L, kind):
    """The trapezoidal rule's exact dyadic tables go to level 20 (n = 524289 nodes per row; the
    Clenshaw-Curtis cap stays 12, include/sg_b200.h): tree and merged modes against the oracle."""
    p = S.random_problem(120 + d, d, L, S.RULE_TRAP, kind)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    assert rel(gpu(api, p), ref) <= HEALTH
    assert rel(gpu(api, p, merge=api.MERGE_MIDPOINT), ref) <= HEALTH
