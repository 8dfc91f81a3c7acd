"""GPU parity of pass L-2 as k_leaf2_sym3 source tasks (DESIGN.md §1 step 4, §6).

Plans whose fused leaf kernel is k_leaf2_sym3 (oscillatory kind, level-2 row {0, 1/2, 1} symmetric,
level 3 of 5 nodes: Clenshaw-Curtis or trapezoidal, combination or delta form) evaluate the
depth-(L-1) points of frontier L-2 as source tasks instead of the generic k_leaf: the excess-(L-1)
sources' level-2 rows (coefficient c(L)), the excess-(L-2) sources' level-2 rows (c(L-1)) and their
level-3 rows (c(L)), with the rows split on small shards.  Each case is checked against the
__float128 oracle (plain Eq 2.6/2.7 enumeration); sharded runs must also sum to the whole.
"""
import mpmath as mp
import pytest

import oracle
import sg_configs as S
from test_gpu_parity import HEALTH, check, rel

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


@pytest.mark.parametrize("seed,d,L,rule,form", [
    (301, 40, 4, S.RULE_CC, 0),      # c5-like: L = 4, ragged d
    (302, 100, 3, S.RULE_CC, 0),     # L = 3: frontier L-2 = 1 (the root pass's children)
    (303, 13, 5, S.RULE_CC, 0),      # L = 5: three stored frontiers before the source pass
    (304, 40, 4, S.RULE_TRAP, 0),    # trapezoidal: dyadic nodes, level 3 exactly symmetric
    (305, 37, 4, S.RULE_CC, 1),      # delta form (coefficient 1, signed delta weights)
    (306, 9, 6, S.RULE_TRAP, 1),
])
def test_source_tasks_vs_oracle(api, seed, d, L, rule, form):
    p = S.random_problem(seed, d, L, rule, S.KIND_OSC)
    check(api, p, form=form)


@pytest.mark.parametrize("world", [3, 8])
def test_source_tasks_sharded(api, world):
    """Small shards split the source tasks' rows; the shards' partials still sum to the whole and
    to the oracle value."""
    import torch
    p = S.random_problem(307, 48, 4, S.RULE_CC, S.KIND_OSC)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    parts = []
    for r in range(world):
        sp = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=r, world=world)
        parts.append(sp.sg_integrate().clone())
        torch.cuda.synchronize()
        sp.close()
    whole = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u)
    a = whole.integrate_host()
    res = whole.sg_finalize(torch.cat(parts), world).cpu().numpy()
    whole.close()
    v_whole = mp.mpf(a[0]) + mp.mpf(a[1])
    v_shards = mp.mpf(float(res[0])) + mp.mpf(float(res[1]))
    assert rel(v_whole, ref) <= HEALTH
    assert rel(v_shards, ref) <= HEALTH
    assert rel(v_shards, v_whole) <= 1e-20


def test_source_pass_terms_and_launch(api):
    """Pass L-2 keeps its point count (the points it evaluates, now in the source-task launch) and
    its profile entry is a real launch."""
    p = S.baseline_config(5)
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u)
    passes = plan.passes()
    assert passes[2].terms == 721726200 and passes[3].terms == 26794085175
    plan.profile_enable(True)
    plan.integrate_host()
    ms = plan.profile_read()
    assert ms[3 + 2 - 1] > 0.05          # pass 2: ~0.43 ms of source tasks on a B200
    plan.close()


@pytest.mark.parametrize("d,L,rule", [(2500, 3, S.RULE_CC), (700, 4, S.RULE_TRAP)])
def test_source_tasks_large_d_no_smem(api, d, L, rule):
    """d large enough that the level-2 factor slice no longer fits shared memory (the fused and the
    source-task launches read it through L1): 1e11-1e12 points, against the 50-digit DP value and the
    separable collapse (an independent evaluation order of the same Eq 2.6 sum)."""
    import pins
    p = S.random_problem(308, d, L, rule, S.KIND_OSC)
    hi, lo = api.integrate(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u)
    v = mp.mpf(hi) + mp.mpf(lo)
    assert rel(v, pins.dp_value(p)) <= HEALTH
    chi, clo = api.integrate(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u, method=api.METHOD_COLLAPSE)
    assert rel(v, mp.mpf(chi) + mp.mpf(clo)) <= 1e-18
