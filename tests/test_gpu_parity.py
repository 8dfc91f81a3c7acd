"""GPU parity: the CUDA path (through the C ABI) against the __float128 oracle on the same seeded inputs.

Gate (BASELINE.json north_star): |A_gpu - A_oracle| <= 1e-12 |A_oracle| in FP64.  The factor-form
double-double path is expected far inside it (<= 1.6e-18 simulated), so a second,
tighter "health" bound (1e-15) flags numerical regressions long before the gate.
"""
import json
import os

import mpmath as mp
import numpy as np
import pytest

import oracle
import pins
import sg_configs as S

pytestmark = pytest.mark.gpu
GATE = 1e-12
HEALTH = 1e-15
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "oracle_full.json")


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2210_14313_b200 import build as B
    B.build()
    from paper_2210_14313_b200 import api as A
    return A


def gpu_value(api, p, **kw):
    hi, lo = api.integrate(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u, **kw)
    return mp.mpf(hi) + mp.mpf(lo), hi


def rel(a, b):
    return abs((a - b) / b) if b != 0 else abs(a - b)


def check(api, p, tol=GATE, health=HEALTH, **kw):
    ref = oracle.integrate_problem(p, eval_mode=1, lo=kw.get("range_lo", 0),
                                   hi=kw.get("range_hi", -1),
                                   include_root=kw.get("range_lo", 0) == 0)
    v, hi = gpu_value(api, p, **kw)
    r = rel(v, mp.mpf(ref.text))
    assert r <= tol, (p.name, float(r), hi, ref.text)
    if health is not None:
        assert r <= health, (p.name, float(r))
    return float(r)


@pytest.mark.parametrize("i", [1, 2])
def test_baseline_small_configs(api, i):
    check(api, S.baseline_config(i))


def test_config3_full_vs_oracle(api):
    p = S.baseline_config(3)
    golden = json.load(open(GOLDEN))["values"]["c3"]
    v, _ = gpu_value(api, p)
    assert rel(v, mp.mpf(golden["text"])) <= HEALTH


@pytest.mark.parametrize("i", [4, 5])
def test_big_configs_full_size(api, i):
    """Full BASELINE sizes in the bench launch configuration: against the stored full-size oracle
    value when present (oracle/make_golden.py), and always against the 50-digit DP pin."""
    p = S.baseline_config(i)
    v, _ = gpu_value(api, p)
    dp = pins.dp_value(p)
    assert rel(v, dp) <= HEALTH
    if os.path.exists(GOLDEN):
        vals = json.load(open(GOLDEN))["values"]
        if p.name in vals:
            assert rel(v, mp.mpf(vals[p.name]["text"])) <= HEALTH


# sampled full-size outputs: contiguous ranges of depth-1 subtrees of configs 4-5, each small enough
# for the oracle to enumerate point by point
@pytest.mark.parametrize("i,lo,hi", [(4, 16900, 16917), (4, 9000, 9008), (4, 16983, 17000),
                                     (5, 9520, 9554), (5, 10100, 10200), (5, 8000, 8003)])
def test_big_configs_sampled_subtrees(api, i, lo, hi):
    p = S.baseline_config(i)
    check(api, p, range_lo=lo, range_hi=hi)


CASES = [
    # seed, d, L, rule, kind   (ragged tails: d not multiple of 32, several tiles per pass)
    (41, 1, 5, S.RULE_CC, S.KIND_EXP), (42, 1, 9, S.RULE_GL, S.KIND_OSC),
    (43, 2, 7, S.RULE_CC, S.KIND_PEAK), (44, 3, 0, S.RULE_GL, S.KIND_GAUSS),
    (45, 5, 1, S.RULE_CC, S.KIND_OSC), (46, 37, 2, S.RULE_CC, S.KIND_GAUSS),
    (47, 33, 3, S.RULE_GL, S.KIND_PEAK), (48, 65, 3, S.RULE_CC, S.KIND_EXP),
    (49, 7, 6, S.RULE_GL, S.KIND_EXP), (50, 12, 5, S.RULE_CC, S.KIND_OSC),
    (51, 130, 2, S.RULE_GL, S.KIND_OSC), (52, 4, 8, S.RULE_CC, S.KIND_GAUSS),
    (53, 300, 2, S.RULE_CC, S.KIND_PEAK), (54, 20, 4, S.RULE_GL, S.KIND_GAUSS),
    # trapezoidal (r = 1) and Gauss-Patterson (r = 3, delayed: repeated levels) rules
    (55, 8, 5, S.RULE_GP, S.KIND_OSC), (56, 50, 3, S.RULE_GP, S.KIND_GAUSS),
    (57, 6, 6, S.RULE_TRAP, S.KIND_EXP), (58, 100, 3, S.RULE_TRAP, S.KIND_PEAK),
    (59, 3, 9, S.RULE_GP, S.KIND_PEAK),
]


@pytest.mark.parametrize("seed,d,L,rule,kind", CASES)
def test_random_problems(api, seed, d, L, rule, kind):
    check(api, S.random_problem(seed, d, L, rule, kind))


@pytest.mark.parametrize("seed,d,L,rule,kind", CASES[::3])
def test_delta_form_equals_combination(api, seed, d, L, rule, kind):
    p = S.random_problem(seed, d, L, rule, kind)
    check(api, p, form=1)


def test_paper_table_rows(api):
    for t, d, N in [("5.6", 5, 8), ("5.7", 10, 6), ("5.8", 10, 8)]:
        check(api, S.paper_table_problem(t, d, N))


def test_shards_sum_to_whole_and_deterministic(api):
    import torch
    p = S.baseline_config(3)
    whole = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u)
    a = whole.integrate_host()
    b = whole.integrate_host()
    assert a == b                               # bitwise reproducible reruns
    world = 4
    parts = []
    for r in range(world):
        sp = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=r, world=world)
        parts.append(sp.sg_integrate().clone())
        torch.cuda.synchronize()
        sp.close()
    gathered = torch.cat(parts)
    res = whole.sg_finalize(gathered, world).cpu().numpy()
    v1 = mp.mpf(a[0]) + mp.mpf(a[1])
    v4 = mp.mpf(res[0]) + mp.mpf(res[1])
    assert rel(v4, v1) <= 1e-20
    whole.close()


def test_factor_table_matches_mpmath(api):
    """K0 element by element: F[l][k][j] = w_j^l E_k(x_j^l) in dd vs 50-digit values."""
    for kind in (S.KIND_EXP, S.KIND_OSC, S.KIND_PEAK, S.KIND_GAUSS):
        p = S.random_problem(60 + kind, 7, 3, S.RULE_CC, kind)
        plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u)
        plan.integrate_host()
        tab, base = plan.debug_tables()
        idx = 0
        for l in range(2, p.L + 2):
            x, w = pins.mp_rule(p.rule, l)
            for k in range(p.d):
                for j in range(len(x)):
                    xm = mp.mpf(x[j]) - mp.mpf(0.5)
                    ck = mp.mpf(p.c[k])
                    if kind == S.KIND_EXP:
                        e = mp.exp(ck * xm)
                    elif kind == S.KIND_OSC:
                        e = mp.expj(ck * xm)
                    elif kind == S.KIND_GAUSS:
                        wk = mp.mpf(p.w[k])
                        e = mp.exp(-ck ** 2 * ((mp.mpf(x[j]) - wk) ** 2 - (mp.mpf(0.5) - wk) ** 2))
                    else:
                        wk = mp.mpf(p.w[k])
                        e = (1 / ck ** 2 + (mp.mpf(0.5) - wk) ** 2) / (1 / ck ** 2 + (mp.mpf(x[j]) - wk) ** 2)
                    ref = mp.mpf(w[j]) * e
                    got = mp.mpf(tab[idx, 0]) + mp.mpf(tab[idx, 1])
                    assert abs(got - mp.re(ref)) <= 1e-30 * max(abs(ref), 1e-300), (kind, l, k, j)
                    if kind == S.KIND_OSC:
                        goti = mp.mpf(tab[idx, 2]) + mp.mpf(tab[idx, 3])
                        assert abs(goti - mp.im(ref)) <= 1e-30 * max(abs(ref), 1e-300)
                    idx += 1
        plan.close()


def test_errors_and_nonfinite(api):
    from paper_2210_14313_b200._lib import SGError
    with pytest.raises(SGError):
        api.Plan(4, 3, S.RULE_CC, S.KIND_EXP, np.ones(4))               # q < d
    with pytest.raises(SGError):
        api.Plan(4, 6, S.RULE_CC, S.KIND_PEAK, np.ones(4))              # w missing
    with pytest.raises(SGError):
        api.Plan(4, 6, S.RULE_CC, S.KIND_EXP, np.array([1, 2, np.nan, 3.0]))
    # exp overflow in the factor table -> NonFiniteIntegrand, result NaN
    p = api.Plan(3, 6, S.RULE_CC, S.KIND_EXP, np.array([2000.0, 1.0, 1.0]))
    with pytest.raises(SGError) as ei:
        p.integrate_host()
    assert ei.value.code == -6
    p.close()


# every last-pass kernel variant must agree with the oracle: fused k_leaf2 (SG_B200_FUSE=1), stored
# frontier + k_leaf1 (SG_B200_NOFUSE=1), stored frontier + generic k_leaf (+ SG_B200_GENERIC_LEAF=1)
@pytest.mark.parametrize("mode", ["fused", "nofuse", "generic"])
@pytest.mark.parametrize("seed,d,L,rule,kind", [
    (61, 40, 3, S.RULE_CC, S.KIND_OSC), (62, 75, 4, S.RULE_CC, S.KIND_GAUSS),
    (63, 33, 4, S.RULE_GL, S.KIND_PEAK), (64, 9, 5, S.RULE_GL, S.KIND_OSC),
    (65, 200, 3, S.RULE_GL, S.KIND_EXP), (66, 45, 4, S.RULE_GP, S.KIND_OSC),
    (67, 60, 3, S.RULE_TRAP, S.KIND_OSC)])
def test_last_pass_variants(api, monkeypatch, mode, seed, d, L, rule, kind):
    if mode == "fused":
        monkeypatch.setenv("SG_B200_FUSE", "1")
    if mode in ("nofuse", "generic"):
        monkeypatch.setenv("SG_B200_NOFUSE", "1")
    if mode == "generic":
        monkeypatch.setenv("SG_B200_GENERIC_LEAF", "1")
    check(api, S.random_problem(seed, d, L, rule, kind))


@pytest.mark.parametrize("mode", ["fused", "nofuse"])
def test_config5_sampled_variants(api, monkeypatch, mode):
    if mode == "fused":
        monkeypatch.setenv("SG_B200_FUSE", "1")
    if mode == "nofuse":
        monkeypatch.setenv("SG_B200_NOFUSE", "1")
    check(api, S.baseline_config(5), range_lo=9400, range_hi=9520)


@pytest.mark.parametrize("i", [1, 2, 3])
def test_cuda_graph_replay_bitwise(api, i):
    """A captured step (CUDA graph) replays to the same bits as the eager step."""
    import torch
    p = S.baseline_config(i)
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u)
    eager = plan.integrate_host()
    g = plan.capture_graph()
    for _ in range(3):
        plan.result().zero_()
        g.replay()
        torch.cuda.synchronize()
        r = plan.result().cpu().numpy()
        assert (float(r[0]), float(r[1])) == eager
    plan.close()


@pytest.mark.parametrize("kind", [S.KIND_OSC, S.KIND_GAUSS])
def test_update_integrand_host_pinned_device(api, kind):
    """sg_update_integrand (the e2e leg's H2D path): new parameters from numpy, pinned host and
    device tensors give bitwise the value of a fresh plan of the new problem, and match the oracle."""
    import torch
    a = S.random_problem(130, 25, 3, S.RULE_CC, kind)
    b = S.random_problem(131, 25, 3, S.RULE_CC, kind)
    fresh = api.Plan(b.d, b.q, b.rule, b.kind, b.c, b.w, b.u)
    want = fresh.integrate_host()
    fresh.close()
    plan = api.Plan(a.d, a.q, a.rule, a.kind, a.c, a.w, a.u)
    w_np = b.w if b.w is not None else None
    for how in ("numpy", "pinned", "device"):
        if how == "numpy":
            c, w = b.c, w_np
        elif how == "pinned":
            c = torch.from_numpy(b.c.copy()).pin_memory()
            w = None if w_np is None else torch.from_numpy(w_np.copy()).pin_memory()
        else:
            c = torch.from_numpy(b.c.copy()).cuda()
            w = None if w_np is None else torch.from_numpy(w_np.copy()).cuda()
        plan.sg_update_integrand(c, w, b.u)
        assert plan.integrate_host() == want, how
        plan.sg_update_integrand(a.c, a.w, a.u)   # back to a, then to b again
    ref = oracle.integrate_problem(b, eval_mode=1)
    assert rel(mp.mpf(want[0]) + mp.mpf(want[1]), mp.mpf(ref.text)) <= HEALTH
    plan.close()


@pytest.mark.parametrize("i", [4, 5])
def test_full_size_properties(api, i):
    """Properties that hold at any size, checked at the full BASELINE sizes in the bench launch
    configuration: the integral is invariant under a permutation of the coordinates (a different
    prefix tree, shard order and task schedule) and the coordinate-wise difference form (reading R6)
    gives the same value as Eq 2.6 — both against the stored full-size oracle value."""
    p = S.baseline_config(i)
    golden = mp.mpf(json.load(open(GOLDEN))["values"][p.name]["text"])
    perm = np.random.default_rng(7).permutation(p.d)
    q = S.Problem(p.name + "_perm", p.d, p.L, p.rule, p.kind, p.c[perm].copy(),
                  None if p.w is None else p.w[perm].copy(), p.u)
    v, _ = gpu_value(api, q)
    assert rel(v, golden) <= HEALTH
    v, _ = gpu_value(api, p, form=1)
    assert rel(v, golden) <= HEALTH


def test_shard_ranges_independent_of_leaf_path(api, monkeypatch):
    """Every rank must cut the same depth-1 ranges whatever leaf path its plan takes (fused or
    stored frontier, factor or s-form arithmetic): the shard cost model depends on the problem only."""
    p = S.baseline_config(5)
    world = 4
    ref = [api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=r, world=world).range()
           for r in range(world)]
    monkeypatch.setenv("SG_B200_NOFUSE", "1")
    nofuse = [api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=r, world=world).range()
              for r in range(world)]
    monkeypatch.delenv("SG_B200_NOFUSE")
    sform = [api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=r, world=world,
                      arith=api.ARITH_SFORM_DD).range() for r in range(world)]
    assert ref == nofuse == sform
    assert ref[0][0] == 0 and ref[-1][1] == ref[-1][2]
    assert all(a[1] == b[0] for a, b in zip(ref, ref[1:]))


@pytest.mark.parametrize("name,d,L,rule,kind,c,w,u", [
    ("osc_huge_phase", 6, 4, S.RULE_CC, S.KIND_OSC, [0.7, 0.2, 0.9, 0.4, 0.1, 0.6], None, 1.0e6 + 0.3),
    ("osc_big_c", 5, 4, S.RULE_GL, S.KIND_OSC, [40.0, -25.0, 10.0, 33.0, -7.0], None, 0.25),
    ("exp_big_c", 5, 4, S.RULE_CC, S.KIND_EXP, [30.0, -20.0, 12.5, 40.0, -35.0], None, 0.0),
    ("peak_sharp", 4, 5, S.RULE_GP, S.KIND_PEAK, [25.0, 18.0, 30.0, 22.0], [0.3, 0.7, 0.5, 0.05], 0.0),
    ("peak_flat", 6, 3, S.RULE_CC, S.KIND_PEAK, [1e-3, 2e-3, 5e-4, 1e-3, 3e-3, 1e-3],
     [0.1, 0.9, 0.5, 0.2, 0.8, 0.4], 0.0),
    ("gauss_wide", 8, 3, S.RULE_TRAP, S.KIND_GAUSS, [5.0, 4.0, 6.0, 3.0, 5.5, 4.5, 2.0, 7.0],
     [0.5, 0.1, 0.9, 0.3, 0.7, 0.2, 0.6, 0.4], 0.0),
])
def test_parameter_extremes(api, name, d, L, rule, kind, c, w, u):
    """Large phases (dd range reduction of 2 pi u), large |c| (wide dynamic range of the factors),
    sharp and flat product peaks, narrow Gaussians: tree, merged and collapse against the oracle."""
    p = S.Problem(name, d, L, rule, kind, np.array(c, dtype=float),
                  None if w is None else np.array(w, dtype=float), u)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    for kw in ({}, {"merge": api.MERGE_MIDPOINT}, {"method": api.METHOD_COLLAPSE}):
        v, _ = gpu_value(api, p, **kw)
        assert rel(v, ref) <= HEALTH, (name, kw, float(rel(v, ref)))


@pytest.mark.parametrize("name,d,L,rule,kind,c,w,u,tol", [
    # exp arguments c (x - 1/2) up to +-160 (m up to ~230 in the 2^m exp(j/64) exp(s) reduction); the
    # integrand's largest value e^470 stays finite
    ("exp_wide", 5, 3, S.RULE_CC, S.KIND_EXP, [320.0, -320.0, 150.0, -1.5, 0.0], None, 0.0, 1e-28),
    # phases up to 5e3 (the one pi/64 reduction: N up to 1e5, every quadrant and table index) and a
    # base phase 2 pi u of ~7.8e5
    ("osc_wide", 4, 3, S.RULE_CC, S.KIND_OSC, [1.0e4, -3.0e3, 77.7, 0.5], None, 123456.789, 1e-26),
    # Gaussian exponents c^2 (x - 1/2)(x + 1/2 - 2 w) up to ~+-310, w at the ends of [0, 1]
    ("gauss_wide", 3, 3, S.RULE_TRAP, S.KIND_GAUSS, [25.0, 20.0, 0.1], [0.0, 1.0, 0.5], 0.0, 1e-28),
    ("peak_wide", 3, 3, S.RULE_GL, S.KIND_PEAK, [100.0, 1e-3, 3.0], [0.5, 0.0, 1.0], 0.0, 1e-29),
])
def test_factor_table_and_base_wide_arguments(api, name, d, L, rule, kind, c, w, u, tol):
    """K0 element by element at wide arguments (the table-driven dd exp / sincos of csrc/dd.cuh over
    their whole reduction ranges): every F[l][k][j] = w_j E_k(x_j) and the base B against 50-digit
    mpmath, to `tol` relative (absolute x |w_j| for the unit-modulus oscillatory factors)."""
    p = S.Problem(name, d, L, rule, kind, np.array(c, dtype=float),
                  None if w is None else np.array(w, dtype=float), u)
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u)
    plan.integrate_host()
    tab, base = plan.debug_tables()
    ck = [mp.mpf(v) for v in p.c]
    wk = [mp.mpf(v) for v in p.w] if p.w is not None else None
    idx = 0
    for l in range(2, p.L + 2):
        x, wt = pins.mp_rule(p.rule, l)
        for k in range(p.d):
            for j in range(len(x)):
                xm = mp.mpf(x[j]) - mp.mpf(0.5)
                if kind == S.KIND_EXP:
                    e = mp.exp(ck[k] * xm)
                elif kind == S.KIND_OSC:
                    e = mp.expj(ck[k] * xm)
                elif kind == S.KIND_GAUSS:
                    e = mp.exp(-ck[k] ** 2 * ((mp.mpf(x[j]) - wk[k]) ** 2 - (mp.mpf(0.5) - wk[k]) ** 2))
                else:
                    e = (1 / ck[k] ** 2 + (mp.mpf(0.5) - wk[k]) ** 2) / (1 / ck[k] ** 2 + (mp.mpf(x[j]) - wk[k]) ** 2)
                ref = mp.mpf(wt[j]) * e
                scale = abs(mp.mpf(wt[j])) if kind == S.KIND_OSC else abs(ref)
                got = mp.mpf(tab[idx, 0]) + mp.mpf(tab[idx, 1])
                assert abs(got - mp.re(ref)) <= tol * scale, (name, l, k, j, float(abs(got - mp.re(ref)) / scale))
                if kind == S.KIND_OSC:
                    goti = mp.mpf(tab[idx, 2]) + mp.mpf(tab[idx, 3])
                    assert abs(goti - mp.im(ref)) <= tol * scale, (name, l, k, j)
                idx += 1
    half = mp.mpf(0.5)
    if kind == S.KIND_EXP:
        B = mp.exp(sum(ck) * half)
    elif kind == S.KIND_OSC:
        B = mp.expj(2 * mp.pi * mp.mpf(p.u) + sum(ck) * half)
    elif kind == S.KIND_GAUSS:
        B = mp.exp(-sum(ck[k] ** 2 * (half - wk[k]) ** 2 for k in range(p.d)))
    else:
        B = mp.fprod(1 / (1 / ck[k] ** 2 + (half - wk[k]) ** 2) for k in range(p.d))
    gb = mp.mpf(base[0]) + mp.mpf(base[1])
    assert abs(gb - mp.re(B)) <= 10 * tol * abs(B), (name, float(abs(gb - mp.re(B)) / abs(B)))
    if kind == S.KIND_OSC:
        assert abs(mp.mpf(base[2]) + mp.mpf(base[3]) - mp.im(B)) <= 10 * tol * abs(B)
    plan.close()
