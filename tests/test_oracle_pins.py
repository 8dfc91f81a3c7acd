"""Pins of the CPU oracle against things other than itself.

Every test here runs without a GPU.  The oracle (oracle/sg_oracle.c) is checked against:
paper-printed values (Tables 5.6-5.8), 50-digit generating-function values of Eq 2.6 (tests/pins.py),
closed-form integrals, weight-sum and polynomial-exactness identities, special cases (d = 1, L = 0,
odd symmetry) and a brute-force tensor enumeration written independently below.
"""
import functools
import itertools
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest

import oracle
import pins
import sg_configs as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def qval(res):
    return mp.mpf(res.text)


# ----------------------------------------------------------------------------------------------
# P4: 1-D rules
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("rule,levels", [(S.RULE_CC, range(1, 10)), (S.RULE_GL, range(1, 16)),
                                         (S.RULE_TRAP, range(1, 12)), (S.RULE_GP, range(1, 21))])
def test_rule_tables_bit_identical_to_mpmath(rule, levels):
    for l in levels:
        x, w = oracle.rule(rule, l)
        px, pw = pins.mp_rule(rule, l)
        assert tuple(x) == px, (rule, l)
        assert tuple(w) == pw, (rule, l)


def test_rule_examples():
    # CC n=3 -> weights (1,4,1)/6 on [0,1] (SPEC.md:70 scaled by 1/2; reading R4)
    x, w = oracle.rule(S.RULE_CC, 2)
    assert list(x) == [0.0, 0.5, 1.0]
    np.testing.assert_allclose(w, [1 / 6, 4 / 6, 1 / 6], rtol=0, atol=1e-16)
    # CC n=5 -> (1,8,12,8,1)/30
    x, w = oracle.rule(S.RULE_CC, 3)
    np.testing.assert_allclose(w, np.array([1, 8, 12, 8, 1]) / 30, rtol=0, atol=1e-16)
    # GL n=2 -> 1/2 -+ 1/(2 sqrt 3), weights 1/2 (SPEC.md:69 mapped)
    x, w = oracle.rule(S.RULE_GL, 2)
    np.testing.assert_allclose(x, [0.5 - 0.5 / math.sqrt(3), 0.5 + 0.5 / math.sqrt(3)], atol=1e-16)
    np.testing.assert_allclose(w, [0.5, 0.5], atol=1e-16)
    # level 1 = midpoint, weight 1 (reading R3)
    for r in (S.RULE_CC, S.RULE_GL):
        assert oracle.rule(r, 1) == (np.array([0.5]), np.array([1.0])) or (
            list(oracle.rule(r, 1)[0]) == [0.5] and list(oracle.rule(r, 1)[1]) == [1.0])


@pytest.mark.parametrize("rule", [S.RULE_CC, S.RULE_GL])
def test_rule_exactness_and_weight_sum(rule):
    for l in range(1, 8):
        x, w = oracle.rule(rule, l)
        n = len(x)
        with mp.workdps(40):
            assert abs(mp.fsum(mp.mpf(a) for a in w) - 1) < 1e-15
            # GL exact to degree 2n-1; CC (odd n) exact to degree n (pin P4)
            deg = 2 * n - 1 if rule == S.RULE_GL else (n if n % 2 else n - 1)
            for k in range(deg + 1):
                q = mp.fsum(mp.mpf(wj) * mp.mpf(xj) ** k for xj, wj in zip(x, w))
                assert abs(q - mp.mpf(1) / (k + 1)) < 5e-15, (rule, l, k)


def test_trapezoid_and_patterson_examples():
    # trapezoid (Eq 2.10) level 3 on [0,1]: h = 1/4, weights (1,2,2,2,1)/8, exact dyadics
    x, w = oracle.rule(S.RULE_TRAP, 3)
    assert list(x) == [0.0, 0.25, 0.5, 0.75, 1.0]
    assert list(w) == [0.125, 0.25, 0.25, 0.25, 0.125]
    # the 3-point Patterson rule is the 3-point Gauss rule: 1/2 -+ sqrt(15)/10, weights 5/18, 4/9
    x, w = oracle.rule(S.RULE_GP, 2)
    gx, gw = oracle.rule(S.RULE_GL, 3)
    np.testing.assert_allclose(x, gx, rtol=0, atol=2e-16)
    np.testing.assert_allclose(w, [5 / 18, 4 / 9, 5 / 18], rtol=0, atol=2e-16)
    assert x[1] == 0.5
    # delayed sequence of PAPER.md:615 (q = 1..10 -> N = 1, 3, 3, 7, 7, 7, 15, 15, 15, 15)
    assert [oracle.node_count(S.RULE_GP, l) for l in range(1, 11)] == [1, 3, 3, 7, 7, 7, 15, 15, 15, 15]
    assert [oracle.node_count(S.RULE_GP, l) for l in (13, 24, 25)] == [31, 31, 63]


@pytest.mark.parametrize("ext", [1, 2, 3, 4, 5])
def test_patterson_exactness_degree(ext):
    """2^{i+1}-1 Patterson points integrate every polynomial of degree <= 3*2^i - 1 exactly, and
    x^{3*2^i} not (the defining property of the Kronrod-Patterson extension; unique given the
    nested node set).  Checked on [-1,1]-symmetric moments of x - 1/2 on [0,1]."""
    l = [2, 4, 7, 13, 25][ext - 1]
    x, w = oracle.rule(S.RULE_GP, l)
    assert len(x) == 2 ** (ext + 1) - 1
    deg = 3 * 2 ** ext - 1
    with mp.workdps(40):
        xs = [mp.mpf(a) - mp.mpf(0.5) for a in x]
        for k in range(0, deg + 2):
            q = mp.fsum(mp.mpf(b) * a ** k for a, b in zip(xs, w))
            scale = mp.mpf(2) ** (-k) / (k + 1)          # |even moment| of (x - 1/2)^k on [0,1]
            exact = mp.mpf(0) if k % 2 else scale
            if k <= deg:
                assert abs(q - exact) < 1e-14 * scale, (ext, k, q - exact)
            elif ext <= 3:
                # beyond the degree the error is 0.16 / 1.8e-3 / 6.7e-8 relative; for the 31- and
                # 63-point rules it falls below the double rounding of the nodes (not testable)
                assert abs(q - exact) > 1e-9 * scale, (ext, k)


def test_trapezoid_error_order():
    """Eq 2.10 error estimate C 2^{-2q}: the error for e^x on [0,1] falls 4x per level."""
    errs = []
    for l in range(3, 9):
        x, w = oracle.rule(S.RULE_TRAP, l)
        with mp.workdps(40):
            q = mp.fsum(mp.mpf(b) * mp.exp(mp.mpf(a)) for a, b in zip(x, w))
            errs.append(q - (mp.e - 1))
    for a, b in zip(errs, errs[1:]):
        assert 3.9 < a / b < 4.1


@pytest.mark.parametrize("rule", [S.RULE_GP, S.RULE_TRAP])
def test_new_rules_nested_exactly(rule):
    for l in range(1, 12 if rule == S.RULE_TRAP else 20):
        xa, _ = oracle.rule(rule, l)
        xb, _ = oracle.rule(rule, l + 1)
        assert set(xa.tolist()) <= set(xb.tolist()), (rule, l)


@functools.lru_cache(maxsize=None)
def _nodes(rule, l):
    return tuple(oracle.rule(rule, l)[0].tolist())


def _distinct_points_formula(rule, d, L):
    """Distinct points of the Smolyak grid with max level L+1 for a nested rule: each point is new
    at exactly one level per coordinate, so the count is [z^{<=L}] (sum_l new_l z^{l-1})^d with
    new_l = #(nodes of level l not in level l-1), taken from the oracle's double tables."""
    prev = set()
    new = []
    for l in range(1, L + 2):
        xs = set(_nodes(rule, l))
        new.append(len(xs - prev))
        prev |= xs
    poly = [1] + [0] * L
    for _ in range(d):
        nw = [0] * (L + 1)
        for a in range(L + 1):
            for b in range(L + 1 - a):
                nw[a + b] += poly[a] * new[b]
        poly = nw
    return sum(poly)


def _distinct_points_brute(rule, d, L):
    pts = set()
    for lv in itertools.product(range(1, L + 2), repeat=d):
        if sum(lv) - d > L:
            continue
        pts.update(itertools.product(*[_nodes(rule, l) for l in lv]))
    return len(pts)


# PAPER.md:322-401 "Total nodes" columns (Gauss-Patterson, r = 3), reading R1: the paper's accuracy
# level q is the maximum 1-D level, L = q - 1.  Rows beyond d = 12 of Tables 4.5/4.6 do not follow
# any nested count (printed 5036449 < 4286913 * 4 growth breaks), so they are not pins.
_NODE_ROWS = (
    [("4.1", 2, q, n) for q, n in [(6, 33), (7, 65), (9, 97), (10, 161), (13, 257), (14, 321)]]
    + [("4.3", 3, q, n) for q, n in [(9, 495), (10, 751), (11, 1135), (13, 1759), (14, 2335),
                                     (15, 2527), (16, 3679)]]
    + [("4.5", d, 10, n) for d, n in [(2, 161), (4, 2881), (8, 206465), (10, 1041185),
                                      (12, 4286913)]]
    + [("4.6", d, 12, n) for d, n in [(2, 161), (4, 6465), (6, 93665), (8, 791169), (10, 5020449),
                                      (12, 25549761)]])


@pytest.mark.parametrize("table,d,q,n", _NODE_ROWS, ids=lambda v: str(v))
def test_paper_total_nodes_gauss_patterson(table, d, q, n):
    assert _distinct_points_formula(S.RULE_GP, d, q - 1) == n
    if d <= 3:
        assert _distinct_points_brute(S.RULE_GP, d, q - 1) == n


def test_cc_nesting_exact():
    for l in range(2, 9):
        xa, _ = oracle.rule(S.RULE_CC, l)
        xb, _ = oracle.rule(S.RULE_CC, l + 1)
        assert set(xa.tolist()) <= set(xb.tolist())
        assert list(xb[::2]) == list(xa)


# ----------------------------------------------------------------------------------------------
# P6: the paper's printed Tables 5.6-5.8 (Gauss-Legendre, [-1,1]^d -> [0,1]^d)
# ----------------------------------------------------------------------------------------------
_ROWS = json.load(open(os.path.join(GOLDEN, "paper_tables_5_6_to_5_8.json")))["rows"]


@pytest.mark.parametrize("row", _ROWS, ids=lambda r: f"T{r['table']}-d{r['d']}-N{r['N']}")
def test_paper_tables_relative_error(row):
    p = S.paper_table_problem(row["table"], row["d"], row["N"])
    res = oracle.integrate_problem(p, eval_mode=1)
    cf = pins.closed_form(p)
    err = float(abs((qval(res) - cf) / cf))
    # printed to 5 significant digits; allow 2.5 units in the 5th digit (truncation vs rounding,
    # double-rounded parameters).  A dropped term or wrong sign moves these by orders of magnitude.
    assert err == pytest.approx(row["rel_err"], rel=2.5e-4), (err, row)


# ----------------------------------------------------------------------------------------------
# P1: generating-function value of Eq 2.6 (50 digits) vs the oracle's plain enumeration
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("i", [1, 2])
def test_dp_pin_baseline_configs(i):
    p = S.baseline_config(i)
    res = oracle.integrate_problem(p)
    v = pins.dp_value(p)
    assert abs((qval(res) - v) / v) < 1e-30
    assert res.npoints == pins.n_points(p.rule, p.d, p.L)


CASES = [
    (7, 3, 2, S.RULE_CC, S.KIND_EXP), (8, 5, 3, S.RULE_CC, S.KIND_OSC),
    (9, 12, 3, S.RULE_GL, S.KIND_PEAK), (10, 20, 2, S.RULE_CC, S.KIND_GAUSS),
    (11, 3, 6, S.RULE_GL, S.KIND_OSC), (12, 2, 7, S.RULE_CC, S.KIND_PEAK),
    (13, 40, 2, S.RULE_GL, S.KIND_GAUSS), (14, 6, 4, S.RULE_GL, S.KIND_EXP),
    (15, 5, 5, S.RULE_GP, S.KIND_OSC), (16, 30, 3, S.RULE_GP, S.KIND_GAUSS),
    (17, 4, 5, S.RULE_TRAP, S.KIND_EXP), (18, 9, 3, S.RULE_TRAP, S.KIND_PEAK),
]


@pytest.mark.parametrize("seed,d,L,rule,kind", CASES)
def test_dp_pin_random(seed, d, L, rule, kind):
    p = S.random_problem(seed, d, L, rule, kind)
    v = pins.dp_value(p)
    for mode in (0, 1):
        res = oracle.integrate_problem(p, eval_mode=mode)
        assert abs((qval(res) - v) / v) < 1e-28, (mode, res.text, v)
    assert res.npoints == pins.n_points(rule, d, L)
    # Delta form (reading R6 of Eq 2.9) is the same number
    assert abs((pins.dp_value(p, "delta") - v) / v) < 1e-40


# Condition numbers kappa = sum |terms| / |A| of the combination sum per BASELINE config (SURVEY.md
# §8c table, "kappa comb"; osc values are bounds).  The __float128 oracle accumulates ~n terms with
# unit roundoff 2^-113, so its relative error is ~kappa * 2^-113 (x a small growth factor).
KAPPA = {1: 128.0, 2: 1.2e5, 3: 5.8e6, 4: 4.4e7, 5: 9.3e9}


def test_golden_full_values_match_dp():
    """Full-size oracle values (written by oracle/make_golden.py) against the 50-digit DP, within
    10 kappa 2^-113 (config 5: 9e-24; measured 3.8e-25) and never looser than 1e-22."""
    path = os.path.join(GOLDEN, "oracle_full.json")
    if not os.path.exists(path):
        pytest.skip("golden full-size oracle values not generated yet")
    data = json.load(open(path))
    assert data["values"], "empty golden file"
    for name, rec in data["values"].items():
        if not (name[0] == "c" and name[1:].isdigit()):
            continue   # extra workloads (corner peak): not a product integrand, no DP pin
        p = S.baseline_config(int(name[1:]))
        v = pins.dp_value(p)
        tol = max(1e-28, 10 * KAPPA[int(name[1:])] * 2.0 ** -113)
        assert tol <= 1e-22
        assert abs((mp.mpf(rec["text"]) - v) / v) < tol, name
        assert rec["npoints"] == pins.n_points(p.rule, p.d, p.L)


# ----------------------------------------------------------------------------------------------
# P7: closed forms (BASELINE.json); P2 weight sum; P3 exactness; P8 special cases
# ----------------------------------------------------------------------------------------------
def test_closed_forms_configs_1_2():
    p = S.baseline_config(1)
    r = qval(oracle.integrate_problem(p))
    cf = pins.closed_form(p)
    assert abs((r - cf) / cf) < 5e-14          # smooth exp, d=4, L=4: Smolyak error ~1.7e-14
    p = S.baseline_config(2)
    r = qval(oracle.integrate_problem(p))
    cf = pins.closed_form(p)
    assert abs((r - cf) / cf) < 1e-8           # ~3.2e-9


@pytest.mark.parametrize("rule", [S.RULE_CC, S.RULE_GL, S.RULE_GP, S.RULE_TRAP])
@pytest.mark.parametrize("d,L", [(1, 5), (2, 4), (5, 3), (30, 2), (4, 7)])
def test_weight_sum_is_one(rule, d, L):
    """f = 1 (exp kind with c = 0): sum of all combination weights is 1 on [0,1]^d.

    Exactly 1 for the exact rules: the integer identity sum_e c(e) #multi-indices(e) = 1.  With the
    double-rounded weights the sum moves by at most sum_e |c(e)| #mi(e) * d * 2^-52; the oracle must
    reproduce the exact sum of the double weights (generating function, 50 digits)."""
    assert sum(pins.coef(d, L, e) * math.comb(e + d - 1, d - 1) for e in range(L + 1)) == 1
    res = oracle.integrate(d, L, rule, S.KIND_EXP, np.zeros(d))
    exact_double_tables = pins.dp_value(S.Problem("one", d, L, rule, S.KIND_EXP, np.zeros(d)))
    assert abs(qval(res) - exact_double_tables) < 1e-28
    bound = sum(abs(pins.coef(d, L, e)) * math.comb(e + d - 1, d - 1) for e in range(L + 1))
    assert abs(qval(res) - 1) <= bound * d * 2.0 ** -52


@pytest.mark.parametrize("rule", [S.RULE_CC, S.RULE_GL, S.RULE_GP])
def test_polynomial_exactness(rule):
    """A exact for prod x_k^{a_k} when sum_k floor(a_k/2) <= L."""
    rng = np.random.default_rng(5)
    d, L = 4, 3
    for _ in range(12):
        a = np.zeros(d, dtype=int)
        budget = L
        for k in rng.permutation(d):
            h = int(rng.integers(0, budget + 1))
            a[k] = 2 * h + int(rng.integers(0, 2))
            budget -= h
        res = oracle.integrate(d, L, rule, 9, np.ones(d), a.astype(float))
        exact = mp.mpf(1)
        for ak in a:
            exact /= (int(ak) + 1)
        # exact for the exact rules; the double-rounded tables move it by O(1e-16)
        assert abs(qval(res) - exact) < 1e-14, a
    # and NOT exact one step beyond (guards against a rule that is secretly too good/bad)
    # x1^2 x2^2 x3^2 x4^2 needs 4 active coordinates, more than L = 3 allows
    a = np.array([2, 2, 2, 2])
    res = oracle.integrate(d, L, rule, 9, np.ones(d), a.astype(float))
    assert abs(qval(res) - mp.mpf(1) / 81) > 1e-6


@pytest.mark.parametrize("rule", [S.RULE_CC, S.RULE_GL, S.RULE_GP, S.RULE_TRAP])
def test_d1_is_the_1d_rule(rule):
    """d = 1: A(q,1) f = J^{q} f (coefficient C(0,0) = 1)."""
    for L in range(0, 6):
        c = np.array([0.7])
        res = oracle.integrate(1, L, rule, S.KIND_EXP, c)
        x, w = pins.mp_rule(rule, L + 1)
        with mp.workdps(40):
            ref = mp.fsum(mp.mpf(wj) * mp.exp(mp.mpf(0.7) * mp.mpf(xj)) for xj, wj in zip(x, w))
        assert abs(qval(res) - ref) < 1e-30


def test_L0_is_midpoint():
    p = S.random_problem(3, 9, 0, S.RULE_CC, S.KIND_GAUSS)
    res = oracle.integrate_problem(p)
    with mp.workdps(40):
        ref = mp.exp(-mp.fsum(mp.mpf(c) ** 2 * (mp.mpf(0.5) - mp.mpf(w)) ** 2
                              for c, w in zip(p.c, p.w)))
    assert abs(qval(res) - ref) < 1e-30
    assert res.npoints == 1


def test_odd_symmetry_gives_zero():
    """cos(pi/2 + sum c_k (x_k - 1/2)) is odd about the centre; CC nodes are symmetric."""
    d = 5
    c = np.array([0.3, 0.9, 0.5, 0.25, 0.75])      # sum c / 2 = 1.35 exactly representable
    u = (math.pi / 2 - 1.35) / (2 * math.pi)
    res = oracle.integrate(d, 4, S.RULE_CC, S.KIND_OSC, c, None, u)
    assert abs(res.hi) < 1e-14


# ----------------------------------------------------------------------------------------------
# P9: brute-force tensor enumeration at tiny d (independent of the oracle's sparse walk)
# ----------------------------------------------------------------------------------------------
def _f_mp(kind, c, w, u, x):
    if kind == S.KIND_EXP:
        return mp.exp(mp.fsum(mp.mpf(a) * mp.mpf(b) for a, b in zip(c, x)))
    if kind == S.KIND_OSC:
        return mp.cos(2 * mp.pi * mp.mpf(u) + mp.fsum(mp.mpf(a) * mp.mpf(b) for a, b in zip(c, x)))
    if kind == S.KIND_PEAK:
        r = mp.mpf(1)
        for a, b, xx in zip(c, w, x):
            r /= (1 / mp.mpf(a) ** 2 + (mp.mpf(xx) - mp.mpf(b)) ** 2)
        return r
    if kind == S.KIND_GAUSS:
        return mp.exp(-mp.fsum(mp.mpf(a) ** 2 * (mp.mpf(xx) - mp.mpf(b)) ** 2
                               for a, b, xx in zip(c, w, x)))
    if kind == S.KIND_CORNER:
        return (1 + mp.fsum(mp.mpf(a) * mp.mpf(b) for a, b in zip(c, x))) ** (-(len(c) + 1))


@pytest.mark.parametrize("seed,d,L,rule,kind", [
    (21, 2, 3, S.RULE_CC, S.KIND_OSC), (22, 3, 2, S.RULE_GL, S.KIND_PEAK),
    (23, 2, 4, S.RULE_GL, S.KIND_EXP), (24, 3, 3, S.RULE_CC, S.KIND_GAUSS),
    (25, 2, 4, S.RULE_GP, S.KIND_OSC), (26, 3, 2, S.RULE_TRAP, S.KIND_PEAK),
    (27, 2, 3, S.RULE_CC, S.KIND_CORNER), (28, 3, 2, S.RULE_GL, S.KIND_CORNER)])
def test_brute_force_tensor_enumeration(seed, d, L, rule, kind):
    p = S.random_problem(seed, d, L, rule, kind)
    w = p.w if p.w is not None else np.zeros(d)
    with mp.workdps(40):
        total = mp.mpf(0)
        merged = {}
        for lv in itertools.product(range(1, L + 2), repeat=d):
            e = sum(lv) - d
            cf = pins.coef(d, L, e)
            if cf == 0:
                continue
            rules = [pins.mp_rule(rule, l) for l in lv]
            for js in itertools.product(*[range(len(r[0])) for r in rules]):
                x = tuple(rules[m][0][js[m]] for m in range(d))
                wt = mp.mpf(cf)
                for m in range(d):
                    wt *= mp.mpf(rules[m][1][js[m]])
                total += wt * _f_mp(kind, p.c, w, p.u, x)
                merged[x] = merged.get(x, mp.mpf(0)) + wt
        # Eq 2.8: the merged single-sum form gives the same value
        total_merged = mp.fsum(wt * _f_mp(kind, p.c, w, p.u, x) for x, wt in merged.items())
        assert any(wt < 0 for wt in merged.values()) or L == 0   # negative weights
    res = oracle.integrate_problem(p)
    assert abs(qval(res) - total) < 1e-28 * max(1, abs(total))
    assert abs(total_merged - total) < 1e-28 * max(1, abs(total))


def test_multi_index_enumeration_example():
    """N_{2,4} = {[1,3],[2,2],[3,1]}, and #multi-indices = C(e+d-1, d-1)."""
    n24 = [lv for lv in itertools.product(range(1, 5), repeat=2) if sum(lv) == 4]
    assert sorted(n24) == [(1, 3), (2, 2), (3, 1)]
    for d, e in [(3, 2), (5, 3)]:
        cnt = sum(1 for lv in itertools.product(range(1, e + 2), repeat=d) if sum(lv) == d + e)
        assert cnt == math.comb(e + d - 1, d - 1)


def test_coefficients_examples():
    """(d=2,q=4): +1 at |l|=4, -1 at |l|=3; (d=3,q=5): +1,-2,+1."""
    assert pins.coef(2, 2, 2) == 1 and pins.coef(2, 2, 1) == -1 and pins.coef(2, 2, 0) == 0
    assert [pins.coef(3, 2, e) for e in (2, 1, 0)] == [1, -2, 1]


# ----------------------------------------------------------------------------------------------
# oracle internals: plain vs active integrand, shard decomposition, thread-count invariance
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("kind", [S.KIND_EXP, S.KIND_OSC, S.KIND_PEAK, S.KIND_GAUSS, S.KIND_CORNER])
def test_active_form_matches_plain_form_pointwise(kind):
    rng = np.random.default_rng(77 + kind)
    d = 60
    p = S.random_problem(100 + kind, d, 3, S.RULE_CC, kind)
    for _ in range(400):
        x = np.full(d, 0.5)
        for k in rng.choice(d, size=int(rng.integers(0, 5)), replace=False):
            x[k] = rng.choice([0.0, 0.14644660940672624, 0.8535533905932737, 1.0, 0.25])
        a, b = oracle.eval_point(kind, p.c, p.w, p.u, x)
        assert abs((a[0] - b[0]) + (a[1] - b[1])) <= 1e-28 * abs(a[0]) + 1e-300


def test_shards_sum_to_whole_and_threads_invariant():
    p = S.random_problem(31, 12, 3, S.RULE_CC, S.KIND_OSC)
    whole = oracle.integrate_problem(p, nthreads=1)
    whole4 = oracle.integrate_problem(p, nthreads=4)
    assert whole.text == whole4.text
    M0 = sum(pins.node_count(p.rule, l) for l in range(2, p.L + 2))
    total = p.d * M0
    cuts = [0, 1, 17, 40, total // 2, total - 3, total]
    acc = mp.mpf(0)
    npts = 0
    for i in range(len(cuts) - 1):
        r = oracle.integrate_problem(p, lo=cuts[i], hi=cuts[i + 1], include_root=(i == 0))
        acc += qval(r)
        npts += r.npoints
    assert npts == whole.npoints
    assert abs(acc - qval(whole)) < 1e-30


# ----------------------------------------------------------------------------------------------
# Genz corner peak (1 + c.x)^-(d+1): the non-separable kind
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("d,rule", [(2, S.RULE_GL), (3, S.RULE_GL), (5, S.RULE_GL), (3, S.RULE_CC)])
def test_corner_peak_converges_to_closed_form(d, rule):
    """Smolyak error against the exact integral (inclusion-exclusion, 50 digits) falls by more than
    4x per level and is below 1e-6 at L = 8: a wrong exponent, a dropped term or a wrong sign leaves
    an O(1) error instead."""
    p = S.random_problem(90 + d, d, 2, rule, S.KIND_CORNER)
    ex = pins.closed_form(p)
    errs = []
    for L in range(0, 9):
        r = oracle.integrate(d, L, rule, S.KIND_CORNER, p.c)
        errs.append(abs((qval(r) - ex) / ex))
    for a, b in zip(errs[2:], errs[3:]):
        assert b < a / 4, errs
    assert errs[-1] < 1e-6, errs


def test_corner_peak_special_cases():
    # d = 1: the 1-D rule applied to (1 + c x)^-2
    for L in range(0, 6):
        res = oracle.integrate(1, L, S.RULE_CC, S.KIND_CORNER, np.array([0.8]))
        x, w = pins.mp_rule(S.RULE_CC, L + 1)
        with mp.workdps(40):
            ref = mp.fsum(mp.mpf(wj) * (1 + mp.mpf(0.8) * mp.mpf(xj)) ** -2 for xj, wj in zip(x, w))
        assert abs(qval(res) - ref) < 1e-30
    # c = 0: f = 1, the sum of all weights (exactly the weight-sum value of the double tables)
    d, L = 6, 3
    res = oracle.integrate(d, L, S.RULE_GL, S.KIND_CORNER, np.zeros(d))
    one = pins.dp_value(S.Problem("one", d, L, S.RULE_GL, S.KIND_EXP, np.zeros(d)))
    assert abs(qval(res) - one) < 1e-28
    # outside the domain (1 + sum min(c, 0) <= 0): rejected
    with pytest.raises(Exception):
        oracle.integrate(3, 2, S.RULE_CC, S.KIND_CORNER, np.array([-0.6, -0.5, 0.3]))


# ----------------------------------------------------------------------------------------------
# oracle measurement helpers (bench.py's CPU legs): point counts, timing samples, FP64 build
# ----------------------------------------------------------------------------------------------
@pytest.mark.parametrize("i", [1, 2, 3, 4, 5])
def test_count_only_walk_equals_generating_function(i):
    """count_only walks the same multi-indices as the evaluation without evaluating: its count is
    n_d^q = [z^e] G(z)^d summed over the band, and oracle.n_points (bench's total)
    is the same number."""
    p = S.baseline_config(i)
    n = oracle.count_points(p)
    assert n == pins.n_points(p.rule, p.d, p.L) == oracle.n_points(p)
    if i <= 2:
        assert n == oracle.integrate_problem(p, eval_mode=1).npoints


def test_timing_sample_is_a_subset_spread_over_the_tree():
    """The CPU timing sample (every s-th depth-2 subtree) evaluates exactly the points count_only
    selects, far fewer than the whole, from subtrees across the whole depth-1 range."""
    p = S.baseline_config(5)
    r, stride, total = oracle.timing_sample(p, int(2e6))
    assert stride > 1 and total == 27521113876
    assert r.npoints == oracle.count_points(p, stride=stride, include_root=False)
    assert 0.5e6 < r.npoints < 8e6
    # the sample reaches the tail of the depth-1 range as well as its head: a shard that holds only
    # the last third of the depth-1 prefixes still contains sampled points
    nd1 = oracle.depth1_count(p)
    assert oracle.count_points(p, stride=stride, lo=2 * nd1 // 3, hi=nd1, include_root=False) > 0
    assert oracle.count_points(p, stride=stride, lo=0, hi=nd1 // 3, include_root=False) > 0
    # stride 1 is the ordinary (unsampled) evaluation
    q = S.baseline_config(1)
    assert oracle.integrate_problem(q, stride=1).text == oracle.integrate_problem(q).text


@pytest.mark.parametrize("i,bound", [(1, 1e-14), (2, 1e-11)])
def test_fp64_build_is_the_same_sum_in_double(i, bound):
    """The FP64 instantiation (-DSGO_FP64) sums the same points in double: it agrees with the quad
    oracle to the conditioning of Eq 2.6 (kappa * 2^-53: c1 kappa 128, c2 kappa <= 1.2e5, SURVEY.md
    §8c) and reports the same point count."""
    p = S.baseline_config(i)
    a = oracle.integrate_problem(p, eval_mode=1)
    b = oracle.integrate_problem(p, eval_mode=1, fp64=True)
    assert a.npoints == b.npoints
    assert b.lo == 0.0 or abs(b.lo) <= abs(b.hi) * 2 ** -52
    assert abs((mp.mpf(b.hi) - qval(a)) / qval(a)) < bound
