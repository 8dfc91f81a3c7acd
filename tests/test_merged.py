"""Midpoint-merged evaluation (SG_MERGE_MIDPOINT, Eq 2.8 and
the Fig 2.1 remark "we would avoid the repeated points").

Every CC level (and every odd GL level) contains the midpoint 1/2, so the Eq 2.6/2.7 point set
repeats each point once per choice of levels of its midpoint coordinates.  The merged tree carries
only non-midpoint nodes and gives a node of depth t and excess b the coefficient
C'(t, b) = sum_{e>=b} c(e) [z^{e-b}] M(z)^{d-t}.

CPU pins (independent of the library's arithmetic): the merged point set, its order, and every
node's merged coefficient against a brute-force regrouping of the itertools enumeration of
Eq 2.6/2.7.  GPU: the merged integral against the oracle (same value: an exact regrouping).
"""
import itertools
from fractions import Fraction

import mpmath as mp
import numpy as np
import pytest

import oracle
import pins
import sg_configs as S


@pytest.fixture(scope="module")
def L():
    from paper_2210_14313_b200 import build as B
    B.build()
    from paper_2210_14313_b200._lib import lib
    return lib()


def _query(L, d, q, rule, kind=0, form=0, rank=0, world=1, lo=0, hi=-1, merge=1):
    import ctypes
    from paper_2210_14313_b200._lib import sg_options
    o = sg_options(form, 0, rank, world, lo, hi, merge)
    sp, tp = ctypes.c_ulonglong(), ctypes.c_ulonglong()
    a, b = ctypes.c_longlong(), ctypes.c_longlong()
    npass = ctypes.c_int()
    rc = L.sg_plan_query(d, q, rule, kind, ctypes.byref(o), ctypes.byref(sp), ctypes.byref(tp),
                         ctypes.byref(a), ctypes.byref(b), ctypes.byref(npass))
    return rc, sp.value, tp.value, a.value, b.value


def _delta_entries(rule, l):
    """Delta^l = J^l - J^{l-1} on the union support (reading R12): {x: Fraction weight}."""
    x1, w1 = oracle.rule(rule, l)
    ent = {float(x): Fraction(float(w)) for x, w in zip(x1, w1)}
    if l >= 2:
        x0, w0 = oracle.rule(rule, l - 1)
        for x, w in zip(x0, w0):
            ent[float(x)] = ent.get(float(x), Fraction(0)) - Fraction(float(w))
    return ent


def _level_entries(rule, l, form):
    """Entries (x, exact weight) of level l in the form's table order (ascending x)."""
    if form == 0:
        x, w = oracle.rule(rule, l)
        return [(float(a), Fraction(float(b))) for a, b in zip(x, w)]
    return sorted(_delta_entries(rule, l).items())


def _brute_merged(d, Lx, rule, form):
    """Regroup every Eq 2.6/2.7 point (form 0) or Delta-form term (form 1) by its non-midpoint
    actives.  Returns {key: merged weight factor} where key = ((k, l, j'), ...) with j' the index
    among the level's non-midpoint entries, and the factor = sum over the group of
    coefficient * prod_{midpoint actives} w^l(1/2) (exact rationals of the double weights)."""
    ents = {l: _level_entries(rule, l, form) for l in range(2, Lx + 2)}
    groups = {}
    for lv in itertools.product(range(1, Lx + 2), repeat=d):
        e = sum(lv) - d
        if e > Lx:
            continue
        cf = pins.coef(d, Lx, e) if form == 0 else 1   # zero below the band (d <= L): the node
        # still exists in the merged tree, with merged coefficient 0 if no copy has a nonzero one
        act = [(k, l) for k, l in enumerate(lv) if l >= 2]
        for js in itertools.product(*[range(len(ents[l])) for _, l in act]):
            key, fac = [], Fraction(cf)
            for (k, l), j in zip(act, js):
                x, w = ents[l][j]
                if x == 0.5:
                    fac *= w
                else:
                    jn = j - sum(1 for xx, _ in ents[l][:j] if xx == 0.5)
                    key.append((k, l, jn))
            key = tuple(key)
            groups[key] = groups.get(key, Fraction(0)) + fac
    return groups


@pytest.mark.parametrize("d,Lx,rule,form", [(4, 4, S.RULE_CC, 0), (5, 3, S.RULE_GL, 0),
                                            (3, 5, S.RULE_CC, 0), (2, 6, S.RULE_GL, 0),
                                            (6, 2, S.RULE_CC, 0), (4, 3, S.RULE_CC, 1),
                                            (3, 4, S.RULE_GL, 1)])
def test_merged_unrank_bijection_and_coefficients(L, d, Lx, rule, form):
    from paper_2210_14313_b200 import api
    groups = _brute_merged(d, Lx, rule, form)
    rc, sp, tp, *_ = _query(L, d, d + Lx, rule, form=form)
    assert rc == 0 and sp == tp == len(groups)
    seq = []
    for i in range(tp):
        cf, trip = api.sg_unrank(d, d + Lx, rule, 0, i, form=form, merge=1)
        key = tuple(trip)
        assert key in groups, (i, key)
        # the library's C'(t, b) (hi part) must be the group's coefficient sum (the non-midpoint
        # weights are common to the group and live in the factor table)
        cref = groups[key]
        assert abs(Fraction(cf) - cref) <= abs(cref) * Fraction(1, 2 ** 52) + Fraction(1, 10 ** 300), \
            (key, cf, float(cref))
        seq.append(key)
    assert len(set(seq)) == len(seq) and seq == sorted(seq)


def _merged_count_gf(rule, d, Lx):
    """Tree nodes of the merged tree: sum_t C(d, t) [z^{<=L}] G~(z)^t, G~ = sum_l (n_l - mid_l) z^{l-1}."""
    from math import comb
    g = [0] * (Lx + 1)
    for l in range(2, Lx + 2):
        x, _ = oracle.rule(rule, l)
        g[l - 1] = int(sum(1 for v in x if v != 0.5))
    tot, pw = 0, [1] + [0] * Lx
    for t in range(0, min(d, Lx) + 1):
        tot += comb(d, t) * sum(pw)
        nxt = [0] * (Lx + 1)
        for i, a in enumerate(pw):
            for j, b in enumerate(g):
                if i + j <= Lx:
                    nxt[i + j] += a * b
        pw = nxt
    return tot


@pytest.mark.parametrize("i", [1, 2, 3, 4, 5])
def test_merged_point_counts_full_size(L, i):
    p = S.baseline_config(i)
    rc, sp, tp, *_ = _query(L, p.d, p.q, p.rule, p.kind)
    assert rc == 0 and sp == tp == _merged_count_gf(p.rule, p.d, p.L)
    assert tp < pins.n_points(p.rule, p.d, p.L)


@pytest.mark.parametrize("i,world", [(5, 8), (4, 3), (3, 4)])
def test_merged_shards_partition(L, i, world):
    p = S.baseline_config(i)
    tot, prev = 0, 0
    for r in range(world):
        rc, sp, tp, lo, hi = _query(L, p.d, p.q, p.rule, p.kind, rank=r, world=world)
        assert rc == 0 and lo == prev
        prev = hi
        tot += sp
    assert tot == tp


# ----------------------------------------------------------------------------------------------
# GPU: merged integral vs the oracle (Eq 2.6 in __float128) — same value
# ----------------------------------------------------------------------------------------------
GATE, HEALTH = 1e-12, 1e-15


@pytest.fixture(scope="module")
def api():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2210_14313_b200 import build as B
    B.build()
    from paper_2210_14313_b200 import api as A
    return A


def _rel(a, b):
    return abs((a - b) / b) if b != 0 else abs(a - b)


def _gpu(api, p, **kw):
    hi, lo = api.integrate(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u, merge=1, **kw)
    return mp.mpf(hi) + mp.mpf(lo), hi


def _check(api, p, **kw):
    ref = oracle.integrate_problem(p, eval_mode=1)
    v, hi = _gpu(api, p, **kw)
    r = _rel(v, mp.mpf(ref.text))
    assert r <= GATE, (p.name, float(r), hi, ref.text)
    assert r <= HEALTH, (p.name, float(r))


@pytest.mark.gpu
@pytest.mark.parametrize("i", [1, 2, 3])
def test_gpu_merged_small_configs(api, i):
    _check(api, S.baseline_config(i))


@pytest.mark.gpu
@pytest.mark.parametrize("i", [4, 5])
def test_gpu_merged_full_size(api, i):
    import json
    import os
    p = S.baseline_config(i)
    v, _ = _gpu(api, p)
    assert _rel(v, pins.dp_value(p)) <= HEALTH
    g = os.path.join(os.path.dirname(__file__), "golden", "oracle_full.json")
    vals = json.load(open(g))["values"]
    if p.name in vals:
        assert _rel(v, mp.mpf(vals[p.name]["text"])) <= HEALTH


MCASES = [
    (71, 1, 5, S.RULE_CC, S.KIND_EXP), (72, 2, 7, S.RULE_GL, S.KIND_OSC),
    (73, 3, 6, S.RULE_CC, S.KIND_PEAK), (74, 5, 1, S.RULE_CC, S.KIND_OSC),
    (75, 37, 2, S.RULE_CC, S.KIND_GAUSS), (76, 33, 3, S.RULE_GL, S.KIND_PEAK),
    (77, 65, 3, S.RULE_CC, S.KIND_OSC), (78, 7, 6, S.RULE_GL, S.KIND_EXP),
    (79, 12, 5, S.RULE_CC, S.KIND_OSC), (80, 130, 4, S.RULE_CC, S.KIND_OSC),
    (81, 20, 4, S.RULE_GL, S.KIND_GAUSS), (82, 4, 0, S.RULE_CC, S.KIND_EXP),
    (86, 9, 5, S.RULE_GP, S.KIND_OSC), (87, 40, 3, S.RULE_TRAP, S.KIND_GAUSS),
]


@pytest.mark.gpu
@pytest.mark.parametrize("form", [0, 1])
@pytest.mark.parametrize("seed,d,Lx,rule,kind", MCASES)
def test_gpu_merged_random(api, form, seed, d, Lx, rule, kind):
    _check(api, S.random_problem(seed, d, Lx, rule, kind), form=form)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["fused", "nofuse", "generic"])
@pytest.mark.parametrize("seed,d,Lx,rule,kind", [(83, 40, 3, S.RULE_CC, S.KIND_OSC),
                                                  (84, 75, 4, S.RULE_CC, S.KIND_GAUSS),
                                                  (85, 33, 4, S.RULE_GL, S.KIND_OSC)])
def test_gpu_merged_last_pass_variants(api, monkeypatch, mode, seed, d, Lx, rule, kind):
    if mode == "fused":
        monkeypatch.setenv("SG_B200_FUSE", "1")
    if mode in ("nofuse", "generic"):
        monkeypatch.setenv("SG_B200_NOFUSE", "1")
    if mode == "generic":
        monkeypatch.setenv("SG_B200_GENERIC_LEAF", "1")
    _check(api, S.random_problem(seed, d, Lx, rule, kind))


@pytest.mark.gpu
def test_gpu_merged_shards_sum_to_whole(api):
    import torch
    p = S.baseline_config(5)
    whole = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, merge=1)
    a = whole.integrate_host()
    assert a == whole.integrate_host()
    world = 3
    parts = []
    for r in range(world):
        sp = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=r, world=world, merge=1)
        parts.append(sp.sg_integrate().clone())
        torch.cuda.synchronize()
        sp.close()
    res = whole.sg_finalize(torch.cat(parts), world).cpu().numpy()
    assert _rel(mp.mpf(res[0]) + mp.mpf(res[1]), mp.mpf(a[0]) + mp.mpf(a[1])) <= 1e-20
    whole.close()
