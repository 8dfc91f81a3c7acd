"""Device K1 unranker and per-point evaluation (sg_eval_points) at the full BASELINE sizes.

Sampled outputs the oracle can compute one by one: for seeded random flat point indices of the full
configs 4-5, the device unranker must return exactly the host unranker's (multi-index, node,
coefficient), and each point's term coefficient * w * f(x), evaluated on the device from the factor
table, must equal the oracle's (__float128 f at the same point, its own rule weights) to 1e-15.
Summing every point's term of a small problem reproduces the integral (an evaluation path that
shares nothing with the prefix tree's partial products).
"""
import mpmath as mp
import numpy as np
import pytest

import oracle
import pins
import sg_configs as S

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


def _oracle_term(p, t, trip, coef):
    x = np.full(p.d, 0.5)
    wprod = mp.mpf(1)
    for (k, l, j) in trip:
        xs, ws = oracle.rule(p.rule, l)
        x[k] = xs[j]
        wprod *= mp.mpf(ws[j])
    a, _ = oracle.eval_point(p.kind, p.c, p.w, p.u, x)
    return mp.mpf(coef) * wprod * (mp.mpf(a[0]) + mp.mpf(a[1]))


@pytest.mark.parametrize("i,world,rank", [(5, 1, 0), (4, 1, 0), (5, 8, 7), (4, 3, 1)])
def test_device_unranker_and_point_terms_full_size(api, i, world, rank):
    p = S.baseline_config(i)
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=rank, world=world)
    shard, total = plan.points()
    rng = np.random.default_rng(100 + i + rank)
    idx = np.unique(np.concatenate([[0, 1, shard - 1], rng.integers(0, shard, 60)]))
    pts, terms = plan.eval_points(idx)
    pts, terms = pts.cpu().numpy(), terms.cpu().numpy()
    with mp.workdps(40):
        for n, ix in enumerate(idx):
            cf, trip = api.sg_unrank(p.d, p.q, p.rule, p.kind, int(ix), rank=rank, world=world)
            t = int(pts[n, 0])
            got = [tuple(int(v) for v in pts[n, 1 + 3 * m: 4 + 3 * m]) for m in range(t)]
            assert t == len(trip) and got == [tuple(tr) for tr in trip], (ix, got, trip)
            want = _oracle_term(p, t, trip, cf)
            have = mp.mpf(terms[n, 0]) + mp.mpf(terms[n, 1])
            assert abs(have - want) <= 1e-15 * abs(want), (ix, have, want)
    plan.close()


@pytest.mark.parametrize("case", [("c1", None), ("rand", (140, 6, 4, S.RULE_GL, S.KIND_OSC)),
                                  ("rand", (141, 9, 3, S.RULE_CC, S.KIND_PEAK)),
                                  ("merged", (142, 7, 4, S.RULE_CC, S.KIND_OSC))])
def test_sum_of_point_terms_is_the_integral(api, case):
    p = S.baseline_config(1) if case[0] == "c1" else S.random_problem(*case[1])
    kw = {"merge": api.MERGE_MIDPOINT} if case[0] == "merged" else {}
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, **kw)
    shard, _ = plan.points()
    assert shard <= 300_000
    _, terms = plan.eval_points(np.arange(shard))
    terms = terms.cpu().numpy()
    with mp.workdps(40):
        s = mp.fsum(mp.mpf(a) + mp.mpf(b) for a, b in terms)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    assert abs(s - ref) <= 1e-15 * abs(ref)
    hi, lo = plan.integrate_host()
    assert abs(s - (mp.mpf(hi) + mp.mpf(lo))) <= 1e-15 * abs(ref)
    plan.close()


def test_eval_points_out_of_range_and_errors(api):
    from paper_2210_14313_b200._lib import SGError
    p = S.baseline_config(2)
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u)
    shard, _ = plan.points()
    pts, terms = plan.eval_points([shard, shard + 5])
    assert (pts[:, 0].cpu().numpy() == -1).all() and np.isnan(terms.cpu().numpy()).all()
    plan.close()
    q = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, method=api.METHOD_COLLAPSE)
    with pytest.raises(SGError):
        q.eval_points([0])
    q.close()


@pytest.mark.parametrize("case", [("c1", None), ("c2", None), ("rand", (150, 12, 4, S.RULE_GP, S.KIND_GAUSS)),
                                  ("merged", (151, 8, 5, S.RULE_CC, S.KIND_OSC)),
                                  ("delta", (152, 30, 3, S.RULE_GL, S.KIND_PEAK))])
def test_plain_method_vs_oracle(api, case):
    """SG_METHOD_PLAIN (every point unranked and evaluated on its own, the paper's SG baseline)."""
    p = S.baseline_config(int(case[0][1])) if case[1] is None else S.random_problem(*case[1])
    kw = {"method": api.METHOD_PLAIN}
    if case[0] == "merged":
        kw["merge"] = api.MERGE_MIDPOINT
    if case[0] == "delta":
        kw["form"] = api.FORM_DELTA
    hi, lo = api.integrate(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u, **kw)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    assert abs(mp.mpf(hi) + mp.mpf(lo) - ref) <= 1e-15 * abs(ref)


def test_plain_method_config4_full_size(api):
    import json
    import os
    p = S.baseline_config(4)
    hi, lo = api.integrate(p.d, p.L, p.rule, p.kind, p.c, p.w, p.u, method=api.METHOD_PLAIN)
    golden = os.path.join(os.path.dirname(__file__), "golden", "oracle_full.json")
    ref = mp.mpf(json.load(open(golden))["values"]["c4"]["text"])
    assert abs(mp.mpf(hi) + mp.mpf(lo) - ref) <= 1e-15 * abs(ref)
