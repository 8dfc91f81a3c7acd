"""CPU-side checks of the C ABI library (no compute calls need a GPU here):
symbols exported vs include/sg_b200.h, host rule tables vs the oracle's (bit-identical, reading R5),
host plan counts vs the generating-function point counts, shard partitions, errors."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import pins
import sg_configs as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2210_14313_b200 import build as B
    B.build()
    from paper_2210_14313_b200._lib import lib
    return lib()


def test_header_symbols_exported(L):
    hdr = open(os.path.join(ROOT, "include", "sg_b200.h")).read()
    names = set(re.findall(r"\b(sg_[a-z_]+)\s*\(", hdr))
    assert len(names) >= 10
    for n in names:
        assert hasattr(L, n), n
    from paper_2210_14313_b200._lib import SYMBOLS
    assert set(SYMBOLS) == names


def _rule(L, rule, level):
    n = pins.node_count(rule, level)
    x = np.zeros(n)
    w = np.zeros(n)
    dp = ctypes.POINTER(ctypes.c_double)
    rc = L.sg_rule_table(rule, level, x.ctypes.data_as(dp), w.ctypes.data_as(dp))
    return rc, x, w


@pytest.mark.parametrize("rule,levels", [(S.RULE_CC, range(1, 11)), (S.RULE_GL, range(1, 30)),
                                         (S.RULE_TRAP, range(1, 21)), (S.RULE_GP, range(1, 30))])
def test_library_rules_bit_identical_to_oracle(L, rule, levels):
    for l in levels:
        rc, x, w = _rule(L, rule, l)
        assert rc == len(x)
        ox, ow = oracle.rule(rule, l)
        assert np.array_equal(x, ox), (rule, l, x - ox)
        assert np.array_equal(w, ow), (rule, l, w - ow)


def test_rule_table_limits(L):
    assert _rule(L, S.RULE_CC, 13)[0] == -2    # SG_EUNSUPPORTED beyond CC level 12
    assert _rule(L, 5, 2)[0] == -1             # no rule 5: SG_EINVAL
    assert _rule(L, S.RULE_TRAP, 20)[0] == (1 << 19) + 1   # trapezoid: exact dyadic tables to level 20
    assert _rule(L, S.RULE_TRAP, 21)[0] == -2
    assert _rule(L, S.RULE_GP, 48)[0] == 63    # 63-point Patterson rule up to level 48
    assert _rule(L, S.RULE_GP, 49)[0] == -2


def _query(L, d, q, rule, kind=0, form=0, rank=0, world=1, lo=0, hi=-1):
    from paper_2210_14313_b200._lib import sg_options
    o = sg_options(form, 0, rank, world, lo, hi)
    sp, tp = ctypes.c_ulonglong(), ctypes.c_ulonglong()
    a, b = ctypes.c_longlong(), ctypes.c_longlong()
    npass = ctypes.c_int()
    rc = L.sg_plan_query(d, q, rule, kind, ctypes.byref(o), ctypes.byref(sp), ctypes.byref(tp),
                         ctypes.byref(a), ctypes.byref(b), ctypes.byref(npass))
    return rc, sp.value, tp.value, a.value, b.value, npass.value


@pytest.mark.parametrize("i", [1, 2, 3, 4, 5])
def test_plan_point_counts_match_generating_function(L, i):
    p = S.baseline_config(i)
    rc, sp, tp, lo, hi, npass = _query(L, p.d, p.q, p.rule, p.kind)
    assert rc == 0
    assert tp == sp == pins.n_points(p.rule, p.d, p.L)
    assert npass == min(p.L, p.d)


@pytest.mark.parametrize("i,world", [(2, 3), (3, 4), (4, 8), (5, 8), (5, 2), (1, 5)])
def test_balanced_shards_partition(L, i, world):
    p = S.baseline_config(i)
    total = pins.n_points(p.rule, p.d, p.L)
    prev_hi, acc = 0, 0
    sizes = []
    for r in range(world):
        rc, sp, tp, lo, hi, _ = _query(L, p.d, p.q, p.rule, p.kind, rank=r, world=world)
        assert rc == 0 and tp == total
        assert lo == prev_hi
        prev_hi = hi
        acc += sp
        sizes.append(sp)
    assert acc == total
    nd1 = p.d * sum(pins.node_count(p.rule, l) for l in range(2, p.L + 2))
    assert prev_hi == nd1
    if total > 10 ** 8:
        # the cut balances the device-time cost model of plan.cpp (fused k_leaf2 points, generic-pass
        # points, k_leaf2 row-run prologues), so points stay within a few percent, not exactly equal
        assert max(sizes) / (total / world) < 1.10


@pytest.mark.parametrize("d,Lv,rule,form", [(5, 0, S.RULE_CC, 0), (1, 1, S.RULE_CC, 1), (1, 0, S.RULE_GL, 0),
                                           (2, 1, S.RULE_GL, 1), (3, 2, S.RULE_CC, 0), (1, 3, S.RULE_CC, 1),
                                           (4, 4, S.RULE_CC, 0), (2, 5, S.RULE_TRAP, 1)])
@pytest.mark.parametrize("world", [2, 3, 5, 8])
def test_shards_partition_tiny(L, d, Lv, rule, form, world):
    """Every world partition of a tiny problem (L = 0: only the root; d = 1; fewer depth-1 prefixes
    than ranks) counts each Smolyak point exactly once: the shard points add up to the total, the
    root sits on rank 0 only (several ranks may get an empty range starting at 0), and the host
    unranker enumerates each shard's points without duplicates across ranks."""
    from paper_2210_14313_b200 import api
    q = d + Lv
    whole = _query(L, d, q, rule, form=form)
    assert whole[0] == 0
    total = whole[2]
    acc, seen = 0, set()
    for r in range(world):
        rc, sp, tp, lo, hi, _ = _query(L, d, q, rule, form=form, rank=r, world=world)
        assert rc == 0 and tp == total
        acc += sp
        for idx in range(sp):
            cf, pt = api.sg_unrank(d, q, rule, 0, idx, form=form, rank=r, world=world)
            key = tuple(pt)
            assert key not in seen, (r, idx, key)
            seen.add(key)
    assert acc == total
    assert len(seen) == total


def test_explicit_range_counts(L):
    p = S.baseline_config(2)
    # subtree points of a depth-1 range must equal the oracle's point count for the same range
    for lo, hi in [(0, 1), (5, 17), (100, 101), (300, 360)]:
        rc, sp, *_ = _query(L, p.d, p.q, p.rule, p.kind, lo=lo, hi=hi)
        assert rc == 0
        r = oracle.integrate_problem(p, lo=lo, hi=hi, include_root=(lo == 0), eval_mode=1)
        assert sp == r.npoints


def test_errors(L):
    assert _query(L, 5, 4, S.RULE_CC)[0] == -1          # q < d: BudgetTooSmall
    assert _query(L, 0, 4, S.RULE_CC)[0] == -1
    assert _query(L, 5, 8, 7)[0] == -1                  # bad rule
    assert _query(L, 5, 8, S.RULE_CC, kind=9)[0] == -1
    assert _query(L, 5, 8, S.RULE_CC, rank=2, world=2)[0] == -1
    assert _query(L, 5, 5 + 12, S.RULE_CC)[0] == -2     # CC level 13
    assert _query(L, 1000, 1000 + 19, S.RULE_GL)[0] in (-2, -3)   # coefficient/size limits
    assert _query(L, 10 ** 5, 10 ** 5 + 8, S.RULE_CC)[0] in (-2, -3)
    assert L.sg_strerror(-3).decode().startswith("point")


# ----------------------------------------------------------------------------------------------
# K1 unranker (north-star subsystem 1): flat index -> multi-index, tensor point, coefficient
# ----------------------------------------------------------------------------------------------
def _brute_points(d, Lx, rule):
    """Independent enumeration of Eq 2.6/2.7 points: every level vector in the band, every tensor
    node index; returned as sparse tuples ((k, l, j), ...) of the active (level >= 2) coordinates."""
    import itertools
    pts = {}
    for lv in itertools.product(range(1, Lx + 2), repeat=d):
        e = sum(lv) - d
        cf = pins.coef(d, Lx, e)
        if cf == 0:
            continue
        act = [(kk, ll) for kk, ll in enumerate(lv) if ll >= 2]
        for js in itertools.product(*[range(pins.node_count(rule, ll)) for _, ll in act]):
            pts[tuple((kk, ll, jj) for (kk, ll), jj in zip(act, js))] = cf
    return pts


@pytest.mark.parametrize("d,Lx,rule", [(4, 4, S.RULE_CC), (5, 3, S.RULE_GL), (3, 5, S.RULE_CC),
                                       (2, 6, S.RULE_GL), (6, 2, S.RULE_CC)])
def test_unrank_is_a_bijection_in_lexicographic_order(L, d, Lx, rule):
    from paper_2210_14313_b200 import api
    brute = _brute_points(d, Lx, rule)
    n = pins.n_points(rule, d, Lx)
    assert len(brute) == n
    seq = []
    for i in range(n):
        cf, trip = api.sg_unrank(d, d + Lx, rule, 0, i)
        key = tuple(trip)
        assert key in brute, (i, key)
        assert cf == brute[key], (i, key)
        seq.append(key)
    assert len(set(seq)) == n                 # bijection
    assert seq == sorted(seq)                 # canonical order = lexicographic (prefix first)
    from paper_2210_14313_b200._lib import SGError
    with pytest.raises(SGError):
        api.sg_unrank(d, d + Lx, rule, 0, n)


def test_unrank_full_size_config5_samples_and_shards(L):
    from paper_2210_14313_b200 import api
    p = S.baseline_config(5)
    n = pins.n_points(p.rule, p.d, p.L)
    rng = np.random.default_rng(9)
    idx = np.sort(rng.integers(0, n, 300))
    keys = []
    for i in idx:
        cf, trip = api.sg_unrank(p.d, p.q, p.rule, p.kind, int(i))
        e = sum(l - 1 for _, l, _ in trip)
        assert cf == pins.coef(p.d, p.L, e)
        assert all(a[0] < b[0] for a, b in zip(trip, trip[1:]))
        assert all(0 <= j < pins.node_count(p.rule, l) and 2 <= l for _, l, j in trip)
        keys.append(tuple(trip))
    assert keys == sorted(keys)
    # shard r's points come from its own depth-1 range
    world = 3
    M0 = sum(pins.node_count(p.rule, l) for l in range(2, p.L + 2))
    for r in range(world):
        rc, sp, tp, lo, hi, _ = _query(L, p.d, p.q, p.rule, p.kind, rank=r, world=world)
        for i in (0, sp // 2, sp - 1):
            cf, trip = api.sg_unrank(p.d, p.q, p.rule, p.kind, int(i), rank=r, world=world)
            if not trip:
                assert r == 0 and i == 0      # the root belongs to rank 0
                continue
            k1, l1, j1 = trip[0]
            r1 = k1 * M0 + sum(pins.node_count(p.rule, l) for l in range(2, l1)) + j1
            assert lo <= r1 < hi


def test_ctypes_structs_match_header(tmp_path):
    """The Python marshalling structs have the C layout of include/sg_b200.h (size and every field
    offset), compiled here with gcc from the header itself."""
    import subprocess
    from paper_2210_14313_b200._lib import sg_integrand_desc, sg_options
    src = tmp_path / "layout.c"
    fields = {"sg_options": [f for f, _ in sg_options._fields_],
              "sg_integrand_desc": [f for f, _ in sg_integrand_desc._fields_]}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "sg_b200.h"', 'int main(void) {']
    for st, fs in fields.items():
        lines.append(f'printf("{st} %zu\\n", sizeof({st}));')
        for f in fs:
            lines.append(f'printf("{st}.{f} %zu\\n", offsetof({st}, {f}));')
    lines += ["return 0;", "}"]
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = dict(l.split() for l in subprocess.check_output([str(exe)], text=True).splitlines())
    for st, cls in (("sg_options", sg_options), ("sg_integrand_desc", sg_integrand_desc)):
        assert int(got[st]) == ctypes.sizeof(cls), st
        for f in fields[st]:
            assert int(got[f"{st}.{f}"]) == getattr(cls, f).offset, (st, f)


@pytest.mark.parametrize("cfg,rank,world", [(4, 0, 1), (4, 0, 8), (4, 7, 8), (4, 3, 4), (5, 0, 1), (5, 5, 8),
                                            (3, 0, 1), (3, 1, 2), (2, 0, 1)])
def test_fused_task_list_tiles_every_row_once(L, tmp_path, cfg, rank, world):
    """The fused pass's task list (plan.cpp: k_mid grouping, long-task row pieces, the guided tail's
    cuts) covers every (parent chunk, k_mid, leaf row) of the shard exactly once: for each chunk the
    k_mids form one contiguous range ending at d - 2, and each k_mid's row ranges, over all tasks and
    lane groups, tile [k_mid + 1, d) without gap or overlap.  (A task lost or claimed twice changes
    the integral; this pins the host side of it without a GPU.)"""
    p = S.baseline_config(cfg)
    fn = str(tmp_path / "tasks.txt")
    os.environ["SG_B200_DUMP_TASKS"] = fn
    try:
        rc = _query(L, p.d, p.q, p.rule, p.kind, rank=rank, world=world)[0]
    finally:
        del os.environ["SG_B200_DUMP_TASKS"]
    assert rc == 0
    lines = open(fn).read().split("\n")
    G, d, CH = map(int, lines[0].split())
    cover = {}   # (chunk first, k_mid) -> list of row intervals
    ntask = 0
    for ln in lines[1:]:
        if not ln:
            continue
        rows, first, ka, kb, kp0, kp1 = map(int, ln.split())
        assert first % CH == 0 and 0 <= ka < kb <= d - 1 and 0 <= kp0 < kp1 <= d
        ntask += 1
        for g in range(G):
            for km in range(ka + g, kb, G):
                r0, r1 = max(km + 1, kp0), min(kp1, d)
                if r1 > r0:
                    cover.setdefault((first, km), []).append((r0, r1))
    assert ntask > 0
    kms = {}
    for (first, km), iv in cover.items():
        iv.sort()
        assert iv[0][0] == km + 1 and iv[-1][1] == d, (first, km, iv[:3])
        for a, b in zip(iv, iv[1:]):
            assert a[1] == b[0], (first, km, a, b)   # no gap, no overlap
        kms.setdefault(first, []).append(km)
    for first, ks in kms.items():
        ks.sort()
        assert ks == list(range(ks[0], d - 1)), (first, ks[0], len(ks))
