"""Scheduling switches of the fused pass that must not change the integral:

* the concurrent pass L-2 beside the fused pass at world 1 (fork1: on by default when the fused grid
  leaves SMs free) — same partial slots, same fixed-order reduction, so bitwise-equal results;
* the guided tail of the fused task list (plan.cpp: tasks cut to <= remaining rows / resident warps)
  — a different grouping of the same terms, so equal to the oracle within the parity bound, at
  every shard of a world;
* the head kernel's helper warp (B's transcendental beside the factor entries) — the base value and
  the factor table against the separate K0 launch (SG_B200_NOHEAD=1), bitwise.
"""
import mpmath as mp
import numpy as np
import pytest

import oracle
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


def _plan(api, p, **kw):
    return api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, **kw)


def _value(api, p, world=1, **kw):
    tot = mp.mpf(0)
    for r in range(world):
        plan = _plan(api, p, rank=r, world=world, **kw)
        hi, lo = plan.integrate_host()
        plan.close()
        tot += mp.mpf(hi) + mp.mpf(lo)
    return tot


@pytest.mark.parametrize("cfg", [1, 2])
def test_fork_at_world1_bitwise(api, monkeypatch, cfg):
    p = S.baseline_config(cfg)
    vals = {}
    for f in ("0", "1"):
        monkeypatch.setenv("SG_B200_FORK1", f)
        plan = _plan(api, p)
        vals[f] = plan.integrate_host()
        plan.close()
    assert vals["0"] == vals["1"]


@pytest.mark.parametrize("seed,d,L,rule,kind", [(201, 60, 3, S.RULE_CC, S.KIND_GAUSS),
                                                (202, 40, 4, S.RULE_GL, S.KIND_PEAK),
                                                (203, 30, 4, S.RULE_CC, S.KIND_EXP),
                                                (204, 25, 4, S.RULE_CC, S.KIND_OSC)])
@pytest.mark.parametrize("guide", ["0", "1", "4"])
def test_guided_tail_vs_oracle(api, monkeypatch, seed, d, L, rule, kind, guide):
    monkeypatch.setenv("SG_B200_GUIDE", guide)
    monkeypatch.setenv("SG_B200_GUIDE_MIN", "4")
    p = S.random_problem(seed, d, L, rule, kind)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    for world in (1, 4):
        v = _value(api, p, world)
        assert abs((v - ref) / ref) <= 1e-15, (world, float(abs((v - ref) / ref)))


@pytest.mark.parametrize("kind", [S.KIND_EXP, S.KIND_OSC, S.KIND_PEAK, S.KIND_GAUSS])
def test_head_helper_warp_matches_k0(api, monkeypatch, kind):
    p = S.random_problem(210 + kind, 37, 3, S.RULE_CC, kind)
    out = {}
    for nh in ("0", "1"):
        monkeypatch.setenv("SG_B200_NOHEAD", nh)
        plan = _plan(api, p)
        plan.integrate_host()
        tab, base = plan.debug_tables()
        out[nh] = (np.asarray(tab).copy(), np.asarray(base).copy())
        plan.close()
    assert np.array_equal(out["0"][0], out["1"][0])
    assert np.array_equal(out["0"][1], out["1"][1])
