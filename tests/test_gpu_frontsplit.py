"""Split frontier passes (sg_kernels.cu: the write-only run kernel k_front for the stored children — their
terms from the stored products — and, concurrently on the side stream, a leaf-only k_leaf for the other
children):
parity against the __float128 oracle with the split forced on every writing pass (fused and unfused
plans, all rules and kinds, sharded), and the full-size unfused config 5 (the 4.3 GB frontier) against
the stored oracle value."""
import json
import os

import mpmath as mp
import pytest

import oracle
import sg_configs as S

pytestmark = pytest.mark.gpu
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


def _sum(api, p, world, **kw):
    tot = mp.mpf(0)
    for r in range(world):
        plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=r, world=world, **kw)
        hi, lo = plan.integrate_host()
        plan.close()
        tot += mp.mpf(hi) + mp.mpf(lo)
    return tot


@pytest.mark.parametrize("nofuse", [False, True])
@pytest.mark.parametrize("seed,d,L,rule,kind", [(91, 30, 4, S.RULE_CC, S.KIND_OSC), (92, 12, 6, S.RULE_CC, S.KIND_EXP),
                                                (93, 20, 5, S.RULE_GL, S.KIND_PEAK), (94, 40, 4, S.RULE_CC, S.KIND_GAUSS),
                                                (95, 9, 6, S.RULE_GP, S.KIND_OSC), (96, 17, 5, S.RULE_TRAP, S.KIND_OSC)])
def test_forced_split_vs_oracle(api, monkeypatch, nofuse, seed, d, L, rule, kind):
    monkeypatch.setenv("SG_B200_FRONT_SPLIT", "1")
    if nofuse:
        monkeypatch.setenv("SG_B200_NOFUSE", "1")
    p = S.random_problem(seed, d, L, rule, kind)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    for world in (1, 3):
        v = _sum(api, p, world)
        assert abs((v - ref) / ref) <= 1e-15, (world, float(abs((v - ref) / ref)))
    # the merged tree and the delta form take the same split
    assert abs((_sum(api, p, 1, form=1) - ref) / ref) <= 1e-15


def test_unfused_config5_split_full_size(api, monkeypatch):
    monkeypatch.setenv("SG_B200_NOFUSE", "1")
    p = S.baseline_config(5)
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u)
    hi, lo = plan.integrate_host()
    plan.close()
    ref = mp.mpf(json.load(open(GOLDEN))["values"]["c5"]["text"])
    assert abs((mp.mpf(hi) + mp.mpf(lo) - ref) / ref) <= 1e-15
