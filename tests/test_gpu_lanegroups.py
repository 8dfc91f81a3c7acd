"""k_leaf2 lane groups (small shards of the real kinds: 32 / G parents per chunk, G k_mid groups per
warp, plan.cpp leaf2_groups): parity against the __float128 oracle with every G forced, and the
8-shard and 4-shard partitions of config 4 (where ranks 0-2 choose G > 1) summing to the stored
full-size oracle value."""
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


def _value(api, p, rank=0, world=1):
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=rank, world=world)
    hi, lo = plan.integrate_host()
    plan.close()
    return mp.mpf(hi) + mp.mpf(lo)


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("seed,d,L,rule,kind", [(71, 60, 3, S.RULE_CC, S.KIND_GAUSS),
                                                (72, 40, 4, S.RULE_GL, S.KIND_PEAK),
                                                (73, 97, 3, S.RULE_CC, S.KIND_EXP),
                                                (74, 33, 4, S.RULE_TRAP, S.KIND_GAUSS)])
def test_forced_lane_groups_vs_oracle(api, monkeypatch, G, seed, d, L, rule, kind):
    monkeypatch.setenv("SG_B200_LEAF2_GROUPS", str(G))
    p = S.random_problem(seed, d, L, rule, kind)
    ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
    for world in (1, 3):
        v = sum((_value(api, p, r, world) for r in range(world)), mp.mpf(0))
        assert abs((v - ref) / ref) <= 1e-15, (G, world, float(abs((v - ref) / ref)))


@pytest.mark.parametrize("world", [4, 8])
def test_config4_shards_with_lane_groups_sum_to_golden(api, world):
    p = S.baseline_config(4)
    ref = mp.mpf(json.load(open(GOLDEN))["values"]["c4"]["text"])
    v = sum((_value(api, p, r, world) for r in range(world)), mp.mpf(0))
    assert abs((v - ref) / ref) <= 1e-15
