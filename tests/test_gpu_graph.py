"""The step as a CUDA graph (the launch mode bench.py times): a replay gives the same bits as the
stream-launched sg_integrate + sg_finalize, and with profiling on, the captured event-record nodes
time every launch of the replay (sg_profile_read)."""
import pytest

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


@pytest.mark.parametrize("i,kw", [(2, {}), (3, {}), (2, {"merge": 1}), (3, {"method": 1})])
@pytest.mark.parametrize("profile", [False, True])
def test_graph_replay_bitwise(api, i, kw, profile):
    import torch
    p = S.baseline_config(i)
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, **kw)
    ref = plan.integrate_host()
    g = plan.capture_graph(profile=profile)
    for _ in range(3):
        plan.result().zero_()
        g.replay()
        torch.cuda.synchronize()
        r = plan.result().cpu().numpy()
        assert (float(r[0]), float(r[1])) == ref
    if profile:
        ms = plan.profile_read()
        assert len(ms) == (4 if kw.get("method") else 4 + len(plan.passes()) - 1)
        assert all(t >= 0.0 for t in ms) and sum(ms) > 0.0
    plan.close()


def test_graph_sharded_partials(api):
    """A rank's captured integrate (no finalize) writes the same partial as the stream call."""
    import torch
    p = S.baseline_config(3)
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=1, world=3)
    ref = plan.sg_integrate().clone()
    torch.cuda.synchronize()
    g = plan.capture_graph(finalize=False, profile=True)
    plan._out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(plan._out, ref)
    plan.close()
