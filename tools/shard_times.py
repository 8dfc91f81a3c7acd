"""Per-shard device time of the rank plans of a world, run one after another on ONE GPU.

    python tools/shard_times.py [config] [worlds...]

The shards are independent (no data-path exchange), so the slowest shard's time is the N-GPU
step time up to the 16-byte all-gather; this projects strong-scaling efficiency t1 / (N max_r t_r)
from one device.  Times: CUDA events around a CUDA-graph replay of sg_integrate (bench.py's launch
configuration), best of 5, L2 flushed in between.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import sg_configs as S  # noqa: E402
from paper_2210_14313_b200 import api  # noqa: E402


def time_plan(plan, flush, reps=5):
    """Best of `reps` CUDA-graph replays of sg_integrate (the launch configuration bench.py times)."""
    for _ in range(2):
        plan.sg_integrate()
    g = plan.capture_graph(finalize=False)
    best = None
    for _ in range(reps):
        if not os.environ.get("SHARD_NOFLUSH"):   # A/B: warm L2 (code and tables resident)
            flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    return best


def phases(plan, flush, reps=5):
    """Per-launch device ms (sg_profile_read: events captured as graph nodes) of the best of `reps`
    CUDA-graph replays."""
    g = plan.capture_graph(finalize=False, profile=True)
    best = None
    for _ in range(reps):
        if not os.environ.get("SHARD_NOFLUSH"):
            flush.fill_(1.0)
        torch.cuda.synchronize()
        g.replay()
        ms = plan.profile_read()
        if best is None or sum(ms) < sum(best):
            best = ms
    plan.profile_enable(False)
    return best


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    worlds = [int(a) for a in sys.argv[2:]] or [2, 4, 8]
    p = S.baseline_config(cfg)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    whole = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u)
    t1 = time_plan(whole, flush)
    if os.environ.get("SHARD_PHASES"):
        print(f"  world=1 launches ms: {[round(x, 4) for x in phases(whole, flush)]}")
    whole.close()
    print(f"{p.name} world=1 {t1:.4f} ms")
    for world in worlds:
        ts, pts = [], []
        for r in range(world):
            sp = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=r, world=world)
            ts.append(time_plan(sp, flush))
            pts.append(sp.points()[0])
            sp.close()
        mx = max(ts)
        if os.environ.get("SHARD_PHASES"):
            r = ts.index(mx)
            sp = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=r, world=world)
            print(f"  rank {r} launches ms: {[round(x, 4) for x in phases(sp, flush)]}")
            sp.close()
        print(f"{p.name} world={world} max={mx:.4f} ms mean={sum(ts) / world:.4f} "
              f"time_imbalance={mx / (sum(ts) / world):.4f} point_imbalance="
              f"{max(pts) / (sum(pts) / world):.4f} projected_eff={t1 / (world * mx):.4f} "
              f"shards_ms={[round(t, 3) for t in ts]}", flush=True)


if __name__ == "__main__":
    main()
