"""Step time from an idle GPU: stream launches (profiling off / on) vs one CUDA-graph replay.

    python tools/graph_gain.py [config] [world] [rank]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import sg_configs as S  # noqa: E402
from paper_2210_14313_b200 import api  # noqa: E402


def best(fn, flush, reps=7):
    out = []
    for _ in range(reps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out), sorted(out)[len(out) // 2]


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    rank = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    p = S.baseline_config(cfg)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=rank, world=world)

    def step():
        plan.sg_finalize(plan.sg_integrate(), 1)

    for _ in range(3):
        step()
    a = best(step, flush)
    plan.profile_enable(True)
    b = best(step, flush)
    g = plan.capture_graph()
    c = best(g.replay, flush)
    print(f"c{cfg} world={world} rank={rank}: stream {a[0]:.4f}/{a[1]:.4f} ms  profiled {b[0]:.4f}/{b[1]:.4f}"
          f"  graph {c[0]:.4f}/{c[1]:.4f} (min/median)")


if __name__ == "__main__":
    main()
