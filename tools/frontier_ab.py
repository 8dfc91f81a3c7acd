"""Frontier-kernel timing (the unfused step, SG_B200_NOFUSE=1): per-launch device ms of graph replays
(profile events as graph nodes), the write pass's algorithmic bytes and GB/s.

    SG_B200_NOFUSE=1 python tools/frontier_ab.py [config] [reps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import sg_configs as S  # noqa: E402
from paper_2210_14313_b200 import api  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    p = S.baseline_config(cfg)
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u)
    passes = plan.passes()
    wpass = max(range(1, len(passes)), key=lambda i: passes[i].written)
    rec = (32 if p.kind == S.KIND_OSC else 16) + 4
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(2):
        plan.sg_integrate()
    g = plan.capture_graph(finalize=False, profile=True)
    best = None
    for _ in range(reps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        g.replay()
        ms = plan.profile_read()
        if best is None or ms[3 + wpass - 1] < best[3 + wpass - 1]:
            best = ms
    k = best[3 + wpass - 1]
    nbytes = passes[wpass].written * rec + passes[wpass - 1].written * rec
    hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                      "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6550.4
    print(json.dumps({"config": cfg, "smem_cap": os.environ.get("SG_B200_PASS_SMEM", "0"),
                      "write_pass": wpass, "kernel_ms": round(k, 4), "launches_ms": [round(x, 4) for x in best],
                      "bytes": nbytes, "gbs": round(nbytes / (k * 1e-3) / 1e9, 1),
                      "frac": round(nbytes / (k * 1e-3) / 1e9 / hbm, 3)}))
    plan.close()


if __name__ == "__main__":
    main()
