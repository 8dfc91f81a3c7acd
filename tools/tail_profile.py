"""Ramp / tail profile of the persistent fused kernel (experiment build, -DSG_TAILPROF).

    python tools/tail_profile.py config world rank [config world rank ...]

Builds libsg_tailprof.so (per-warp globaltimer start / exit, SM id, task count, rows of the fused
k_leaf2 launch), runs a CUDA-graph replay of the plan after an L2 flush, and prints: kernel span
(first warp start -> last warp exit), the warp-busy fraction sum(busy) / (warps x span), the exit-time
percentiles, and the busy fraction of the slowest SM.  Only the k_leaf2 kernel is instrumented (the
real kinds' fused kernel; not sym3 / pairs).
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
EXTRA = tuple(x for x in os.environ.get("TP_DEFINES", "").split(",") if x)   # extra -D (A/B variants)
LIBP = os.path.join(ROOT, "paper_2210_14313_b200",
                    "libsg_tailprof" + "".join("_" + x.replace("=", "") for x in EXTRA) + ".so")


def main():
    os.environ["SG_B200_LIB"] = LIBP
    from paper_2210_14313_b200 import build as B
    B.build(defines=("SG_TAILPROF",) + EXTRA, out=LIBP)
    import numpy as np
    import torch

    import sg_configs as S
    from paper_2210_14313_b200 import _lib, api
    L = _lib.lib()
    args = [int(a) for a in sys.argv[1:]] or [4, 1, 0, 4, 8, 7]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    M = 16384
    for c, world, rank in zip(args[0::3], args[1::3], args[2::3]):
        p = S.baseline_config(c)
        plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=rank, world=world)
        for _ in range(2):
            plan.sg_integrate()
        g = plan.capture_graph(finalize=False)
        assert L.sg_tailprof_reset() == 0   # records of an earlier plan's launch
        for _ in range(3):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
        t0 = (ctypes.c_ulonglong * M)()
        t1 = (ctypes.c_ulonglong * M)()
        sm, nt, rw = (ctypes.c_uint * M)(), (ctypes.c_uint * M)(), (ctypes.c_uint * M)()
        assert L.sg_tailprof_read(t0, t1, sm, nt, rw, M) == 0
        a0, a1 = np.array(t0[:], dtype=np.int64), np.array(t1[:], dtype=np.int64)
        used = a1 > 0
        a0, a1 = a0[used], a1[used]
        smv, ntv, rwv = np.array(sm[:])[used], np.array(nt[:])[used], np.array(rw[:])[used]
        base = a0.min()
        s0, s1 = (a0 - base) / 1e3, (a1 - base) / 1e3   # us
        span = s1.max()
        busy = (s1 - s0).sum() / (len(s0) * span)
        pct = np.percentile(s1, [0, 10, 50, 90, 100])
        start_pct = np.percentile(s0, [0, 50, 100])
        per_sm_last = np.array([s1[smv == k].max() for k in np.unique(smv)])
        per_sm_first = np.array([s1[smv == k].min() for k in np.unique(smv)])
        # active warps over time (20 bins)
        bins = np.linspace(0, span, 21)
        act = [int(((s0 <= t) & (s1 > t)).sum()) for t in (bins[:-1] + bins[1:]) / 2]
        print(f"{p.name} world={world} rank={rank}: warps {len(s0)} span {span:.1f} us, warp-busy {busy:.3f}, "
              f"starts us {np.round(start_pct, 1).tolist()}, exits us (0/10/50/90/100%) {np.round(pct, 1).tolist()}")
        print(f"   SM last exit min/median/max {per_sm_last.min():.1f}/{np.median(per_sm_last):.1f}/{per_sm_last.max():.1f} us;"
              f" SM first exit median {np.median(per_sm_first):.1f} us; tasks/warp mean {ntv.mean():.2f} max {ntv.max()};"
              f" rows/warp mean {rwv.mean():.0f} min {rwv.min()} max {rwv.max()}")
        print(f"   active warps per 5% of span: {act}", flush=True)
        # which warps finish last: CTA rank among the CTAs of its SM (0 = lowest block index) and the
        # warp's index in its CTA, for the warps that exit in the last 10% of the span
        widx = np.nonzero(used)[0]
        wpc = int(os.environ.get("TP_WPC", "8"))
        cta = widx // wpc
        late = s1 > 0.9 * span
        rank_in_sm = np.zeros(len(widx), dtype=int)
        for k in np.unique(smv):
            sel = np.nonzero(smv == k)[0]
            ctas = np.unique(cta[sel])
            for r_, cc in enumerate(ctas):
                rank_in_sm[sel[cta[sel] == cc]] = r_
        print(f"   late warps {int(late.sum())}: CTA rank in SM {np.bincount(rank_in_sm[late], minlength=3).tolist()}, "
              f"warp in CTA {np.bincount((widx % wpc)[late], minlength=wpc).tolist()}; rows/warp by CTA rank "
              f"{[int(rwv[rank_in_sm == r_].mean()) for r_ in range(rank_in_sm.max() + 1)]}", flush=True)
        plan.close()


if __name__ == "__main__":
    main()
