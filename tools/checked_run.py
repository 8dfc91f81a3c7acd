"""Checked build run: bounds checks of every frontier read / write and write counts of every partial slot
(libsg_b200_checked.so, -DSG_CHECKS; kernels_common.cuh), the substitute for compute-sanitizer, which
is closed on this GPU pool.  For every case and every step:
  * no frontier index outside its buffer's capacity, no leaf row / mid row outside the factor table;
  * every partial slot written exactly once (a task claimed twice by the atomic task counters, or
    never, or a slot raced by two writers shows up as a count != 1);
  * three reruns give bitwise-identical results (the fixed-order reduction; a data race would not);
  * the value equals the __float128 oracle (small cases) or the stored full-size value (configs).

    python tools/checked_run.py [--quick] > profiles/rNN_checked_run.txt
"""
from __future__ import annotations

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CHECKED = os.path.join(ROOT, "paper_2210_14313_b200", "libsg_b200_checked.so")


def main():
    quick = "--quick" in sys.argv
    os.environ["SG_B200_LIB"] = CHECKED   # before the package is imported (_lib reads it once)
    from paper_2210_14313_b200 import build as B
    B.build(defines=("SG_CHECKS",), out=CHECKED)
    import mpmath as mp
    import torch

    import oracle
    import sg_configs as S
    from paper_2210_14313_b200 import _lib, api
    assert _lib.LIB_PATH == CHECKED, _lib.LIB_PATH
    L = _lib.lib()
    L.sg_chk_begin.argtypes = [ctypes.c_void_p]
    L.sg_chk_end.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong)]
    mp.mp.dps = 40
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_full.json")))["values"]

    def run_plan(p, rank, world, kw, env):
        old = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        try:
            plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, rank=rank, world=world, **kw)
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        vals, checked = [], 0
        for _ in range(3):
            assert L.sg_chk_begin(plan._h) == 0
            part = plan.sg_integrate()
            res = plan.sg_finalize(part, 1)
            out = (ctypes.c_longlong * 7)()
            assert L.sg_chk_end(plan._h, out) == 0
            viol, first, bad, nslots = out[0], list(out[1:5]), out[5], out[6]
            assert viol == 0, ("bounds violation", p.name, rank, world, kw, env, first)
            assert bad == 0, ("partial slots not written exactly once", p.name, rank, world, kw, env, bad, nslots)
            r = res.cpu().numpy()
            vals.append((float(r[0]), float(r[1])))
            checked = nslots
        plan.close()
        assert len(set(vals)) == 1, ("reruns differ", p.name, vals)
        return mp.mpf(vals[0][0]) + mp.mpf(vals[0][1]), checked

    cases = [
        ("c1", S.baseline_config(1), {}, {}, [1, 3], None),
        ("c2", S.baseline_config(2), {}, {}, [1, 3], None),
        ("c3", S.baseline_config(3), {}, {}, [1, 8], None),
        ("c4", S.baseline_config(4), {}, {}, [1, 8], None),
        ("c5", S.baseline_config(5), {}, {}, [1, 8], None),
        ("c5 merged", S.baseline_config(5), {"merge": api.MERGE_MIDPOINT}, {}, [1, 8], "merged"),
        ("c2 unfused", S.baseline_config(2), {}, {"SG_B200_NOFUSE": "1"}, [1, 3], None),
        ("c2 generic leaf", S.baseline_config(2), {}, {"SG_B200_GENERIC_LEAF": "1"}, [1], None),
        ("c4 no fork / no head", S.baseline_config(4), {}, {"SG_B200_NOFORK": "1", "SG_B200_NOHEAD": "1"}, [8], None),
        ("c4 lane groups 8", S.baseline_config(4), {}, {"SG_B200_LEAF2_GROUPS": "8"}, [1, 8], None),
        ("osc d=40 L=3 (source tasks)", S.random_problem(61, 40, 3, S.RULE_CC, S.KIND_OSC), {}, {}, [1, 3], None),
        ("gauss d=30 L=4", S.random_problem(62, 30, 4, S.RULE_CC, S.KIND_GAUSS), {}, {}, [1, 3], None),
        ("peak d=25 L=4 GL", S.random_problem(63, 25, 4, S.RULE_GL, S.KIND_PEAK), {}, {}, [1, 3], None),
        ("exp d=12 L=5", S.random_problem(64, 12, 5, S.RULE_CC, S.KIND_EXP), {}, {}, [1, 3], None),
        ("merged osc d=20 L=4", S.random_problem(65, 20, 4, S.RULE_CC, S.KIND_OSC), {"merge": api.MERGE_MIDPOINT}, {}, [1, 3], None),
        ("collapse d=20 L=4", S.random_problem(66, 20, 4, S.RULE_CC, S.KIND_OSC), {"method": api.METHOD_COLLAPSE}, {}, [1], None),
        ("s-form dd corner d=8 L=4", S.random_problem(67, 8, 4, S.RULE_CC, S.KIND_CORNER), {"arith": api.ARITH_SFORM_DD}, {}, [1, 3], None),
        ("unfused osc d=30 L=4", S.random_problem(68, 30, 4, S.RULE_CC, S.KIND_OSC), {}, {"SG_B200_NOFUSE": "1"}, [1, 3], None),
        ("split unfused osc d=30 L=4", S.random_problem(68, 30, 4, S.RULE_CC, S.KIND_OSC), {},
         {"SG_B200_NOFUSE": "1", "SG_B200_FRONT_SPLIT": "1"}, [1, 3], None),
        ("split exp d=12 L=6", S.random_problem(92, 12, 6, S.RULE_CC, S.KIND_EXP), {}, {"SG_B200_FRONT_SPLIT": "1"}, [1, 3], None),
        ("c5 unfused (split 4.3 GB frontier)", S.baseline_config(5), {}, {"SG_B200_NOFUSE": "1"}, [1], None),
        ("trapezoid d=33 L=4", S.random_problem(74, 33, 4, S.RULE_TRAP, S.KIND_GAUSS), {}, {}, [1, 3], None),
        ("patterson d=8 L=5", S.random_problem(55, 8, 5, S.RULE_GP, S.KIND_OSC), {}, {}, [1, 3], None),
    ]
    if quick:
        cases = [c for c in cases if not c[0].startswith("c5")]
    print(f"checked build: {CHECKED}")
    worst = 0.0
    for name, p, kw, env, worlds, _ in cases:
        if name.startswith("c") and p.name in gold and "merge" not in kw:
            ref = mp.mpf(gold[p.name]["text"])
        elif name.startswith("c") and p.name in gold:
            ref = mp.mpf(gold[p.name]["text"])
        else:
            ref = mp.mpf(oracle.integrate_problem(p, eval_mode=1).text)
        for world in worlds:
            tot, slots = mp.mpf(0), 0
            for rank in range(world):
                v, n = run_plan(p, rank, world, kw, env)
                tot += v
                slots += n
            err = float(abs((tot - ref) / ref))
            worst = max(worst, err)
            print(f"{name:32s} world={world}: 0 bounds violations, {slots} partial slots each written "
                  f"exactly once per step (x3 steps), bitwise-equal reruns, rel_err={err:.2e}", flush=True)
            assert err <= 1e-15, (name, world, err)
    print(f"CHECKED_RUN_OK worst rel_err {worst:.2e}")
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
