"""FP64 instantiation of the plain oracle (oracle/sg_oracle.c built with -DSGO_FP64) on the full BASELINE
configs: wall time, points/s and its error against the __float128 oracle value of tests/golden (itself
pinned to the 50-digit DP value, tests/test_oracle_pins.py).  A CPU speed baseline that is not
parity-grade: its error shows the conditioning of Eq 2.6.  Calls only oracle/.

    python tools/oracle_fp64.py [--configs 1,2,3,4,5] [--threads N] [--out profiles/rNN_oracle_fp64.json]
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import mpmath as mp  # noqa: E402

import oracle  # noqa: E402
import sg_configs as S  # noqa: E402


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or platform.machine()


def run(configs, threads):
    gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_full.json")))["values"]
    rows = {}
    mp.mp.dps = 40
    for i in configs:
        p = S.baseline_config(i)
        r = oracle.integrate_problem(p, eval_mode=1, nthreads=threads, fp64=True)
        ref = mp.mpf(gold[p.name]["text"])
        got = mp.mpf(r.hi) + mp.mpf(r.lo)
        rows[p.name] = {"points": r.npoints, "seconds": round(r.seconds, 3),
                        "points_per_s": r.npoints / r.seconds if r.seconds > 0 else None,
                        "value": r.hi, "rel_err_vs_quad_oracle": float(abs((got - ref) / ref))}
        print(p.name, json.dumps(rows[p.name]), flush=True)
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = run([int(x) for x in a.configs.split(",") if x], a.threads)
    rec = {"what": "plain oracle, FP64 instantiation (-DSGO_FP64: Eq 2.6/2.7 point enumeration, "
                   "double sums and double integrand, active-coordinate form), full configs",
           "cores": a.threads or os.cpu_count(), "cpu": cpu_model(), "configs": rows}
    if a.out:
        json.dump(rec, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
