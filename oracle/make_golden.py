"""Write tests/golden/oracle_full.json: the oracle's full-size values for BASELINE configs 1-5.

Calls only ``oracle/`` (and the seeded input module).  Usage:
    python -m oracle.make_golden [--configs 1,2,3,4,5,cp] [--threads N]
Configs 4-5 take core-hours (4.5e9 / 2.75e10 quad transcendentals); results are merged into the
existing file config by config, so the script can be run in pieces.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import time

import oracle
import sg_configs as S

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "oracle_full.json")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args()
    data = {"generator": "oracle/make_golden.py (oracle.integrate, eval_mode=1, __float128)",
            "values": {}}
    if os.path.exists(OUT):
        data = json.load(open(OUT))
    for name in [s for s in args.configs.split(",") if s]:
        # BASELINE configs by number; "cp" = the corner-peak workload of the dd s-form path
        p = S.corner_config() if name == "cp" else S.baseline_config(int(name))
        t0 = time.time()
        r = oracle.integrate_problem(p, eval_mode=1, nthreads=args.threads)
        data["values"][p.name] = {
            "text": r.text, "hi": r.hi, "lo": r.lo, "npoints": r.npoints,
            "seconds": round(r.seconds, 3), "threads": args.threads or os.cpu_count(),
            "host": platform.processor() or platform.machine(),
            "d": p.d, "L": p.L, "rule": p.rule, "kind": p.kind,
        }
        json.dump(data, open(OUT + ".tmp", "w"), indent=1)
        os.replace(OUT + ".tmp", OUT)
        print(p.name, r.text, r.npoints, f"{time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
