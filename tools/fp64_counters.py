"""FP64 work per Smolyak point of the dominant leaf launch, from ncu's SASS counters.

Run mode (under ncu, on the GPU box; one sg_integrate of one config, nothing else):
    ncu --metrics sm__sass_thread_inst_executed_op_dfma_pred_on.sum,\
sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,\
gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ctr_c5_tree.csv \
        python tools/fp64_counters.py --run --config 5 --variant tree > gpurun_out/ctr_c5_tree.json

Parse mode (here): combine every ctr_<name>.csv / .json pair of a directory into
profiles/fp64_counters.json: for each run the launch with the longest duration among the leaf /
pass kernels is the dominant launch; flops per point = (2 DFMA + DADD + DMUL) / the pass's points,
FP64 instructions per point = (DFMA + DADD + DMUL) / points.
    python tools/fp64_counters.py --parse gpurun_out --tag r02a
"""
from __future__ import annotations

import argparse
import csv
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "profiles", "fp64_counters.json")
M = {"sm__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma",
     "sm__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd",
     "sm__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul",
     "gpu__time_duration.sum": "ns"}


def run(cfg, variant):
    import torch
    import sg_configs as S
    from paper_2210_14313_b200 import api
    p = S.baseline_config(cfg)
    kw = {"merge": api.MERGE_MIDPOINT} if variant == "merged" else {}
    plan = api.Plan(p.d, p.q, p.rule, p.kind, p.c, p.w, p.u, **kw)
    passes = plan.passes()
    dom = max(range(1, len(passes)), key=lambda i: passes[i].terms)
    plan.sg_integrate()
    torch.cuda.synchronize()
    print(json.dumps({"config": cfg, "variant": variant, "dominant_pass": dom,
                      "points": passes[dom].terms, "passes": [q.terms for q in passes]}))


def parse_csv(path):
    launches = {}
    with open(path) as f:
        rows = [r for r in csv.reader(f)]
    hdr = None
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        key = (int(d["ID"]), d["Kernel Name"])
        name = M.get(d["Metric Name"])
        if name:
            launches.setdefault(key, {})[name] = float(d["Metric Value"].replace(",", ""))
    return [dict(id=k[0], kernel=k[1], **v) for k, v in sorted(launches.items())]


def parse(directory, tag):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {"launches": {}}
    data["what"] = ("ncu SASS FP64 thread-instruction counters of each config's dominant leaf launch "
                    "(tools/fp64_counters.py); flops = 2 DFMA + DADD + DMUL")
    for js in sorted(glob.glob(os.path.join(directory, "ctr_*.json"))):
        csvp = js[:-5] + ".csv"
        if not os.path.exists(csvp):
            continue
        meta = json.loads([ln for ln in open(js) if ln.startswith("{")][-1])
        launches = [x for x in parse_csv(csvp) if x["kernel"].startswith(("k_leaf", "void k_leaf", "void k_pass", "k_pass"))]
        if not launches:
            continue
        dom = max(launches, key=lambda x: x.get("ns", 0))
        pts = meta["points"]
        flops = 2 * dom["dfma"] + dom["dadd"] + dom.get("dmul", 0)
        inst = dom["dfma"] + dom["dadd"] + dom.get("dmul", 0)
        key = f"c{meta['config']}_{meta['variant']}"
        data["launches"][key] = {
            "kernel": dom["kernel"][:120], "points": pts, "dfma": dom["dfma"], "dadd": dom["dadd"],
            "dmul": dom.get("dmul", 0), "ncu_ns": dom.get("ns"),
            "flops_per_point": flops / pts, "fp64_inst_per_point": inst / pts,
            "dfma_per_point": dom["dfma"] / pts, "dadd_per_point": dom["dadd"] / pts,
            "dmul_per_point": dom.get("dmul", 0) / pts,
            "source": f"{tag}: {os.path.relpath(csvp, ROOT)}"}
        print(key, json.dumps(data["launches"][key]))
    json.dump(data, open(OUT, "w"), indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--run", action="store_true")
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--variant", default="tree", choices=["tree", "merged"])
    ap.add_argument("--parse", default=None)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    if a.run:
        run(a.config, a.variant)
    elif a.parse:
        parse(a.parse, a.tag)


if __name__ == "__main__":
    main()
