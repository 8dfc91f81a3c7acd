"""Summarise ncu reports / launch lists into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py <tag> <rep1.ncu-rep> [...] [--launches c5=launches.csv ...]

Writes profiles/<tag>_ncu_summary.md (key metrics per captured kernel + per-launch shares) and
updates profiles/traffic.json (DRAM bytes per launch of each config's dominant kernel).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
    "sm__sass_thread_inst_executed_op_dfma_pred_on.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
    "sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for i, h in enumerate(hdr):
            if h in KEYS or h in ("Kernel Name",):
                d[h] = (vals[i], units[i])
        res.append(d)
    return res


def to_bytes(v, u):
    v = float(v)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    out = []
    for r in rows[1:]:
        out.append((r[ki], float(r[vi].replace(",", ""))))
    return out


def main():
    tag = sys.argv[1]
    args = sys.argv[2:]
    reps = [a for a in args if a.endswith(".ncu-rep")]
    lls = [a.split("=", 1) for a in args if "=" in a]
    lines = [f"# ncu summary {tag}", "",
             "Captured with `ncu --set full --clock-control none --import-source on` (one launch each, "
             "cold cache, serialised replay; times are ncu's, never bench values).", ""]
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tfile)) if os.path.exists(tfile) else {}
    for rep in reps:
        ds = raw(rep)
        # traffic.json: the dominant (longest) captured launch of each config
        top = max(ds, key=lambda d: float(d["gpu__time_duration.sum"][0])) if ds else None
        for d in ds:
            name = d.get("Kernel Name", ("?", ""))[0]
            lines.append(f"## {os.path.basename(rep)} — `{name}`")
            lines.append("")
            lines.append("| metric | value | unit |")
            lines.append("|---|---|---|")
            for k in KEYS:
                if k in d:
                    lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
            lines.append("")
            base = os.path.basename(rep)
            for cfg in ("c4", "c5", "c3"):
                if f"_{cfg}_" in base and "leaf" in base and d is top:
                    rb = to_bytes(*d["dram__bytes_read.sum"])
                    wb = to_bytes(*d["dram__bytes_write.sum"])
                    traffic[cfg] = rb + wb
    for cfg, path in lls:
        ls = launches(path)
        total = sum(t for _, t in ls)
        lines.append(f"## launch list {cfg} (`{os.path.basename(path)}`, gpu__time_duration.sum)")
        lines.append("")
        lines.append("| kernel | ns | share |")
        lines.append("|---|---|---|")
        for n, t in ls:
            lines.append(f"| `{n[:60]}` | {t:.0f} | {t / total:.1%} |")
        lines.append("")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(tfile, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
