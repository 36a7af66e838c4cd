#!/usr/bin/env python
"""Summarise ncu CSV logs / reports (gpurun_out/) into profiles/.

  python tools/ncu_summary.py launches <launches.csv> <out.md>          # per-kernel time share
  python tools/ncu_summary.py dram <dram.csv> <out.md> <config> [traffic.json]
  python tools/ncu_summary.py full <report.ncu-rep> <out.md>            # key --set full metrics
"""
import collections
import csv
import json
import os
import subprocess
import sys

# bench.py kernel-id names (roofline.kernel) -> ncu kernel-name prefixes
KID = {"gram": ("k_gram",), "project": ("k_project",), "spmm": ("k_spmm<",)}


def _rows(path):
    return [r for r in csv.reader(open(path)) if len(r) > 10]


def per_launch(path):
    rows = _rows(path)
    h = rows[0]
    iN, iM, iV, iID = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        lid = int(r[iID])
        names[lid] = r[iN].split("(")[0].replace("void ", "")
        try:
            per[lid][r[iM]] = float(r[iV].replace(",", ""))
        except ValueError:
            pass
    return names, per


def launches(src, out):
    names, per = per_launch(src)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for lid, m in per.items():
        a = agg[names[lid]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    with open(out, "w") as f:
        f.write(f"# ncu launch list summary ({os.path.basename(src)})\n\n"
                "`ncu --metrics gpu__time_duration.sum --clock-control none` over one bench step "
                "(cold-cache, serialised launches: compare SHARES, not absolute times).\n\n"
                "| kernel | launches | total us | us/launch | share |\n|---|---|---|---|---|\n")
        for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"| `{k}` | {a[0]} | {a[1] / 1e3:.1f} | {a[1] / a[0] / 1e3:.1f} | {100 * a[1] / tot:.1f}% |\n")
    print(open(out).read())


def dram(src, out, config, traffic_json=None):
    names, per = per_launch(src)
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for lid, m in per.items():
        a = agg[names[lid]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0)
        a[3] += m.get("dram__bytes_write.sum", 0.0)
    with open(out, "w") as f:
        f.write(f"# DRAM traffic per launch, config {config} ({os.path.basename(src)})\n\n"
                "`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                "--clock-control none` over one bench step; averages over all launches of each kernel.\n\n"
                "| kernel | launches | us/launch | read MB/launch | write MB/launch | DRAM GB/s |\n"
                "|---|---|---|---|---|---|\n")
        for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
            gbs = (a[2] + a[3]) / a[1] if a[1] else 0.0
            f.write(f"| `{k}` | {a[0]} | {a[1] / a[0] / 1e3:.1f} | {a[2] / a[0] / 1e6:.1f} | "
                    f"{a[3] / a[0] / 1e6:.1f} | {gbs:.0f} |\n")
    print(open(out).read())
    if traffic_json:
        d = json.load(open(traffic_json)) if os.path.exists(traffic_json) else {}
        ent = {}
        for kid, prefixes in KID.items():
            hits = [a for k, a in agg.items() if any(k.split("::")[-1].startswith(p) for p in prefixes)
                    and "true>" not in k]      # (not the residual SpMM variant)
            n = sum(a[0] for a in hits)
            if n:
                ent[kid] = sum(a[2] + a[3] for a in hits) / n
        d[f"config{config}"] = ent
        json.dump(d, open(traffic_json, "w"), indent=1)


FULL_KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
             "Compute (SM) Throughput", "Registers Per Thread", "Block Size", "Grid Size",
             "Theoretical Occupancy", "Achieved Occupancy", "Eligible Warps Per Scheduler",
             "Issued Warp Per Scheduler", "No Eligible", "Dynamic Shared Memory Per Block"]
RAW_KEYS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]


def full(rep, out):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    vals = {}
    name = ""
    rows = list(csv.reader(det.splitlines()))
    if rows:
        h = rows[0]
        iN, iM, iU, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
        for r in rows[1:]:
            if len(r) <= iV:
                continue
            name = name or r[iN]
            if r[iM] in FULL_KEYS:
                vals.setdefault(r[iM], f"{r[iV]} {r[iU]}".strip())
    rr = list(csv.reader(raw.splitlines()))
    d = dict(zip(rr[0], rr[2])) if len(rr) > 2 else {}
    units = dict(zip(rr[0], rr[1])) if len(rr) > 1 else {}

    def num(v):
        try:
            return float(v.replace(",", ""))
        except ValueError:
            return None
    stalls = sorted(((k.split("stalled_")[1], num(v)) for k, v in d.items()
                     if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
                     and num(v) is not None), key=lambda t: -t[1])
    with open(out, "w") as f:
        f.write(f"# ncu --set full: {os.path.basename(rep)}\n\n`{name}`\n\n| metric | value |\n|---|---|\n")
        for k in FULL_KEYS:
            if k in vals:
                f.write(f"| {k} | {vals[k]} |\n")
        for k in RAW_KEYS:
            if k in d:
                f.write(f"| {k} | {d[k]} {units.get(k, '')} |\n")
        tot = sum(v for _, v in stalls) or 1.0
        f.write("\nWarp-stall samples (top 8):\n\n| reason | share |\n|---|---|\n")
        for k, v in stalls[:8]:
            f.write(f"| {k} | {100 * v / tot:.1f}% |\n")
    print(open(out).read())


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif mode == "dram":
        dram(sys.argv[2], sys.argv[3], sys.argv[4], sys.argv[5] if len(sys.argv) > 5 else None)
    elif mode == "full":
        full(sys.argv[2], sys.argv[3])
