#!/usr/bin/env python
"""Summarise an ncu --set full report: key SOL / memory / occupancy metrics and the top stall lines."""
import csv
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active",
        "Issue Slots Busy", "Registers Per Thread", "Achieved Active Warps Per SM", "Theoretical Active Warps per SM",
        "Executed Instructions", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput", "Dynamic Shared Memory Per Block",
        "Grid Size", "Block Size"]


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    res = []
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in KEYS:
            res.append((d.get("Kernel Name", "")[:60], d["Metric Name"], d.get("Metric Unit", ""), d["Metric Value"]))
    return res


def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    vals = rows[2:]
    res = {}
    for nm in names:
        if nm in hdr:
            i = hdr.index(nm)
            res[nm] = [(v[i], units[i]) for v in vals]
    return res


def stalls(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    iS, iE, iW = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    items = []
    tot_e = tot_w = 0
    for r in rows[2:]:
        try:
            e, w = int(r[iE]), int(r[iW])
        except Exception:
            continue
        tot_e += e
        tot_w += w
        items.append((w, e, r[iS].strip()))
    items.sort(reverse=True)
    return tot_e, tot_w, items[:top]


if __name__ == "__main__":
    rep = sys.argv[1]
    for k in details(rep):
        print(f"{k[1]:<40} {k[3]:>16} {k[2]}")
    r = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
                  "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
                  "l1tex__t_sector_hit_rate.pct", "lts__t_bytes.sum", "l1tex__t_bytes.sum"])
    for k, v in r.items():
        print(f"{k:<55} {v}")
    if "--stalls" in sys.argv:
        te, tw, items = stalls(rep)
        print(f"instructions executed {te}, stall samples {tw}")
        for w, e, s in items:
            print(f"{w:>8} {e:>11}  {s[:90]}")
