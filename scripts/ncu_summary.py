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


def stall_reasons(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, v = rows[0], rows[2]
    res = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(x)) for h, x in zip(hdr, v)
           if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and x.replace(".", "").isdigit()]
    tot = sum(x for _, x in res) or 1.0
    return [(h, x / tot) for h, x in sorted(res, key=lambda t: -t[1])]


if __name__ == "__main__":
    rep = sys.argv[1]
    if "--json" in sys.argv:
        import json
        import os
        r = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"])
        def val(k, scale):
            v, u = r[k][0]
            f = float(v)
            return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                        "msecond": 1e-3, "second": 1}.get(u, scale)
        print(json.dumps({"report": os.path.basename(rep), "dram_read_bytes": val("dram__bytes_read.sum", 1),
                          "dram_write_bytes": val("dram__bytes_write.sum", 1),
                          "duration_s": val("gpu__time_duration.sum", 1)}))
        sys.exit(0)
    for k in details(rep):
        print(f"{k[1]:<40} {k[3]:>16} {k[2]}")
    r = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
                  "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
                  "l1tex__t_sector_hit_rate.pct", "lts__t_bytes.sum", "l1tex__t_bytes.sum"])
    for k, v in r.items():
        print(f"{k:<55} {v}")
    for h, f in stall_reasons(rep)[:8]:
        print(f"stall {h:<30} {f * 100:5.1f}%")
    if "--stalls" in sys.argv:
        te, tw, items = stalls(rep)
        print(f"instructions executed {te}, stall samples {tw}")
        for w, e, s in items:
            print(f"{w:>8} {e:>11}  {s[:90]}")
