#!/usr/bin/env python
"""On the GPU box: ncu captures of the bench's dominant kernel per workload -> profiles/ncu_traffic.json
(read by bench.py as roofline.traffic / roofline.ncu).  For each config: one ncu pass over a short
bench run (the same build, the same launch configuration bench.py times), the compute kernel's
DRAM bytes read + written, L2 hit rate and duration.  configs 1 and 2 use `--set full`; the R-MAT 26
kernel (17 GB of C per launch: --set full's replay save/restore is impractical) uses the metric list
only.  Usage: python scripts/ncu_traffic.py [out.json]"""
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NCU = "/usr/local/cuda/bin/ncu"
METRICS = "dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum"
# demangled-name filters: the compute kernels only (not the plan-time k_tile_span etc.)
KERNEL = {"rowsplit": ("regex:k_tile<", "k_tile<ROWSPLIT>"), "merge": ("regex:k_merge_[wf]<", "k_merge_w")}


def sha16():
    with open(os.path.join(ROOT, "paper_1803_08601_b200", "libspmm.so"), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()[:16]


def capture(cfg, algo_kind, full):
    kregex, kname = KERNEL[algo_kind]
    cmd = [NCU, "--clock-control", "none", "--kernel-name-base", "demangled", "-k", kregex, "-s", "1", "-c", "1",
           "--csv", "--page", "raw"]
    cmd += ["--set", "full", "--metrics", METRICS] if full else ["--metrics", METRICS]
    cmd += [sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(cfg), "--steps", "1", "--warmup", "3",
            "--no-e2e", "--no-cpu-baseline", "--no-extras"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=3000).stdout
    lines = [ln for ln in out.splitlines() if ln.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, units, vals = rows[0], rows[1], rows[2]

    def get(name):
        i = hdr.index(name)
        v = float(vals[i].replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                    "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1, "second": 1, "%": 1}.get(units[i], 1)
    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    dur = get("gpu__time_duration.sum")
    return kname, {"dram_bytes": int(rd + wr), "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
                   "l2_hit_pct": round(get("lts__t_sector_hit_rate.pct"), 2), "ncu_duration_ms": round(dur * 1e3, 4),
                   "dram_gbs_under_ncu": round((rd + wr) / dur / 1e9, 1),
                   "capture": "ncu --set full" if full else "ncu --metrics " + METRICS,
                   "kernel_name": vals[hdr.index("Kernel Name")][:90]}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "ncu_traffic.json")
    sha = sha16()
    sys.path.insert(0, ROOT)
    from paper_1803_08601_b200 import build as B
    src = B.source_sha16()
    res = {}
    for cfg, algo, full in ((1, "rowsplit", True), (2, "merge", True), (4, "merge", False)):
        kname, ent = capture(cfg, algo, full)
        ent["lib_sha16"] = sha
        ent["src_sha16"] = src
        res[f"config{cfg}_n64|{kname}"] = ent
        print(cfg, json.dumps(ent), flush=True)
    with open(out, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
