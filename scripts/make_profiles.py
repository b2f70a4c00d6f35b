#!/usr/bin/env python
"""Copy the ncu evidence of round TAG from gpurun_out/ into profiles/ (tracked) and derive
profiles/ncu_traffic.json (DRAM bytes per launch of the compute kernel, read by bench.py) and
profiles/<TAG>_launch_shares.txt (per-kernel share of one bench step from the launch lists)."""
import collections
import csv
import json
import os
import shutil
import sys

TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = os.path.join(ROOT, "gpurun_out")
dst = os.path.join(ROOT, "profiles")
os.makedirs(dst, exist_ok=True)

KEYS = {"rowsplit_c1": "config1_n64|k_tile<ROWSPLIT>", "merge_c2": "config2_n64|k_tile<MERGE>",
        "merge_c1": "config1_n64|k_tile<MERGE>", "rowsplit_c0": "config0_n64|k_tile<ROWSPLIT>"}
traffic_path = os.path.join(dst, "ncu_traffic.json")
traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
for line in open(os.path.join(src, f"ncu_traffic_{TAG}.jsonl")):
    d = json.loads(line)
    name = d["report"].replace("prof_", "").replace(".ncu-rep", "")
    if name in KEYS:
        traffic[KEYS[name]] = int(d["dram_read_bytes"] + d["dram_write_bytes"])
json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)

for f in os.listdir(src):
    if f.endswith(f"_{TAG}.txt") and f.startswith("ncu_"):
        shutil.copy(os.path.join(src, f), os.path.join(dst, f"{TAG}_{f[:-len(f'_{TAG}.txt')]}.txt"))

out = []
for cfg in ("c1", "c2"):
    f = os.path.join(src, f"launches_{cfg}_{TAG}.csv")
    if not os.path.exists(f):
        continue
    shutil.copy(f, os.path.join(dst, f"{TAG}_launches_{cfg}.csv"))
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    hdr = rows[0]
    iK, iV = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        if "spmm::" in r[iK] and "k_max_row" not in r[iK]:
            agg[r[iK].split("(")[0].replace("void ", "")].append(float(r[iV]) / 1e3)
    # steps = number of k_tile launches; one step = one launch of each path kernel
    step = sum(sum(v) / len(v) for v in agg.values())
    out.append(f"config {cfg[1:]} (bench.py --config {cfg[1:]}), ncu launch list, cold-cache serialised launches:")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        mean = sum(v) / len(v)
        out.append(f"  {k:45s} launches {len(v):3d}  mean {mean:9.2f} us  share of step {mean / step * 100:5.1f}%")
    out.append(f"  one step = {step:.2f} us\n")
open(os.path.join(dst, f"{TAG}_launch_shares.txt"), "w").write("\n".join(out) + "\n")
print("\n".join(out))
