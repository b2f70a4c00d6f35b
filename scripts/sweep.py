#!/usr/bin/env python
"""Run bench.py for several library variants / configs and print one compact line each (tuning only)."""
import json
import os
import subprocess
import sys

libs = [a for a in sys.argv[1:] if a.endswith(".so")] or ["paper_1803_08601_b200/libspmm.so"]
cases = os.environ.get("CASES", "1:auto,2:auto").split(",")
extra = os.environ.get("BENCH_ARGS", "").split()
for lib in libs:
    for case in cases:
        cfg, algo = case.split(":")
        env = dict(os.environ, SPMM_LIB=os.path.abspath(lib))
        cmd = [sys.executable, "bench.py", "--config", cfg, "--algo", algo, "--steps", "20", "--warmup", "3",
               "--no-e2e", "--no-cpu-baseline"] + extra
        p = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=900)
        try:
            d = json.loads(p.stdout.strip().splitlines()[-1])
            r = d["roofline"]
            print(f"{os.path.basename(lib):28s} cfg{cfg} {algo:8s} {d['config']['algo']:8s} step {d['ms_per_step']*1e3:8.1f} us"
                  f"  kernel {r['avg_launch_ms']*1e3:8.1f} us  {d['value']:9.1f} GFLOP/s  frac {r['frac']:.3f}", flush=True)
        except Exception:
            print(lib, case, "FAILED", p.stderr[-800:], flush=True)
