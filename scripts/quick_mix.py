#!/usr/bin/env python
"""Tuning helper (not product code): time a few config-3 matrices with one kernel for each library
variant given on the command line (SPMM_LIB per subprocess).  CASES env: name:n,... over
{uniform_d16, uniform_d2, lognormal7, banded_w5, banded_w16, aspect_d4}."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(algo):
    import torch
    sys.path.insert(0, ROOT)
    from paper_1803_08601_b200 import spmm as S
    from paper_1803_08601_b200 import synth
    dev = torch.device("cuda")
    M = 1 << 20
    mk = {"uniform_d16": lambda: synth.uniform_rows(M, M, 16, 1819, dev),
          "uniform_d2": lambda: synth.uniform_rows(M, M, 2, 1805, dev),
          "lognormal7": lambda: synth.lognormal_rows(M, M, 7.92, 1890, device=dev),
          "banded_w5": lambda: synth.banded(M, 2, 2, dev),
          "banded_w16": lambda: synth.banded(M, device=dev),
          "aspect_d4": lambda: synth.aspect(1 << 24, 1 << 22, dev)}
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
    out = []
    for case in os.environ.get("CASES", "uniform_d16:64,uniform_d2:16,lognormal7:64,banded_w5:64,banded_w16:64").split(","):
        name, n = case.split(":")
        n = int(n)
        p = mk[name]()
        val = synth.values(p.nnz, 7, "f32_plus_times", device=dev)
        B = synth.dense(p.k, n, 8, "f32_plus_times", device=dev)
        C = torch.empty(p.m, n, device=dev)
        op = S.CsrSpmm(p.row_offsets, p.col_indices, val, p.k)
        op.plan(n, algo)
        inf = op.info()
        sets = []
        for it in range(8):
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(inf["launches_per_execute"] + 1)]
            for e in evs:
                e.record()
            sets.append(evs)
        torch.cuda.synchronize()
        for evs in sets:  # library-recorded events: no host call overhead in the interval
            flush.zero_()
            op.set_timing_events(evs)
            op.execute(B, C)
        torch.cuda.synchronize()
        op.set_timing_events([])
        ts = [evs[0].elapsed_time(evs[-1]) * 1e3 for evs in sets[2:]]
        op.close()
        out.append(f"{name}:n{n} {sorted(ts)[len(ts)//2]:8.1f}us{'*' if inf.get('b_staging') else ' '}")
    print("  ".join(out), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child(sys.argv[2])
        sys.exit(0)
    algo = os.environ.get("ALGO", "rowsplit")
    for lib in sys.argv[1:]:
        env = dict(os.environ, SPMM_LIB=os.path.abspath(lib))
        r = subprocess.run([sys.executable, __file__, "--child", algo], env=env, capture_output=True, text=True)
        print(f"{os.path.basename(lib):22s}", r.stdout.strip() or r.stderr[-600:], flush=True)
