#!/usr/bin/env python
"""NEXT-4 measurement: the paper's Fig. 7 experiment on B200.

A 100,000 x 100,000 matrix whose rows each hold a fixed percentage of nonzeros drawn without replacement
(synth.uniform_rows, the paper's generator), times a 100,000 x 64 dense B, fp32.  Times the row-split,
merge-based and A/B-tiled (NEXT-4 second half) kernels (library-recorded CUDA events, L2 flushed before each rep) against a dense fp32 GEMM
of the same product (torch.matmul -> cuBLAS sgemm, TF32 disabled: the fp32 CUDA-core GEMM, as the paper's
cuBLAS sgemm), and reports the density at which the sparse path stops beating the dense one (the paper:
merge-based SpMM beats GEMM below 9% fill on a K40c).  Sampled rows of each kernel are checked against the
oracle.  Not part of the product path."""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1803_08601_b200 import spmm as S  # noqa: E402
from paper_1803_08601_b200 import synth  # noqa: E402


def time_spmm(op, B, C, flush, reps):
    nev = op.info()["launches_per_execute"] + 1
    sets = []
    for _ in range(reps + 1):
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(nev)]
        for e in evs:
            e.record()
        sets.append(evs)
    torch.cuda.synchronize()
    for evs in sets:
        flush.zero_()
        op.set_timing_events(evs)
        op.execute(B, C)
    torch.cuda.synchronize()
    op.set_timing_events([])
    ts = sorted(evs[0].elapsed_time(evs[-1]) for evs in sets[1:])
    return ts[len(ts) // 2]


def time_gemm(A, B, flush, reps):
    ts = []
    for _ in range(reps + 1):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        C = torch.matmul(A, B)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    del C
    return sorted(ts[1:])[len(ts[1:]) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=100_000)
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--pcts", default="0.01,0.1,0.5,1,2,5,9,12,15")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/density_sweep")
    args = ap.parse_args()
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False
    dev = torch.device("cuda")
    m = k = args.m
    n = args.n
    flush = torch.empty(int(2 * torch.cuda.get_device_properties(dev).L2_cache_size) // 4, device=dev)
    B = synth.dense(k, n, 7001, "f32_plus_times", device=dev)
    C = torch.empty(m, n, device=dev)
    res = []
    lines = []
    for pct in [float(x) for x in args.pcts.split(",")]:
        d = max(1, int(round(pct / 100.0 * k)))
        p = synth.uniform_rows(m, k, d, 7000 + d, device=dev)
        val = synth.values(p.nnz, 7002, "f32_plus_times", device=dev)
        rec = {"pct": pct, "d": d, "nnz": p.nnz}
        rows = np.unique(np.random.default_rng(d).integers(0, m, 64))
        pc = p.to("cpu")
        ref = oracle.spmm("f32_plus_times", m, k, n, pc.row_offsets, pc.col_indices, val.cpu(), B.cpu(), rows=rows)
        for algo in ("rowsplit", "merge", "tiled"):
            op = S.CsrSpmm(p.row_offsets, p.col_indices, val, k)
            op.plan(n, algo)
            rec[f"{algo}_ms"] = time_spmm(op, B, C, flush, args.reps)
            ok, worst, _ = oracle.check_f32(C.cpu().numpy()[rows], ref[0], ref[1], 1e-5)
            rec[f"{algo}_parity"] = bool(ok)
            op.close()
        op = S.CsrSpmm(p.row_offsets, p.col_indices, val, k)
        rec["auto_pick"] = op.plan(n, "auto")
        op.close()
        A = torch.zeros(m, k, device=dev)
        r_idx = torch.repeat_interleave(torch.arange(m, device=dev), d)
        A[r_idx, p.col_indices.long()] = val
        del r_idx
        rec["gemm_ms"] = time_gemm(A, B, flush, args.reps)
        del A
        torch.cuda.empty_cache()
        best = min(rec["rowsplit_ms"], rec["merge_ms"], rec["tiled_ms"])
        rec["best_sparse_over_gemm"] = best / rec["gemm_ms"]
        res.append(rec)
        lines.append(f"{pct:6.2f}% d={d:6d} nnz={p.nnz:11d}  rowsplit {rec['rowsplit_ms']:9.3f} ms  merge "
                     f"{rec['merge_ms']:9.3f} ms  tiled {rec['tiled_ms']:9.3f} ms  sgemm {rec['gemm_ms']:9.3f} ms  "
                     f"best/gemm {rec['best_sparse_over_gemm']:6.3f}  AUTO {rec['auto_pick']:8s}  parity "
                     f"{rec['rowsplit_parity'] and rec['merge_parity'] and rec['tiled_parity']}")
        print(lines[-1], flush=True)
        del p, val
        torch.cuda.empty_cache()
    cross = None
    for a, b in zip(res, res[1:]):
        if a["best_sparse_over_gemm"] < 1.0 <= b["best_sparse_over_gemm"]:
            # log-linear interpolation of the ratio in density
            la, lb = np.log(a["pct"]), np.log(b["pct"])
            t = (0 - np.log(a["best_sparse_over_gemm"])) / (np.log(b["best_sparse_over_gemm"]) - np.log(a["best_sparse_over_gemm"]))
            cross = float(np.exp(la + t * (lb - la)))
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump(res, open(args.out + ".json", "w"), indent=1)
    line = (f"crossover (best sparse kernel = fp32 sgemm): {cross:.2f}% fill" if cross else
            "no crossover inside the swept range (best sparse kernel faster than sgemm at every density)"
            if all(r["best_sparse_over_gemm"] < 1 for r in res) else "sparse slower than sgemm at every swept density")
    print(line)
    hdr = (f"Fig. 7 on B200 (PAPER.md:275): {m} x {k} uniform rows, n = {n}, fp32; SpMM timed with library events, "
           f"sgemm = torch.matmul fp32 (TF32 off); L2 flushed before every rep; median of {args.reps}")
    open(args.out + ".txt", "w").write("\n".join([hdr] + lines + [line]) + "\n")


if __name__ == "__main__":
    main()
