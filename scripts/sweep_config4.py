#!/usr/bin/env python
"""BASELINE.json configs[3]: n sweep {1,4,16,32,64,128} over the 26-matrix SuiteSparse-shaped synthetic
mix (SURVEY.md §8(d) cfg 4), both kernels timed on every case (CUDA events, L2 flushed before each
rep), sampled-row parity against the oracle for both kernels, and the accuracy of the §5.4 heuristic
(PAPER policy: merge iff d < 9.35) and of the AUTO policy (+ skew guard) against the
faster kernel -- the paper's accuracy definition.  Writes a JSON list + a text table.
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1803_08601_b200 import spmm as S  # noqa: E402
from paper_1803_08601_b200 import synth  # noqa: E402


def time_algo(op, B, C, reps, flush):
    """Median execute time from CUDA events the library records on the stream right before its first
    and after its last kernel (spmm_csr_set_timing_events), so host-side call overhead is excluded."""
    nev = op.info()["launches_per_execute"] + 1
    sets = []
    for _ in range(reps + 2):
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
    ts = sorted(evs[0].elapsed_time(evs[-1]) for evs in sets[2:])
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--small", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ns", default="1,4,16,32,64,128")
    ap.add_argument("--out", default="gpurun_out/config4")
    args = ap.parse_args()
    dev = torch.device("cuda")
    ns = [int(x) for x in args.ns.split(",")]
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(int(2 * l2) // 4, dtype=torch.float32, device=dev)
    mats = synth.config4_mix(device=dev, small=args.small)
    results = []
    for mi, p in enumerate(mats):
        val = synth.values(p.nnz, 4000 + mi, "f32_plus_times", device=dev)
        lens = (p.row_offsets[1:] - p.row_offsets[:-1])
        d = p.nnz / p.m
        pc = p.to("cpu")
        rng = np.random.default_rng(mi)
        rows = np.unique(np.concatenate([rng.integers(0, p.m, 200), [0, p.m - 1],
                                         torch.topk(lens.cpu(), min(8, p.m)).indices.numpy()]))
        for n in ns:
            B = synth.dense(p.k, n, 5000 + mi, "f32_plus_times", device=dev)
            C = torch.empty(p.m, n, dtype=torch.float32, device=dev)
            rec = {"matrix": p.name, "m": p.m, "k": p.k, "nnz": p.nnz, "d": d, "max_row": int(lens.max()), "n": n}
            ref = oracle.spmm("f32_plus_times", p.m, p.k, n, pc.row_offsets, pc.col_indices, val.cpu(), B.cpu(),
                              rows=rows)
            algos = ["rowsplit", "merge"] + (["tiled"] if (n % 4 == 0 and 32 <= n <= 128) else [])
            for algo in algos:
                op = S.CsrSpmm(p.row_offsets, p.col_indices, val, p.k)
                op.plan(n, algo)
                ms = time_algo(op, B, C, args.reps, flush)
                ok, worst, _ = oracle.check_f32(C.cpu().numpy()[rows], ref[0], ref[1], 1e-5)
                rec[f"{algo}_ms"] = ms
                rec[f"{algo}_gflops"] = 2.0 * p.nnz * n / (ms / 1e3) / 1e9
                rec[f"{algo}_parity"] = ok
                op.close()
            op = S.CsrSpmm(p.row_offsets, p.col_indices, val, p.k)
            rec["paper_pick"] = op.plan(n, "auto", policy="paper")
            rec["auto_pick"] = op.plan(n, "auto", policy="auto")
            op.close()
            rec["best"] = min(algos, key=lambda a: rec[f"{a}_ms"])
            rec["best2"] = "rowsplit" if rec["rowsplit_ms"] <= rec["merge_ms"] else "merge"  # the paper's choice set
            results.append(rec)
            tl = f" tiled {rec['tiled_ms']*1e3:9.1f}us" if "tiled_ms" in rec else ""
            print(f"{p.name:28s} n={n:3d} d={d:7.2f} rs {rec['rowsplit_ms']*1e3:9.1f}us merge {rec['merge_ms']*1e3:9.1f}us{tl}"
                  f" best {rec['best']:8s} paper {rec['paper_pick']:8s} auto {rec['auto_pick']:8s}"
                  f" parity {all(rec[f'{a}_parity'] for a in algos)}", flush=True)
            del B, C
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump(results, open(args.out + ".json", "w"), indent=1)
    lines = []
    for n in ns:
        rs = [r for r in results if r["n"] == n]
        # the paper's accuracy is over its two kernels; AUTO is also scored over all three
        acc_p = sum(r["paper_pick"] == r["best2"] for r in rs) / len(rs)
        acc_a = sum(r["auto_pick"] == r["best"] for r in rs) / len(rs)
        best_t = [r[f"{r['best']}_ms"] for r in rs]
        loss_p = math.exp(np.mean([math.log(r[f"{r['paper_pick']}_ms"] / b) for r, b in zip(rs, best_t)]))
        loss_a = math.exp(np.mean([math.log(r[f"{r['auto_pick']}_ms"] / b) for r, b in zip(rs, best_t)]))
        # best single threshold on d for this n (merge iff d < t)
        cands = sorted(set([0.0] + [r["d"] for r in rs] + [1e9]))
        best_thr, best_acc = None, -1
        for t in cands:
            a = sum((("merge" if r["d"] < t else "rowsplit") == r["best2"]) for r in rs) / len(rs)
            if a > best_acc:
                best_thr, best_acc = t, a
        lines.append(f"n={n:3d}: accuracy PAPER {acc_p*100:5.1f}%  AUTO {acc_a*100:5.1f}%  geomean slowdown vs best "
                     f"PAPER {loss_p:.3f}x AUTO {loss_a:.3f}x  refit threshold d<{best_thr:.2f} -> {best_acc*100:.1f}%")
    allp = all(all(v for k2, v in r.items() if k2.endswith("_parity")) for r in results)
    lines.append(f"parity (sampled rows, both kernels, every case): {'PASS' if allp else 'FAIL'}")
    open(args.out + ".txt", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
