#!/usr/bin/env python
"""SURVEY.md §8(f) NEXT-2, remainder: the paper's 1-D nonzero split (PAPER.md:80, its own choice, :89)
against the 2-D merge path as the merge kernel's phase-1 partition, same items per task,
same compute kernel, timed on R-MAT 22 / 26, lognormal row lengths (corpus means 7.92 and 62.5,
PAPER.md:217, :237) and a many-empty-rows matrix (the pathology the paper names at PAPER.md:89), at
n in {1, 16, 64}.  CUDA events recorded by the library around its launches, L2 flushed before every
rep; sampled rows of both results checked against the oracle.  The paper's claim under test: the two
partitions "possess similar performance characteristics" except on many empty rows.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import oracle  # noqa: E402
from paper_1803_08601_b200 import spmm as S  # noqa: E402
from paper_1803_08601_b200 import synth  # noqa: E402
from sweep_config4 import time_algo  # noqa: E402


def many_empty(m: int, frac_nonempty: float, d: int, seed: int, device):
    """m x m, a seeded fraction of the rows holds d uniform columns, every other row is empty."""
    h = synth.counter_u32(seed, 30, torch.arange(m, device=device, dtype=torch.int64))
    keep = h < int(frac_nonempty * 2**32)
    lens = torch.where(keep, torch.full_like(h, d), torch.zeros_like(h))
    E = int(lens.sum())
    rows = torch.repeat_interleave(torch.arange(m, device=device, dtype=torch.int64), lens)
    cols = (synth.counter_u32(seed, 31, torch.arange(E, device=device, dtype=torch.int64)) * m) >> 32
    keys = torch.unique(rows * m + cols, sorted=True)
    return synth._csr_from_sorted_keys(keys, m, m, f"many_empty_m{m}_{frac_nonempty}_d{d}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ns", default="1,16,64")
    ap.add_argument("--big", action="store_true", help="include R-MAT 26 (n = 64 only)")
    ap.add_argument("--out", default="gpurun_out/ablation_partition")
    args = ap.parse_args()
    dev = torch.device("cuda")
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(int(2 * l2) // 4, dtype=torch.float32, device=dev)
    seed = synth.STRUCT_SEED + 3
    mats = [("rmat22", lambda: synth.config_pattern(2, device=dev)),
            ("lognormal7.92", lambda: synth.lognormal_rows(1 << 22, 1 << 22, 7.92, seed + 87, device=dev)),
            ("lognormal62.5", lambda: synth.lognormal_rows(1 << 20, 1 << 20, 62.5, seed + 142, device=dev)),
            ("many_empty_1pct_d64", lambda: many_empty(1 << 24, 0.01, 64, seed + 7, dev)),
            ("many_empty_10pct_d16", lambda: many_empty(1 << 22, 0.10, 16, seed + 8, dev))]
    if args.big:
        mats.append(("rmat26", lambda: synth.config_pattern(4, device=dev)))
    ns = [int(x) for x in args.ns.split(",")]
    res = []
    for name, mk in mats:
        p = mk()
        val = synth.values(p.nnz, 4100, "f32_plus_times", device=dev)
        lens = p.row_offsets[1:] - p.row_offsets[:-1]
        rng = np.random.default_rng(7)
        rows = np.unique(np.concatenate([rng.integers(0, p.m, 2000), [0, p.m - 1],
                                         torch.topk(lens, min(16, p.m)).indices.cpu().numpy()]))
        pc_ro = p.row_offsets.cpu()
        for n in (ns if name != "rmat26" else [64]):
            B = synth.dense(p.k, n, 4200, "f32_plus_times", device=dev)
            C = torch.empty(p.m, n, dtype=torch.float32, device=dev)
            # oracle on the sampled rows only (rows are independent)
            sub_ro = np.concatenate([[0], np.cumsum((pc_ro[rows + 1] - pc_ro[rows]).numpy())]).astype(np.int32)
            idx = np.concatenate([np.arange(int(pc_ro[r]), int(pc_ro[r + 1])) for r in rows]).astype(np.int64)
            colc = p.col_indices[torch.from_numpy(idx).to(dev)].cpu().numpy()
            valc = val[torch.from_numpy(idx).to(dev)].cpu().numpy()
            ref = oracle.spmm("f32_plus_times", len(rows), p.k, n, sub_ro, colc, valc, B.cpu().numpy())
            rec = {"matrix": name, "m": p.m, "nnz": p.nnz, "d": p.nnz / p.m, "max_row": int(lens.max()),
                   "empty_rows": int((lens == 0).sum()), "n": n}
            items = None
            for part in ("merge_path", "nonzero_split"):
                op = S.CsrSpmm(p.row_offsets, p.col_indices, val, p.k)
                op.plan(n, "merge", partition=part, items_per_cta=items or 0)
                items = items or op.info()["items_per_cta"]
                ms = time_algo(op, B, C, args.reps, flush)
                ok, worst, _ = oracle.check_f32(C[torch.from_numpy(rows).to(dev)].cpu().numpy(), ref[0], ref[1], 1e-5)
                rec[f"{part}_ms"] = ms
                rec[f"{part}_tasks"] = op.info()["num_ctas"]
                rec[f"{part}_parity"] = bool(ok)
                op.close()
            rec["items_per_task"] = items
            rec["ratio_1d_over_2d"] = rec["nonzero_split_ms"] / rec["merge_path_ms"]
            res.append(rec)
            print(f"{name:22s} n={n:3d} d={rec['d']:6.2f} empty={rec['empty_rows'] / p.m * 100:5.1f}% "
                  f"2-D {rec['merge_path_ms'] * 1e3:9.1f} us  1-D {rec['nonzero_split_ms'] * 1e3:9.1f} us  "
                  f"1-D/2-D {rec['ratio_1d_over_2d']:.3f}  items {items}  parity "
                  f"{rec['merge_path_parity'] and rec['nonzero_split_parity']}", flush=True)
            del B, C
        del p, val
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump(res, open(args.out + ".json", "w"), indent=1)


if __name__ == "__main__":
    main()
