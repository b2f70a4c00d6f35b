"""Experiment (not product code): does splitting B's n = 64 columns into column tiles, one SpMM pass per
tile with A re-read per pass (the paper's 32-column C tiles), raise the L2 hit rate
of the B-row gathers enough to pay for the extra A reads on R-MAT?  Times the merge and row-split
kernels on configs 2 / 4 with L2 flushed before every rep.

usage: python scripts/exp_coltile.py [cfg ...]
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_08601_b200 import spmm as S  # noqa: E402
from paper_1803_08601_b200 import synth  # noqa: E402


def timeit(fn, flush, reps=7):
    ts = []
    for _ in range(2):
        flush.zero_()
        fn()
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [2]
    dev = torch.device("cuda", 0)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(int(2 * l2) // 4, dtype=torch.float32, device=dev)
    n = 64
    for cfg in cfgs:
        p = synth.config_pattern(cfg, device=dev)
        vals = synth.values(p.nnz, synth.STRUCT_SEED + cfg + 100, "f32_plus_times", device=dev)
        B = synth.dense(p.k, n, synth.STRUCT_SEED + cfg + 200, "f32_plus_times", device=dev)
        C = torch.empty(p.m, n, dtype=torch.float32, device=dev)
        ref = None
        for algo in ("merge", "rowsplit"):
            for w in (64, 32, 16):
                op = S.CsrSpmm(p.row_offsets, p.col_indices, vals, p.k)
                op.plan(w, algo)
                tiles = [(B[:, j:j + w], C[:, j:j + w]) for j in range(0, n, w)]

                def run():
                    for b, c in tiles:
                        op.execute(b, c)
                t = timeit(run, flush)
                if ref is None:
                    ref = C.clone()
                err = float((C - ref).abs().max())
                print(f"cfg {cfg} {algo:8s} col tile {w:3d} x {n // w}: {t:8.3f} ms  (max diff vs first {err:.2e})",
                      flush=True)
                op.close()
        del p, vals, B, C, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
