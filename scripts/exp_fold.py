"""Experiment: merge worker shapes at small n -- whole warp (k_merge_w) vs lane-folded slots
(k_merge_f) -- and static vs queued tasks, on skewed matrices of the config-3 mix (R-MAT 20 ef 16,
lognormal 7.92, aspect 2^14 x 1024), timed with library-recorded CUDA events, L2 flushed per rep.
Reports time and the fraction of the SURVEY §8(d) byte roofline."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_1803_08601_b200 import spmm as S  # noqa: E402
from paper_1803_08601_b200 import synth  # noqa: E402
from sweep_config4 import time_algo  # noqa: E402


def main():
    dev = torch.device("cuda")
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.empty(int(2 * l2) // 4, dtype=torch.float32, device=dev)
    peak = 6446.9
    seed = synth.STRUCT_SEED + 3
    mats = [("rmat20_ef16", synth.rmat(20, 16, seed + 66, device=dev)),
            ("lognormal7.92", synth.lognormal_rows(1 << 20, 1 << 20, 7.92, seed + 87, device=dev)),
            ("aspect_m16384", synth.aspect(1 << 24, 1 << 14, device=dev)),
            ("rmat22", synth.config_pattern(2, device=dev))]
    ns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8,16,32,64").split(",")]
    for name, p in mats:
        val = synth.values(p.nnz, 4100, "f32_plus_times", device=dev)
        distinct = int(torch.unique(p.col_indices).numel())
        for n in ns:
            B = synth.dense(p.k, n, 4200, "f32_plus_times", device=dev)
            C = torch.empty(p.m, n, dtype=torch.float32, device=dev)
            balg = 4 * (p.m + 1) + 8 * p.nnz + 4 * n * distinct + 4 * n * p.m
            line = f"{name:14s} n={n:3d}"
            for worker in (["warp", "folded"] if n <= 16 else ["warp"]):
                for tpw in (1, 2, 4, 8):
                    op = S.CsrSpmm(p.row_offsets, p.col_indices, val, p.k)
                    op.plan(n, "merge", merge_worker=worker, tasks_per_warp=tpw)
                    ms = time_algo(op, B, C, 5, flush)
                    op.close()
                    frac = balg / (ms / 1e3) / 1e9 / peak
                    line += f" | {worker[0]}{tpw} {ms * 1e3:8.1f}us {frac:.3f}"
            op = S.CsrSpmm(p.row_offsets, p.col_indices, val, p.k)
            op.plan(n, "rowsplit")
            ms = time_algo(op, B, C, 5, flush)
            op.close()
            line += f" | rowsplit {ms * 1e3:8.1f}us {balg / (ms / 1e3) / 1e9 / peak:.3f}"
            print(line, flush=True)
            del B, C


if __name__ == "__main__":
    main()
