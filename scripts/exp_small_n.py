"""Experiment: AUTO-planned SpMM at small n (1..16) on the skewed matrices of the config-3 mix, timed with
library-recorded CUDA events, L2 flushed per rep; prints time and the SURVEY §8(d) byte-roofline fraction.
The library is the in-tree one or $SPMM_LIB (for A/B of build variants)."""
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
            ("rmat20_ef4", synth.rmat(20, 4, seed + 64, device=dev)),
            ("lognormal7.92", synth.lognormal_rows(1 << 20, 1 << 20, 7.92, seed + 87, device=dev)),
            ("aspect_m16384", synth.aspect(1 << 24, 1 << 14, device=dev)),
            ("rmat22", synth.config_pattern(2, device=dev))]
    ns = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8,16").split(",")]
    tag = os.environ.get("SPMM_LIB", "in-tree")
    for name, p in mats:
        val = synth.values(p.nnz, 4100, "f32_plus_times", device=dev)
        distinct = int(torch.unique(p.col_indices).numel())
        line = f"{tag[-24:]:24s} {name:14s}"
        for n in ns:
            B = synth.dense(p.k, n, 4200, "f32_plus_times", device=dev)
            C = torch.empty(p.m, n, dtype=torch.float32, device=dev)
            balg = 4 * (p.m + 1) + 8 * p.nnz + 4 * n * distinct + 4 * n * p.m
            op = S.CsrSpmm(p.row_offsets, p.col_indices, val, p.k)
            algo = op.plan(n, "auto")
            ms = time_algo(op, B, C, 7, flush)
            info = op.info()
            op.close()
            frac = balg / (ms / 1e3) / 1e9 / peak
            w = "f" if info.get("merge_worker_lanes", 32) < 32 and algo == "merge" else algo[0]
            line += f" | n={n:2d} {w} {ms * 1e3:7.1f}us {frac:.3f}"
            del B, C
        print(line, flush=True)


if __name__ == "__main__":
    main()
