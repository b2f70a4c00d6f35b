"""Run one planned SpMM a few times (for ncu captures): python scripts/run_one.py <matrix> <n> <algo> [worker] [tpw]
matrix: rmat20 | rmat22 | lognormal | aspect | banded | rmat26"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1803_08601_b200 import spmm as S  # noqa: E402
from paper_1803_08601_b200 import synth  # noqa: E402


def pattern(name, dev):
    seed = synth.STRUCT_SEED + 3
    if name == "rmat20":
        return synth.rmat(20, 16, seed + 66, device=dev)
    if name == "rmat22":
        return synth.config_pattern(2, device=dev)
    if name == "rmat26":
        return synth.config_pattern(4, device=dev)
    if name == "lognormal":
        return synth.lognormal_rows(1 << 20, 1 << 20, 7.92, seed + 87, device=dev)
    if name == "aspect":
        return synth.aspect(1 << 24, 1 << 14, device=dev)
    if name == "banded":
        return synth.config_pattern(1, device=dev)
    raise ValueError(name)


def main():
    name, n, algo = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    worker = sys.argv[4] if len(sys.argv) > 4 else "auto"
    tpw = int(sys.argv[5]) if len(sys.argv) > 5 else 0
    dev = torch.device("cuda")
    p = pattern(name, dev)
    val = synth.values(p.nnz, 4100, "f32_plus_times", device=dev)
    B = synth.dense(p.k, n, 4200, "f32_plus_times", device=dev)
    C = torch.empty(p.m, n, dtype=torch.float32, device=dev)
    op = S.CsrSpmm(p.row_offsets, p.col_indices, val, p.k)
    op.plan(n, algo, merge_worker=worker, tasks_per_warp=tpw)
    for _ in range(3):
        op.execute(B, C)
    torch.cuda.synchronize()
    print(op.info())


if __name__ == "__main__":
    main()
