#!/usr/bin/env python
"""Per-rank work of the multi-GPU row-block partition, measured on ONE B200 (this build can reach one GPU).

For P in {1, 2, 4, 8} and both row partitions of spmm_partition_rows (0 = nnz-balanced, the north_star's;
1 = merge-path balanced, rows + nonzeros), every rank's row block of BASELINE configs[4] (R-MAT scale 26,
n = 64, or --config 2 for scale 22) is planned (AUTO) and executed on its own, with L2 flushed before each
run -- exactly the local work rank r does on its own GPU after the B broadcast (each B200 has its own L2
and HBM).  T_spmm(P) = max over ranks; the strong-scaling speedup T_spmm(1) / T_spmm(P) is what the
north_star's ">= 6x at 8 GPUs" is about (the broadcast of B and the optional all-gather of C are separate
NVLink steps, not included).  Each rank's result is checked on 2^16 sampled rows against
the CPU oracle (oracle.check_f32: |C - C_ref| <= 1e-5 (|A||B|)_ij, the north_star bound).  Not product
code."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1803_08601_b200 import dist  # noqa: E402
from paper_1803_08601_b200 import spmm as S  # noqa: E402
from paper_1803_08601_b200 import synth  # noqa: E402


def run_block(ro, col, val, k, B, n, flush, reps):
    m = ro.numel() - 1
    C = torch.empty(m, n, device=B.device)
    op = S.CsrSpmm(ro, col, val, k)
    algo = op.plan(n, "auto")
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
    op.close()
    ts = sorted(evs[0].elapsed_time(evs[-1]) for evs in sets[1:])
    return ts[len(ts) // 2], algo, C


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4, choices=[2, 4])
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="gpurun_out/scaling_emulation")
    args = ap.parse_args()
    dev = torch.device("cuda")
    n = args.n
    p = synth.config_pattern(args.config, device=dev)
    seed = synth.STRUCT_SEED + args.config
    val = synth.values(p.nnz, seed + 100, "f32_plus_times", device=dev)
    B = synth.dense(p.k, n, seed + 200, "f32_plus_times", device=dev)
    flush = torch.empty(int(2 * torch.cuda.get_device_properties(dev).L2_cache_size) // 4, device=dev)
    t1, algo1, C1 = run_block(p.row_offsets, p.col_indices, val, p.k, B, n, flush, args.reps)
    rng = torch.Generator(device="cpu").manual_seed(5)
    sample = torch.randint(0, p.m, (1 << 16,), generator=rng).to(dev)
    del C1
    # oracle on the sampled rows (rows are independent, so the sampled check is exact for those rows)
    ref_C, ref_bound = oracle.spmm("f32_plus_times", p.m, p.k, n, p.row_offsets.cpu().numpy(),
                                   p.col_indices.cpu().numpy(), val.cpu().numpy(), B.cpu().numpy(),
                                   rows=sample.cpu().numpy())
    torch.cuda.empty_cache()
    ro_cpu = p.row_offsets.cpu()
    lines = [f"config {args.config}: m = {p.m}, nnz = {p.nnz}, n = {n}; T_spmm(1) = {t1:.3f} ms ({algo1})"]
    res = {"config": args.config, "m": p.m, "nnz": p.nnz, "n": n, "t1_ms": t1, "algo1": algo1, "runs": []}
    for mode in (0, 1):
        for P in (2, 4, 8):
            bounds = dist.partition_rows(ro_cpu, P, mode)
            times, algos, nnzs, rows = [], [], [], []
            ok = True
            for r in range(P):
                r0, r1 = bounds[r], bounds[r + 1]
                ro, col, v = dist.slice_rows(p.row_offsets, p.col_indices, val, r0, r1)
                t, a, C = run_block(ro.contiguous(), col, v, p.k, B, n, flush, args.reps)
                sel = ((sample >= r0) & (sample < r1)).cpu().numpy()
                got = C[sample[torch.from_numpy(sel).to(dev)] - r0].cpu().numpy()
                ok &= bool(oracle.check_f32(got, ref_C[sel], ref_bound[sel], 1e-5)[0])
                times.append(t)
                algos.append(a)
                nnzs.append(int(ro[-1]))
                rows.append(r1 - r0)
                del C
            tmax = max(times)
            res["runs"].append({"mode": mode, "P": P, "bounds": bounds, "times_ms": times, "algos": algos,
                                "nnz": nnzs, "rows": rows, "tmax_ms": tmax, "speedup": t1 / tmax, "check": ok})
            lines.append(f"partition {'nnz-balanced ' if mode == 0 else 'merge-path   '} P={P}: T_spmm = max {tmax:8.3f} ms "
                         f"(min {min(times):8.3f}) speedup {t1 / tmax:5.2f}x  efficiency {t1 / tmax / P * 100:5.1f}%  "
                         f"kernels {','.join(sorted(set(algos)))}  sampled rows match the oracle {ok}")
            print(lines[-1], flush=True)
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump(res, open(args.out + ".json", "w"), indent=1)
    hdr = ("per-rank local SpMM of the row-block partition, each rank's block run alone on one B200 with L2 "
           "flushed (emulates P GPUs; B broadcast / C all-gather excluded), scripts/scaling_emulation.py")
    open(args.out + ".txt", "w").write("\n".join([hdr] + lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
