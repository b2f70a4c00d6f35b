#!/usr/bin/env python
"""bench.py -- SpMM GFLOP/s and HBM GB/s (fraction of roofline) at n=64 on 1..N B200.

One "step" = one C = A*B through spmm_csr_execute (the whole hot path of SURVEY.md §8(a): for the
row-split choice one kernel, for merge: partition + compute + carry fix-up) over one synthetic input
resident in HBM.  Default workload = BASELINE.json configs[1]: banded m = k = 2^20, 16 nnz/row,
n = 64, fp32 (the AUTO heuristic picks row split there).  L2 is flushed (2x L2 bytes written) before
every timed step.  Multi-GPU (torchrun): weak scaling on the banded family (global banded matrix of
N*2^20 rows, rank r owns row block r, B broadcast from rank 0 over NCCL and timed separately), or
strong scaling with nnz-balanced row blocks for the R-MAT configs.

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (oracle/, plain C) on a
bounded sample of the same workload instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1803_08601_b200 import synth  # noqa: E402

METRIC = "SpMM GFLOP/s and HBM GB/s (fraction of roofline) at n=64, 1/2/4/8 B200"
UNIT = "GFLOP/s"

WORKLOADS = {
    1: "banded m=k=2^20 (x N ranks, weak), 16 nnz/row, n=64, fp32 plus-times (BASELINE configs[1])",
    2: "R-MAT scale 22, avg deg 16, n=64, fp32 plus-times (BASELINE configs[2])",
    4: "R-MAT scale 26, avg deg 16, n=64, fp32 plus-times, row blocks (BASELINE configs[4])",
    0: "tiny uniform m=k=1024, 16 nnz/row, n=64, fp32 plus-times (BASELINE configs[0])",
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ------------------------------------------------------------------------------------------------
# clocks sampler (NVML), run during the timed regions
# ------------------------------------------------------------------------------------------------
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
           0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
           0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


class ClockSampler:
    def __init__(self, device_index: int, interval: float = 0.002):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._active = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[device_index]) if vis else device_index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return
        self.interval = interval
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            if self._active.is_set():
                try:
                    mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                    try:
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                    except Exception:
                        r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                    util = nv.nvmlDeviceGetUtilizationRates(self.h).gpu
                    self.samples.append((mhz, r, util))
                except Exception:
                    pass
            time.sleep(self.interval)

    def start(self):
        self._active.set()

    def pause(self):
        self._active.clear()

    def stop(self):
        self._stop.set()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"], "samples": 0}
        loaded = [s for s in self.samples if not (s[1] & 0x1)] or self.samples
        reasons = set()
        for _, r, _ in loaded:
            for bit, name in REASONS.items():
                if r & bit and bit != 0x1:
                    reasons.add(name)
        med = statistics.median([s[0] for s in loaded]) if loaded else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons), "samples": len(loaded)}


# ------------------------------------------------------------------------------------------------
# workloads
# ------------------------------------------------------------------------------------------------
def build_local(cfg: int, rank: int, world: int, dev, part_mode: int, distributed: bool = False):
    """Local CSR block (device) + global k + scaling mode."""
    if cfg == 1:
        M = 1 << 20
        mg = M * world
        p = synth.banded(mg, device=dev, row_begin=rank * M, row_end=(rank + 1) * M)
        return p, mg, rank * M * 16, "weak"
    if cfg == 0:
        return synth.config_pattern(0, device=dev), 1024, 0, "weak"
    full = synth.config_pattern(cfg, device=dev)
    if not distributed:
        return full, full.k, 0, "strong"
    from paper_1803_08601_b200 import dist
    bounds = dist.partition_rows(full.row_offsets.cpu(), world, part_mode)
    r0, r1 = bounds[rank], bounds[rank + 1]
    ro = full.row_offsets[r0:r1 + 1]
    z0, z1 = int(ro[0]), int(ro[-1])
    p = synth.CsrPattern(r1 - r0, full.k, (ro - z0).contiguous(), full.col_indices[z0:z1].contiguous(), full.name)
    return p, full.k, z0, "strong"


def bytes_alg(p: synth.CsrPattern, n: int) -> int:
    """4(m+1) + 8 nnz + 4n |distinct cols| + 4n m (fp32/int32 values, int32 indices)."""
    distinct = int(torch.unique(p.col_indices).numel()) if p.nnz else 0
    return 4 * (p.m + 1) + 8 * p.nnz + 4 * n * distinct + 4 * n * p.m


def load_traffic(workload_key: str):
    f = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(f) as fh:
            return json.load(fh).get(workload_key)
    except Exception:
        return None


# ------------------------------------------------------------------------------------------------
# oracle timing (cpu_baseline / --impl reference)
# ------------------------------------------------------------------------------------------------
def oracle_time_sample(p_cpu: synth.CsrPattern, val_cpu, B_cpu, n: int, budget_s: float):
    """Time the oracle (as it stands, all host cores via OpenMP) on the workload: the first R rows
    when the whole matrix would exceed budget_s, else the whole matrix repeated until about budget_s
    of CPU time has elapsed.  Returns (gflops, seconds_per_run, rows, flops_per_run, runs)."""
    import oracle
    ro = p_cpu.row_offsets.numpy()
    col = p_cpu.col_indices.numpy()
    vals = val_cpu.numpy()
    m = p_cpu.m

    def run(R):
        sub_ro = ro[:R + 1]
        z = int(sub_ro[-1])
        t0 = time.perf_counter()
        oracle.spmm("f32_plus_times", R, p_cpu.k, n, sub_ro, col[:z], vals[:z], B_cpu, ldb=n)
        return time.perf_counter() - t0, 2.0 * z * n

    R = min(m, 4096)
    dt, fl = run(R)
    while dt < 0.05 * budget_s and R < m:
        R = min(m, R * 4)
        dt, fl = run(R)
    if R < m:
        R = min(m, max(1, int(R * budget_s / max(dt, 1e-6))))
        dt, fl = run(R)
    runs, tot = 1, dt
    while tot < budget_s:  # whole workload fits the budget: repeat it
        d2, _ = run(R)
        tot += d2
        runs += 1
    return fl * runs / tot / 1e9, tot / runs, R, fl, runs


def oracle_one_thread(p_cpu, val_cpu, B_np, n, budget_s):
    """The oracle with OpenMP limited to one thread (restored afterwards); (GFLOP/s, rows) or None."""
    import ctypes
    import oracle
    try:
        gomp = ctypes.CDLL("libgomp.so.1")
        prev = gomp.omp_get_max_threads()
    except OSError:
        return None
    ro = p_cpu.row_offsets.numpy()
    col = p_cpu.col_indices.numpy()
    vals = val_cpu.numpy()
    gomp.omp_set_num_threads(1)
    try:
        R = min(p_cpu.m, 2048)
        while True:
            z = int(ro[R])
            t0 = time.perf_counter()
            oracle.spmm("f32_plus_times", R, p_cpu.k, n, ro[:R + 1], col[:z], vals[:z], B_np, ldb=n)
            dt = time.perf_counter() - t0
            if dt > 0.25 * budget_s or R >= p_cpu.m:
                return 2.0 * z * n / dt / 1e9, R
            R = min(p_cpu.m, R * 4)
    finally:
        gomp.omp_set_num_threads(prev)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ------------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 2, 4])
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--algo", default="auto", choices=["auto", "rowsplit", "merge"])
    ap.add_argument("--partition", default="merge_path", choices=["merge_path", "nonzero_split"])
    ap.add_argument("--items", type=int, default=0)
    ap.add_argument("--row-partition", type=int, default=1, help="multi-GPU: 0 nnz-balanced, 1 merge-path")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--gather-c", action="store_true", help="multi-GPU: also time an all-gather of C")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "timing rules: at least 3 warm-up steps"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n = args.n
    workload = WORKLOADS[args.config]
    # launched by torchrun (even with one rank): run the multi-GPU path -- NCCL process group, row-block
    # partition, broadcast of B, max-over-ranks reductions, optional all-gather of C
    distributed = world > 1 or "LOCAL_RANK" in os.environ

    if args.impl == "reference":
        return run_reference(args, world, rank, workload)

    import torch.distributed as tdist
    from paper_1803_08601_b200 import spmm as S

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if distributed:
        tdist.init_process_group("nccl", device_id=dev)

    def barrier():
        if distributed:
            tdist.barrier()

    kind = "f32_plus_times"
    seed = synth.STRUCT_SEED + args.config
    p, kg, zoff, scaling = build_local(args.config, rank, world, dev, args.row_partition, distributed)
    vals = synth.values(p.nnz, seed + 100, kind, device=dev, offset=zoff)
    # B: generated on rank 0, broadcast to all ranks (north_star: "B is replicated by an NCCL broadcast")
    B = torch.empty(kg, n, dtype=torch.float32, device=dev)
    if rank == 0:
        B.copy_(synth.dense(kg, n, seed + 200, kind, device=dev))
    bcast_ms = None
    if distributed:
        torch.cuda.synchronize()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tdist.broadcast(B, src=0)
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        bcast_ms = float(t.item())
    C = torch.empty(p.m, n, dtype=torch.float32, device=dev)

    op = S.CsrSpmm(p.row_offsets, p.col_indices, vals, kg)
    chosen = op.plan(n, args.algo, "plus_times", partition=args.partition, items_per_cta=args.items)
    info = op.info()
    nev = info["launches_per_execute"] + 1
    dominant = 1 if chosen == "rowsplit" else 2  # index of the dominant kernel's end event
    balg = bytes_alg(p, n)
    flops_local = 2.0 * p.nnz * n

    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.empty(int(2 * l2) // 4 + 1024, dtype=torch.float32, device=dev)
    sampler = ClockSampler(local_rank)

    def step(events=None):
        if events is not None:
            op.set_timing_events(events)
        op.execute(B, C)

    # warm-up
    for _ in range(args.warmup):
        if not args.no_flush:
            flush_buf.zero_()
        step()
    torch.cuda.synchronize()

    # timed region: K steps, per-step CUDA events recorded by the library around each kernel
    evsets = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)] for _ in range(args.steps)]
    for evs in evsets:  # torch creates the CUDA event lazily on first record: force creation
        for e in evs:
            e.record()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    for k in range(args.steps):
        if not args.no_flush:
            flush_buf.zero_()
        step(evsets[k])
    torch.cuda.synchronize()
    sampler.pause()
    barrier()
    op.set_timing_events([])
    step_ms = [ev[0].elapsed_time(ev[-1]) for ev in evsets]
    dom_ms = [ev[dominant - 1].elapsed_time(ev[dominant]) for ev in evsets]
    tot = torch.tensor([sum(step_ms), sum(dom_ms)], dtype=torch.float64, device=dev)
    if distributed:
        tdist.all_reduce(tot, op=tdist.ReduceOp.MAX)
        agg = torch.tensor([flops_local, float(balg), float(p.nnz)], dtype=torch.float64, device=dev)
        tdist.all_reduce(agg)
        flops_all, balg_all, nnz_all = (float(x) for x in agg.tolist())
    else:
        flops_all, balg_all, nnz_all = flops_local, float(balg), float(p.nnz)
    total_ms, dom_total_ms = float(tot[0]), float(tot[1])

    # warm-L2 companion number (the cold, flushed figure is primary): same steps, no flush
    warm_sets = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)] for _ in range(min(args.steps, 20))]
    for evs in warm_sets:
        for e in evs:
            e.record()
    torch.cuda.synchronize()
    for evs in warm_sets:
        step(evs)
    torch.cuda.synchronize()
    op.set_timing_events([])
    warm_ms = sorted(ev[0].elapsed_time(ev[-1]) for ev in warm_sets)[len(warm_sets) // 2]

    # optional all-gather of C, timed separately from the SpMM
    allgather_ms = None
    if distributed and args.gather_c:
        rows = torch.tensor([p.m], dtype=torch.int64, device=dev)
        allr = [torch.empty_like(rows) for _ in range(world)]
        tdist.all_gather(allr, rows)
        mx = max(int(r.item()) for r in allr)
        pad = torch.zeros(mx, n, dtype=C.dtype, device=dev)
        pad[:p.m] = C
        parts = [torch.empty_like(pad) for _ in range(world)]
        tdist.all_gather(parts, pad)  # warm-up
        torch.cuda.synchronize()
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        tdist.all_gather(parts, pad)
        g1.record()
        torch.cuda.synchronize()
        t = torch.tensor([g0.elapsed_time(g1)], device=dev)
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        allgather_ms = float(t.item())
        del parts, pad
    ms_per_step = total_ms / args.steps
    value = flops_all * args.steps / (total_ms / 1e3) / 1e9
    gbs = balg_all * args.steps / (total_ms / 1e3) / 1e9
    peak, peak_src = peaks()
    # roofline of the dominant kernel (this rank's algorithmic bytes / its average launch duration)
    dom_avg_ms = sum(dom_ms) / len(dom_ms)
    achieved = balg / (dom_avg_ms / 1e3) / 1e9
    kernel_name = "k_tile<ROWSPLIT>" if chosen == "rowsplit" else "k_tile<MERGE>"
    traffic = load_traffic(f"config{args.config}_n{n}|{kernel_name}") if world == 1 else None

    # ---------------- e2e: host buffers through the public API ----------------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, p, vals, B, kg, n, world, rank, dev, sampler, flops_all, tdist if distributed else None)
    sampler.stop()
    clocks = sampler.summary()

    # ---------------- cpu baseline (rank 0, N=1) ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        p_cpu = p.to("cpu")
        gfl, dt, R, fl, runs = oracle_time_sample(p_cpu, vals.cpu(), B.cpu().numpy(), n, args.cpu_budget)
        cpu = {"value": round(gfl, 4), "unit": UNIT, "cores": cores(), "kind": "oracle",
               "sample": f"oracle (plain C, fp64 accumulation + |A||B| bound, OpenMP) on the first {R} of {p.m} "
                         f"rows of the same workload ({fl / 2 / n:.0f} nnz) x {runs} runs, {dt:.3f} s per run"}
        # the oracle at 1 thread too (a smaller sample of the same rows)
        g1 = oracle_one_thread(p_cpu, vals.cpu(), B.cpu().numpy(), n, budget_s=4.0)
        if g1 is not None:
            cpu["value_1thread"] = round(g1[0], 4)
            cpu["sample_1thread"] = f"first {g1[1]} rows, 1 OpenMP thread"
            cpu["cpu_model"] = cpu_model()

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload, "n": n, "m_local": p.m, "k": kg, "nnz_total": int(nnz_all),
                       "algo": chosen, "policy": "auto" if args.algo == "auto" else "forced",
                       "partition": args.partition if chosen == "merge" else None,
                       "l2": "flushed before every timed step (2x L2 bytes written)" if not args.no_flush
                       else "not flushed",
                       "parallelism": f"row-block x{world}", "bcast_B_ms": bcast_ms, "allgather_C_ms": allgather_ms,
                       "step_plus_collectives_ms": (round(ms_per_step + (bcast_ms or 0.0) + (allgather_ms or 0.0), 5)
                                                    if (bcast_ms is not None or allgather_ms is not None) else None),
                       "mean_row_length": info["mean_row_length"], "max_row_length": info["max_row_length"]},
            "ms_per_step_median_rank0": round(statistics.median(step_ms), 5), "ms_per_step_min_rank0": round(min(step_ms), 5),
            "hbm_gbs_alg": round(gbs, 1), "bytes_alg_per_step": int(balg_all),
            "frac_of_roofline_step": round(gbs / peak, 4),
            "warm_l2_ms_per_step": round(warm_ms, 5), "frac_vs_nominal_8000": round(achieved / 8000.0, 4),
            "roofline": {"bound": "hbm", "kernel": kernel_name, "achieved": round(achieved, 1), "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "bytes_alg_per_launch": balg,
                         "avg_launch_ms": round(dom_avg_ms, 5)},
            "e2e": e2e, "gpu_launches": info["launches_per_execute"] * args.steps,
            "clocks": clocks, "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    op.close()
    if distributed:
        tdist.destroy_process_group()


def run_e2e(args, p, vals, B, kg, n, world, rank, dev, sampler, flops_all, tdist):
    """Same metric through the public API with HOST (pinned) buffers: every step copies the step's
    inputs (CSR block + B) host->device, creates + plans + executes, and reads C back."""
    from paper_1803_08601_b200 import spmm as S
    ro_h = p.row_offsets.cpu().pin_memory()
    col_h = p.col_indices.cpu().pin_memory()
    val_h = vals.cpu().pin_memory()
    B_h = B.cpu().pin_memory() if rank == 0 else None
    C_h = torch.empty(p.m, n, dtype=torch.float32).pin_memory()
    ro_d, col_d, val_d = torch.empty_like(p.row_offsets), torch.empty_like(p.col_indices), torch.empty_like(vals)
    B_d = torch.empty_like(B)
    C_d = torch.empty(p.m, n, dtype=torch.float32, device=dev)
    h2d = ro_h.numel() * 4 + col_h.numel() * 4 + val_h.numel() * 4 + (B_h.numel() * 4 if B_h is not None else 0)
    d2h = C_h.numel() * 4
    steps = max(3, min(args.steps, 10))

    def one():
        ro_d.copy_(ro_h, non_blocking=True)
        col_d.copy_(col_h, non_blocking=True)
        val_d.copy_(val_h, non_blocking=True)
        if B_h is not None:
            B_d.copy_(B_h, non_blocking=True)
        if tdist is not None:
            tdist.broadcast(B_d, src=0)
        op = S.CsrSpmm(ro_d, col_d, val_d, kg)
        op.plan(n, args.algo, "plus_times", partition=args.partition, items_per_cta=args.items)
        op.execute(B_d, C_d)
        C_h.copy_(C_d, non_blocking=True)
        op.close()

    one()
    torch.cuda.synchronize()
    if tdist is not None:
        tdist.barrier()
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        one()
    e1.record()
    torch.cuda.synchronize()
    sampler.pause()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if tdist is not None:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms = float(t.item()) / steps
    return {"value": round(flops_all / (ms / 1e3) / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 4), "steps": steps,
            "includes": "H2D(CSR block, B) + create + plan + execute + D2H(C) per step" +
                        (" + NCCL broadcast of B" if tdist is not None else "")}


def run_reference(args, world, rank, workload):
    """--impl reference: the oracle (plain C, oracle/) as it stands, on the host cores, rank 0 only."""
    if rank != 0:
        return
    n = args.n
    kind = "f32_plus_times"
    seed = synth.STRUCT_SEED + args.config
    if args.config == 1:
        p = synth.banded(1 << 20)
    else:
        p = synth.config_pattern(args.config, device="cuda" if torch.cuda.is_available() else "cpu").to("cpu")
    vals = synth.values(p.nnz, seed + 100, kind)
    B = synth.dense(p.k, n, seed + 200, kind).numpy()
    total_budget = 150.0
    per_step = max(0.5, min(15.0, total_budget / max(1, args.steps + args.warmup)))
    gfl, dt, R, fl, _ = oracle_time_sample(p, vals, B, n, per_step)
    # warm-up + K steps on that sample
    import numpy as np
    import oracle
    ro = p.row_offsets.numpy()[:R + 1]
    z = int(ro[-1])
    col = p.col_indices.numpy()[:z]
    v = vals.numpy()[:z]
    for _ in range(args.warmup):
        oracle.spmm(kind, R, p.k, n, ro, col, v, B, ldb=n)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.spmm(kind, R, p.k, n, ro, col, v, B, ldb=n)
        ts.append(time.perf_counter() - t0)
    tot = sum(ts)
    value = 2.0 * z * n * args.steps / tot / 1e9
    sample = (f"oracle (plain C, fp64 accumulation + |A||B| bound, OpenMP) on the first {R} of {p.m} rows "
              f"({z} nnz) of the same workload per step")
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot / args.steps * 1e3, 3),
           "higher_is_better": True, "scaling": "weak" if args.config in (0, 1) else "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": workload, "n": n},
           "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores(), "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
