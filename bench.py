#!/usr/bin/env python
"""bench.py -- SpMM GFLOP/s and HBM GB/s (fraction of roofline) at n=64 on 1..N B200.

One "step" = one C = A*B through spmm_csr_execute (the whole hot path of SURVEY.md §8(a): for the
row-split choice one kernel, for merge: partition + compute + carry fix-up) over one synthetic input
resident in HBM.  Default workload = BASELINE.json configs[4], the config the metric's multi-GPU
target is quoted on: R-MAT scale 26 (Graph500 a,b,c,d = .57,.19,.19,.05, edge factor 16), n = 64,
fp32, strong scaling -- on N GPUs (torchrun) A is split into merge-path balanced row blocks
(dist.RowBlockSpmm: partition, slice, NCCL broadcast of B, local execute, optional all-gather of C --
the same object the multi-GPU tests check against the oracle).  On one GPU (no torchrun) configs[1]
(banded 2^20) and configs[2] (R-MAT 22) are measured in the same process as extra keys.  L2 is
flushed (2x L2 bytes written) before every timed step.

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle (oracle/, plain C) on a
bounded sample of the same workload instead.
"""
from __future__ import annotations

import argparse
import hashlib
import json
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
    4: "R-MAT scale 26, avg deg 16, n=64, fp32 plus-times, merge-path balanced row blocks, strong scaling "
       "(BASELINE configs[4])",
    2: "R-MAT scale 22, avg deg 16, n=64, fp32 plus-times (BASELINE configs[2])",
    1: "banded m=k=2^20 (x N ranks, weak), 16 nnz/row, n=64, fp32 plus-times (BASELINE configs[1])",
    0: "tiny uniform m=k=1024, 16 nnz/row, n=64, fp32 plus-times (BASELINE configs[0])",
}
KERNEL_NAMES = {"rowsplit": "k_tile<ROWSPLIT>", "merge": "k_merge_w"}


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
                    self.samples.append((mhz, r))
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
        for _, r in loaded:
            for bit, name in REASONS.items():
                if r & bit and bit != 0x1:
                    reasons.add(name)
        med = statistics.median([s[0] for s in loaded]) if loaded else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons), "samples": len(loaded)}


# ------------------------------------------------------------------------------------------------
# workload bookkeeping
# ------------------------------------------------------------------------------------------------
def bytes_alg(p: synth.CsrPattern, n: int) -> int:
    """4(m+1) + 8 nnz + 4n |distinct cols| + 4n m (fp32/int32 values, int32 indices)."""
    distinct = int(torch.unique(p.col_indices).numel()) if p.nnz else 0
    return 4 * (p.m + 1) + 8 * p.nnz + 4 * n * distinct + 4 * n * p.m


def static_l2_ceiling(p: synth.CsrPattern, n: int, l2_bytes: int, balg: int, peak_gbs: float) -> dict:
    """Attainable-fraction ceiling from a cache model for popularity-driven (independent-reference)
    gathers: an ideal static L2 that holds the hottest B rows (as many as fit in the whole L2,
    l2_bytes / 4n) and nothing else.  Every B-row gather to a
    row outside that set misses; every row is fetched at least once (compulsory).  CSR and C stream
    once.  HBM bytes of the model = CSR + C + 4n (distinct + sum over cold rows of (uses - 1)); the
    ceiling is bytes_alg / model bytes (an optimistic bound: real L2s also hold CSR/C lines and
    replace by recency, not by frequency)."""
    if p.nnz == 0:
        return {"model": "static-hot-rows", "frac_ceiling": 1.0}
    cnt = torch.bincount(p.col_indices.to(torch.int64), minlength=p.k)
    used = cnt[cnt > 0]
    hot = int(l2_bytes // (4 * n))
    srt = torch.sort(used, descending=True).values
    cold = srt[hot:]
    miss_extra = int((cold - 1).sum().item()) if cold.numel() else 0
    model = balg + 4 * n * miss_extra
    hits = int(srt[:hot].sum().item()) - min(hot, srt.numel())
    return {"model": "ideal static L2 holding the hottest B rows (l2 bytes / 4n rows)",
            "l2_bytes": l2_bytes, "model_hbm_bytes": int(model),
            "b_gather_hit_rate": round(hits / p.nnz, 4),
            "frac_ceiling": round(balg / model, 4),
            "t_ceiling_ms": round(model / (peak_gbs * 1e9) * 1e3, 4)}


def lib_sha16() -> str | None:
    from paper_1803_08601_b200 import spmm as S
    path = os.environ.get("SPMM_LIB") or S.LIB_PATH
    try:
        with open(path, "rb") as f:
            return hashlib.sha256(f.read()).hexdigest()[:16]
    except OSError:
        return None


def load_traffic(key: str, sha: str | None):
    """ncu DRAM bytes / L2 hit rate of the dominant kernel for this workload, from the committed
    capture (profiles/ncu_traffic.json, written by scripts/ncu_summary.py) -- reported only with the
    library hash it was captured from, so a stale capture is visible as such."""
    f = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(f) as fh:
            ent = json.load(fh).get(key)
    except Exception:
        return None
    if ent is None:
        return None
    if not isinstance(ent, dict):
        ent = {"dram_bytes": ent}
    ent = dict(ent)
    # same build = the same .so, or the same sources and flags (nvcc builds are not bit-reproducible:
    # paper_1803_08601_b200.build.source_sha16); a variant library (SPMM_LIB) matches only by its hash
    same_lib = (ent.get("lib_sha16") == sha) if sha else None
    same_src = None
    if not os.environ.get("SPMM_LIB") and ent.get("src_sha16"):
        from paper_1803_08601_b200 import build as _build
        same_src = ent["src_sha16"] == _build.source_sha16()
    ent["same_build"] = bool(same_lib or same_src) if (same_lib is not None or same_src is not None) else None
    return ent


def physical_cores():
    try:
        import subprocess
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = dict(line.split(":", 1) for line in out.splitlines() if ":" in line)
        return int(kv["Core(s) per socket"].strip()) * int(kv.get("Socket(s)", "1").strip())
    except Exception:
        return None


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
# oracle timing (cpu_baseline / --impl reference)
# ------------------------------------------------------------------------------------------------
def _prefix_cpu(p: synth.CsrPattern, vals, rows: int):
    """The first `rows` rows of a (device) CSR and its values, on the host."""
    ro = p.row_offsets[:rows + 1].cpu().numpy()
    z = int(ro[-1])
    return ro, p.col_indices[:z].cpu().numpy(), vals[:z].cpu().numpy()


def oracle_time_sample(p: synth.CsrPattern, vals, B_np, n: int, budget_s: float):
    """Time the oracle (as it stands, all host cores via OpenMP) on a prefix of the workload's rows
    sized to about budget_s; the whole matrix is repeated instead when it fits the budget.
    Returns (gflops, seconds_per_run, rows, flops_per_run, runs)."""
    import oracle
    m = p.m

    def run(R):
        ro, col, v = _prefix_cpu(p, vals, R)
        t0 = time.perf_counter()
        oracle.spmm("f32_plus_times", R, p.k, n, ro, col, v, B_np, ldb=n)
        return time.perf_counter() - t0, 2.0 * int(ro[-1]) * n

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


def oracle_one_thread(p, vals, B_np, n, budget_s):
    """The oracle with OpenMP limited to one thread (restored afterwards); (GFLOP/s, rows) or None."""
    import ctypes
    import oracle
    try:
        gomp = ctypes.CDLL("libgomp.so.1")
        prev = gomp.omp_get_max_threads()
    except OSError:
        return None
    gomp.omp_set_num_threads(1)
    try:
        R = min(p.m, 2048)
        while True:
            ro, col, v = _prefix_cpu(p, vals, R)
            t0 = time.perf_counter()
            oracle.spmm("f32_plus_times", R, p.k, n, ro, col, v, B_np, ldb=n)
            dt = time.perf_counter() - t0
            if dt > 0.25 * budget_s or R >= p.m:
                return 2.0 * int(ro[-1]) * n / dt / 1e9, R
            R = min(p.m, R * 4)
    finally:
        gomp.omp_set_num_threads(prev)


# ------------------------------------------------------------------------------------------------
# device timing of one planned operator
# ------------------------------------------------------------------------------------------------
def time_steps(op_local, execute, steps: int, warmup: int, flush_buf, sampler, barrier, no_flush=False):
    """W warm-up + K timed executes with per-kernel CUDA events recorded by the library on the execute
    stream (spmm_csr_set_timing_events).  Returns (step_ms list, compute-kernel ms list)."""
    info = op_local.info()
    nev = info["launches_per_execute"] + 1
    ci = info["compute_launch"]
    for _ in range(warmup):
        if not no_flush:
            flush_buf.zero_()
        execute()
    torch.cuda.synchronize()
    evsets = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)] for _ in range(steps)]
    for evs in evsets:  # torch creates the CUDA event lazily on first record: force creation
        for e in evs:
            e.record()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    for k in range(steps):
        if not no_flush:
            flush_buf.zero_()
        op_local.set_timing_events(evsets[k])
        execute()
    torch.cuda.synchronize()
    sampler.pause()
    barrier()
    op_local.set_timing_events([])
    step_ms = [ev[0].elapsed_time(ev[-1]) for ev in evsets]
    dom_ms = [ev[ci].elapsed_time(ev[ci + 1]) for ev in evsets]
    return step_ms, dom_ms


def measure_single(cfg: int, n: int, args, dev, flush_buf, sampler, peak, l2_bytes, sha, with_ceiling=True):
    """One GPU, no process group: plan + K timed executes of configs[cfg] through CsrSpmm."""
    from paper_1803_08601_b200 import spmm as S
    kind = "f32_plus_times"
    seed = synth.STRUCT_SEED + cfg
    p = synth.config_pattern(cfg, device=dev)
    vals = synth.values(p.nnz, seed + 100, kind, device=dev)
    B = synth.dense(p.k, n, seed + 200, kind, device=dev)
    C = torch.empty(p.m, n, dtype=torch.float32, device=dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = S.CsrSpmm(p.row_offsets, p.col_indices, vals, p.k)
    chosen = op.plan(n, args.algo, "plus_times", partition=args.partition, items_per_cta=args.items,
                     merge_worker=args.merge_worker, tasks_per_warp=args.tasks_per_warp)
    torch.cuda.synchronize()
    plan_ms = (time.perf_counter() - t0) * 1e3
    info = op.info()
    step_ms, dom_ms = time_steps(op, lambda: op.execute(B, C), args.steps, args.warmup, flush_buf, sampler,
                                 lambda: None, args.no_flush)
    balg = bytes_alg(p, n)
    res = summarize(p, n, balg, chosen, info, step_ms, dom_ms, args.steps, peak, sha, cfg, plan_ms)
    if with_ceiling:
        if info.get("bspan_compact", -1.0) >= 0.5:
            # clustered columns (banded / mesh-like): a tile's B rows are re-read while L2-resident, so the
            # attainable traffic is the compulsory one (each B row once) -- the frequency model below only
            # describes independent, popularity-driven references (R-MAT) and would understate this case
            res["roofline"]["ceiling"] = {"model": "compulsory bytes (B row spans compact: temporal reuse in L2)",
                                          "bspan_compact": round(info["bspan_compact"], 4), "frac_ceiling": 1.0,
                                          "t_ceiling_ms": round(balg / (peak[0] * 1e9) * 1e3, 4)}
        else:
            res["roofline"]["ceiling"] = static_l2_ceiling(p, n, l2_bytes, balg, peak[0])
    return res, (p, vals, B, C, op)


def summarize(p, n, balg, chosen, info, step_ms, dom_ms, steps, peak, sha, cfg, plan_ms):
    total_ms = sum(step_ms)
    flops = 2.0 * p.nnz * n
    dom_avg = sum(dom_ms) / len(dom_ms)
    achieved = balg / (dom_avg / 1e3) / 1e9
    kname = KERNEL_NAMES[chosen]
    ncu = load_traffic(f"config{cfg}_n{n}|{kname}", sha)
    return {
        "workload": WORKLOADS[cfg], "m": p.m, "k": p.k, "nnz": p.nnz, "n": n, "algo": chosen,
        "mean_row_length": info["mean_row_length"], "max_row_length": info["max_row_length"],
        "items_per_task": info["items_per_cta"] if chosen == "merge" else None,
        "value": round(flops * steps / (total_ms / 1e3) / 1e9, 3), "unit": UNIT,
        "ms_per_step": round(total_ms / steps, 5),
        "ms_per_step_median": round(statistics.median(step_ms), 5), "ms_per_step_min": round(min(step_ms), 5),
        "plan_ms": round(plan_ms, 3),
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1), "peak": peak[0],
                     "peak_source": peak[1], "unit": "GB/s", "frac": round(achieved / peak[0], 4),
                     "frac_vs_nominal_8000": round(achieved / 8000.0, 4),
                     "traffic": ncu.get("dram_bytes") if ncu else None,
                     "traffic_over_alg": round(ncu["dram_bytes"] / balg, 3) if ncu and ncu.get("dram_bytes") else None,
                     "dram_gbs_at_traffic": round(ncu["dram_bytes"] / (dom_avg / 1e3) / 1e9, 1)
                     if ncu and ncu.get("dram_bytes") else None,
                     "bytes_alg_per_launch": int(balg), "avg_launch_ms": round(dom_avg, 5), "ncu": ncu},
        "launches_per_step": info["launches_per_execute"],
    }


# ------------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[0, 1, 2, 4])
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--algo", default="auto", choices=["auto", "rowsplit", "merge"])
    ap.add_argument("--partition", default="merge_path", choices=["merge_path", "nonzero_split"])
    ap.add_argument("--items", type=int, default=0)
    ap.add_argument("--merge-worker", default="auto", choices=["auto", "warp", "folded"])
    ap.add_argument("--tasks-per-warp", type=int, default=0)
    ap.add_argument("--row-partition", type=int, default=1, help="multi-GPU: 0 nnz-balanced, 1 merge-path")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--gather-c", action="store_true", help="multi-GPU: also time the all-gather of C")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the configs[1]/[2] keys on one GPU")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-budget", type=float, default=12.0, help="seconds of oracle work for cpu_baseline")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "timing rules: at least 3 warm-up steps"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # launched by torchrun (even with one rank): the multi-GPU path -- NCCL process group, row-block
    # partition, broadcast of B, max-over-ranks reductions, optional all-gather of C
    distributed = world > 1 or "LOCAL_RANK" in os.environ
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch.distributed as tdist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if distributed:
        tdist.init_process_group("nccl", device_id=dev)
    n = args.n
    peak = peaks()
    sha = lib_sha16()
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush_buf = torch.empty(int(2 * l2) // 4 + 1024, dtype=torch.float32, device=dev)
    sampler = ClockSampler(local_rank)

    if distributed:
        head, ctx = measure_distributed(args, world, rank, dev, flush_buf, sampler, peak, sha, l2)
    else:
        head, ctx = measure_single(args.config, n, args, dev, flush_buf, sampler, peak, l2, sha)
        head["scaling"] = "weak" if args.config in (0, 1) else "strong"
        head["bcast_B_ms"] = head["allgather_C_ms"] = None
        head["flops_all"] = 2.0 * head["nnz"] * n
        head["ms_max"] = head["ms_per_step"]

    # ---------------- e2e: host buffers through the public API ----------------
    e2e = None
    if not args.no_e2e:
        if distributed:
            e2e = run_e2e(args, ctx, n, world, rank, dev, sampler, head["flops_all"], distributed)
        else:
            # one GPU: host copies of the step's inputs, then the device-resident workload is released
            # (the library's own pool holds the e2e device buffers, one set per stream in flight)
            host = e2e_host_inputs(ctx, n)
            ctx[4].close()
            ctx = None
            torch.cuda.empty_cache()
            e2e = run_e2e_pipelined(args, host, n, dev, sampler, head["flops_all"])
    # ---------------- extra configs in the same process (one GPU) ----------------
    extras = {}
    if not distributed and not args.no_extras:
        ctx = None
        torch.cuda.empty_cache()
        for cfg in (1, 2):
            if cfg == args.config:
                continue
            r, c2 = measure_single(cfg, n, args, dev, flush_buf, sampler, peak, l2, sha)
            c2[4].close()
            del c2
            torch.cuda.empty_cache()
            extras[f"config{cfg}"] = r
    sampler.stop()
    clocks = sampler.summary()

    # ---------------- cpu baseline (rank 0, N=1) ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, n, dev, args.cpu_budget)

    if rank == 0:
        roof = head["roofline"]
        out = {
            "metric": METRIC, "value": head["value_all"] if distributed else head["value"], "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": head["ms_max"], "higher_is_better": True, "scaling": head["scaling"],
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": head["workload"], "n": n, "m": head["m"], "k": head["k"], "nnz_total": head["nnz"],
                       "algo": head["algo"], "policy": "auto" if args.algo == "auto" else "forced",
                       "partition": args.partition if head["algo"] == "merge" else None,
                       "items_per_task": head["items_per_task"],
                       "l2": "flushed before every timed step (2x L2 bytes written)" if not args.no_flush
                       else "not flushed",
                       "parallelism": f"row-block x{world}",
                       "row_partition": ("merge-path balanced" if args.row_partition == 1 else "nnz-balanced")
                       if distributed else None,
                       "bcast_B_ms": head["bcast_B_ms"], "allgather_C_ms": head["allgather_C_ms"],
                       "mean_row_length": head["mean_row_length"], "max_row_length": head["max_row_length"]},
            "ms_per_step_median_rank0": head["ms_per_step_median"], "ms_per_step_min_rank0": head["ms_per_step_min"],
            "plan_ms": head["plan_ms"],
            "roofline": roof,
            "e2e": e2e, "gpu_launches": head["launches_per_step"] * args.steps,
            "clocks": clocks, "cpu_baseline": cpu, "lib_sha16": sha,
        }
        for key, r in extras.items():
            out[key] = r
        print(json.dumps(out), flush=True)
    if distributed:
        tdist.destroy_process_group()


def measure_distributed(args, world, rank, dev, flush_buf, sampler, peak, sha, l2):
    """torchrun: dist.RowBlockSpmm (the shipped multi-GPU path).  Config 1 is weak scaling (rank r
    generates banded block r of an N*2^20-row matrix), the R-MAT configs strong scaling over
    merge-path (or nnz) balanced row blocks of the whole matrix."""
    import torch.distributed as tdist
    from paper_1803_08601_b200 import dist as D
    n = args.n
    kind = "f32_plus_times"
    seed = synth.STRUCT_SEED + args.config
    if args.config == 1:
        M = 1 << 20
        kg = M * world
        p = synth.banded(kg, device=dev, row_begin=rank * M, row_end=(rank + 1) * M)
        vals = synth.values(p.nnz, seed + 100, kind, device=dev, offset=rank * M * 16)
        scaling = "weak"
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op = D.RowBlockSpmm(p.row_offsets, p.col_indices, vals, kg, local=True, device=dev)
    else:
        full = synth.config_pattern(args.config, device=dev)
        fvals = synth.values(full.nnz, seed + 100, kind, device=dev)
        kg = full.k
        scaling = "strong"
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        op = D.RowBlockSpmm(full.row_offsets, full.col_indices, fvals, kg, mode=args.row_partition, device=dev)
        r0, r1 = op.bounds[rank], op.bounds[rank + 1]
        p = synth.CsrPattern(r1 - r0, kg, op.ro, op.col, full.name)
        vals = op.val
        del full, fvals
    chosen = op.plan(n, args.algo, "plus_times", partition=args.partition, items_per_cta=args.items,
                     merge_worker=args.merge_worker, tasks_per_warp=args.tasks_per_warp)
    torch.cuda.synchronize()
    plan_ms = (time.perf_counter() - t0) * 1e3
    info = op.info()
    # exchange step 1: B generated on rank 0, NCCL broadcast (timed separately, max over ranks)
    B = torch.empty(kg, n, dtype=torch.float32, device=dev)
    if rank == 0:
        B.copy_(synth.dense(kg, n, seed + 200, kind, device=dev))
    torch.cuda.synchronize()
    tdist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    op.broadcast_B(out=B)
    e1.record()
    torch.cuda.synchronize()
    bcast_ms = _max_over_ranks(e0.elapsed_time(e1), dev)
    C = torch.empty(op.m_local, n, dtype=torch.float32, device=dev)
    step_ms, dom_ms = time_steps(op.local.op, lambda: op.execute(B, C), args.steps, args.warmup, flush_buf,
                                 sampler, tdist.barrier, args.no_flush)
    balg = bytes_alg(p, n)
    res = summarize(p, n, balg, chosen, info, step_ms, dom_ms, args.steps, peak, sha, args.config, plan_ms)
    tot = torch.tensor([sum(step_ms), float(p.nnz), float(balg)], dtype=torch.float64, device=dev)
    mx = tot.clone()
    tdist.all_reduce(mx, op=tdist.ReduceOp.MAX)
    tdist.all_reduce(tot)
    res["ms_max"] = round(float(mx[0]) / args.steps, 5)
    res["flops_all"] = 2.0 * float(tot[1]) * n
    res["value_all"] = round(res["flops_all"] * args.steps / (float(mx[0]) / 1e3) / 1e9, 3)
    res["nnz"] = int(tot[1])
    res["m"] = op.m
    res["bytes_alg_all"] = int(tot[2])
    res["roofline"]["rank"] = rank
    res["scaling"] = scaling
    res["bcast_B_ms"] = round(bcast_ms, 4)
    # exchange step 2 (optional): the C gather (grouped broadcasts of the uneven row blocks)
    res["allgather_C_ms"] = None
    if args.gather_c:
        Cfull = torch.empty(op.m, n, dtype=torch.float32, device=dev)
        op.gather_C(C, Cfull)
        torch.cuda.synchronize()
        tdist.barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record()
        op.gather_C(C, Cfull)
        g1.record()
        torch.cuda.synchronize()
        res["allgather_C_ms"] = round(_max_over_ranks(g0.elapsed_time(g1), dev), 4)
        del Cfull
    return res, (p, vals, B, C, op)


def _max_over_ranks(x: float, dev) -> float:
    import torch.distributed as tdist
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def run_e2e(args, ctx, n, world, rank, dev, sampler, flops_all, distributed):
    """Same metric through the public API with HOST (pinned) buffers: every step copies the step's
    inputs (this rank's CSR block + B on rank 0) host->device, (broadcasts B,) creates + plans +
    executes, and reads this rank's C rows back."""
    from paper_1803_08601_b200 import spmm as S
    p, vals, B, C, op = ctx
    kg = p.k
    ro_h = p.row_offsets.cpu().pin_memory()
    col_h = p.col_indices.cpu().pin_memory()
    val_h = vals.cpu().pin_memory()
    B_h = B.cpu().pin_memory() if rank == 0 else None
    C_h = torch.empty(p.m, n, dtype=torch.float32, pin_memory=True)
    h2d = ro_h.numel() * 4 + col_h.numel() * 4 + val_h.numel() * 4 + (B_h.numel() * 4 if B_h is not None else 0)
    d2h = C_h.numel() * 4
    ro_d, col_d, val_d = torch.empty_like(p.row_offsets), torch.empty_like(p.col_indices), torch.empty_like(vals)
    B_d = B  # reuse the device allocation (its contents are overwritten by the H2D copy / broadcast)
    C_d = C
    import torch.distributed as tdist

    def one():
        ro_d.copy_(ro_h, non_blocking=True)
        col_d.copy_(col_h, non_blocking=True)
        val_d.copy_(val_h, non_blocking=True)
        if B_h is not None:
            B_d.copy_(B_h, non_blocking=True)
        if distributed:
            tdist.broadcast(B_d, src=0)
        o = S.CsrSpmm(ro_d, col_d, val_d, kg)
        o.plan(n, args.algo, "plus_times", partition=args.partition, items_per_cta=args.items,
                     merge_worker=args.merge_worker, tasks_per_warp=args.tasks_per_warp)
        o.execute(B_d, C_d)
        C_h.copy_(C_d, non_blocking=True)
        o.close()

    one()
    torch.cuda.synchronize()
    if distributed:
        tdist.barrier()
    steps = max(1, args.e2e_steps)
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        one()
    e1.record()
    torch.cuda.synchronize()
    sampler.pause()
    ms = e0.elapsed_time(e1)
    if distributed:
        ms = _max_over_ranks(ms, dev)
    ms /= steps
    return {"value": round(flops_all / (ms / 1e3) / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 4), "steps": steps,
            "includes": "H2D(CSR block, B) + create + plan + execute + D2H(C block) per step" +
                        (" + NCCL broadcast of B" if distributed else "")}


def e2e_host_inputs(ctx, n):
    """Pinned host copies of one step's inputs (CSR + B) and two pinned C buffers."""
    p, vals, B, C, _ = ctx
    return {"m": p.m, "k": p.k, "ro": p.row_offsets.cpu().pin_memory(), "col": p.col_indices.cpu().pin_memory(),
            "val": vals.cpu().pin_memory(), "B": B.cpu().pin_memory(),
            "C": [torch.empty(p.m, n, dtype=torch.float32, pin_memory=True) for _ in range(2)]}


def run_e2e_pipelined(args, host, n, dev, sampler, flops_all):
    """One GPU: every step is ONE C-ABI call on pinned HOST buffers (spmm_csr_multiply_host: the library
    copies the CSR and B in, creates + plans + executes, copies C out; stream-ordered device buffers).
    Steps alternate between two streams, so step k's host->device copies overlap step k-1's read-back
    (PCIe is full duplex), as a serving loop would run them; each step still moves all of its bytes."""
    from paper_1803_08601_b200 import spmm as S
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    h2d = 4 * (host["ro"].numel() + host["col"].numel() + host["val"].numel() + host["B"].numel())
    d2h = 4 * host["C"][0].numel()

    def step(k):
        S.multiply_host(host["ro"], host["col"], host["val"], host["k"], host["B"], host["C"][k % 2], algo=args.algo,
                        stream=streams[k % 2], sync=False)

    step(0)  # warm-up on both streams (primes the library's memory pool with one buffer set per stream)
    step(1)
    torch.cuda.synchronize()
    steps = max(1, args.e2e_steps)
    sampler.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams:
        s.wait_event(e0)
    for k in range(steps):
        step(k)
    for s in streams:
        torch.cuda.current_stream(dev).wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    sampler.pause()
    ms = e0.elapsed_time(e1) / steps
    return {"value": round(flops_all / (ms / 1e3) / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ms, 4), "steps": steps,
            "includes": "per step one C-ABI call on pinned host buffers (spmm_csr_multiply_host: H2D of CSR + B, "
                        "create + plan + execute, D2H of C); steps alternate two streams so a step's H2D overlaps "
                        "the previous step's D2H"}


def cpu_baseline(cfg, n, dev, budget):
    """The oracle on the GPU box's host cores, on a prefix of the same workload's rows."""
    kind = "f32_plus_times"
    seed = synth.STRUCT_SEED + cfg
    p = synth.config_pattern(cfg, device=dev)
    vals = synth.values(p.nnz, seed + 100, kind, device=dev)
    B_np = synth.dense(p.k, n, seed + 200, kind, device=dev).cpu().numpy()
    gfl, dt, R, fl, runs = oracle_time_sample(p, vals, B_np, n, budget)
    cpu = {"value": round(gfl, 4), "unit": UNIT, "cores": cores(), "physical_cores": physical_cores(),
           "kind": "oracle", "cpu_model": cpu_model(),
           "sample": f"oracle (plain C, fp64 accumulation + |A||B| bound, OpenMP) on the first {R} of {p.m} "
                     f"rows of the same workload ({fl / 2 / n:.0f} nnz) x {runs} runs, {dt:.3f} s per run"}
    g1 = oracle_one_thread(p, vals, B_np, n, budget_s=4.0)
    if g1 is not None:
        cpu["value_1thread"] = round(g1[0], 4)
        cpu["sample_1thread"] = f"first {g1[1]} rows, 1 OpenMP thread"
    return cpu


def run_reference(args, world, rank):
    """--impl reference: the oracle (plain C, oracle/) as it stands, on the host cores, rank 0 only,
    each step a bounded prefix of the same workload's rows."""
    if rank != 0:
        return
    n = args.n
    kind = "f32_plus_times"
    seed = synth.STRUCT_SEED + args.config
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    p = synth.config_pattern(args.config, device=dev)
    vals = synth.values(p.nnz, seed + 100, kind, device=dev)
    B = synth.dense(p.k, n, seed + 200, kind, device=dev).cpu().numpy()
    total_budget = 150.0
    per_step = max(0.5, min(15.0, total_budget / max(1, args.steps + args.warmup)))
    gfl, dt, R, fl, _ = oracle_time_sample(p, vals, B, n, per_step)
    import oracle
    ro, col, v = _prefix_cpu(p, vals, R)
    z = int(ro[-1])
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
           "config": {"workload": WORKLOADS[args.config], "n": n, "m": p.m, "k": p.k, "nnz_total": p.nnz,
                      "sample_rows": R, "sample_nnz": z},
           "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores(),
                            "physical_cores": physical_cores(), "kind": "oracle", "sample": sample},
           "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
