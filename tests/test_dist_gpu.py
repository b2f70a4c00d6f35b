"""Multi-GPU path with the CUDA local SpMM (-m gpu): dist.RowBlockSpmm -- the code bench.py times --
against the CPU oracle.  Only one GPU is available to this build, so the exchange steps run
  * under NCCL with world size 1 (the real process-group / broadcast / grouped all-gather plumbing), and
  * under gloo with world size 2, both ranks on cuda:0 (two row blocks, real cross-rank exchange),
each with gather=True, both row partitions, fp32 checked against the oracle's |A||B| bound and the
exact semirings (int32 plus-times, min-plus) bit for bit (north_star tolerance)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1803_08601_b200 import synth

pytestmark = pytest.mark.gpu

KINDS = ["f32_plus_times", "i32_plus_times", "f32_min_plus", "i32_min_plus"]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(scale, kind, n):
    p = synth.rmat(scale, 16, 1800 + scale)
    val = synth.values(p.nnz, 1900 + scale, kind)
    B = synth.dense(p.k, n, 2000 + scale, kind)
    return p, val, B


def _worker(rank, world, port, backend, scale, kind, n, mode, algo, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    kw = {"device_id": dev} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        from paper_1803_08601_b200 import dist as D
        p, val, B = _case(scale, kind, n)
        sr = "plus_times" if kind.endswith("plus_times") else "min_plus"
        op = D.RowBlockSpmm(p.row_offsets, p.col_indices, val, p.k, mode=mode, device=dev)
        chosen = op.plan(n, algo, sr)
        Bd = op.broadcast_B(B.to(dev) if rank == 0 else None)
        C_local = op.execute(Bd)
        C_full = op.gather_C(C_local)
        torch.cuda.synchronize()
        q.put((rank, op.bounds, chosen, C_local.cpu().numpy(), C_full.cpu().numpy()))
        op.close()
    except Exception as e:  # surface worker failures to the test
        q.put((rank, None, repr(e), None, None))
        raise
    finally:
        dist.destroy_process_group()


def _run(world, backend, scale, kind, n, mode, algo):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, scale, kind, n, mode, algo, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r, bounds, chosen, cl, cf = q.get(timeout=300)
        assert bounds is not None, f"rank {r} failed: {chosen}"
        res[r] = (bounds, chosen, cl, cf)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    return res


def _check(kind, got, ref):
    if kind == "f32_plus_times":
        ok, worst, _ = oracle.check_f32(got, ref[0], ref[1], 1e-5)
        assert ok, f"worst |err|/bound = {worst}"
    else:
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo")])
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("kind", KINDS)
def test_row_blocks_cuda_vs_oracle(world, backend, mode, kind):
    scale, n = 13, 64
    res = _run(world, backend, scale, kind, n, mode, "auto")
    p, val, B = _case(scale, kind, n)
    ref = oracle.spmm(kind, p.m, p.k, n, p.row_offsets, p.col_indices, val, B)
    bounds = res[0][0]
    assert bounds[0] == 0 and bounds[-1] == p.m and len(bounds) == world + 1
    for r in range(world):
        assert res[r][0] == bounds
        r0, r1 = bounds[r], bounds[r + 1]
        ref_blk = (ref[0][r0:r1], ref[1][r0:r1]) if kind == "f32_plus_times" else ref[r0:r1]
        _check(kind, res[r][2], ref_blk)   # the rank's own rows
        _check(kind, res[r][3], ref)       # all of C after the gather, on every rank


@pytest.mark.parametrize("algo", ["rowsplit", "merge"])
def test_row_blocks_rmat16_both_kernels(algo):
    scale, n, kind = 16, 32, "f32_plus_times"
    res = _run(2, "gloo", scale, kind, n, 1, algo)
    p, val, B = _case(scale, kind, n)
    ref = oracle.spmm(kind, p.m, p.k, n, p.row_offsets, p.col_indices, val, B)
    for r in range(2):
        assert res[r][1] == algo
        _check(kind, res[r][3], ref)


# ------------------------------------------------------------------------------------------------
# NEXT-3: iterative SpMM with row-distributed X (CUDA local, split kernel, accumulate epilogue)
# NEXT-1: C all-gather fused into the SpMM (peer stores through CUDA IPC mappings)
# ------------------------------------------------------------------------------------------------
def _iter_worker(rank, world, port, backend, scale, kind, n, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    kw = {"device_id": dev} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        from paper_1803_08601_b200 import dist as D
        p, val, _ = _case(scale, kind, n)
        X = synth.dense(p.m, n, 3000 + scale, kind)
        sr = "plus_times" if kind.endswith("plus_times") else "min_plus"
        op = D.IterativeRowBlockSpmm(p.row_offsets, p.col_indices, val, mode=mode, device=dev)
        op.plan(n, "auto", sr)
        r0, r1 = op.bounds[rank], op.bounds[rank + 1]
        Y1 = op.step(X[r0:r1].to(dev))
        Y2 = op.step(X[r0:r1].to(dev))  # a second step reuses the gathered-X buffer and both plans
        torch.cuda.synchronize()
        q.put((rank, op.bounds, Y1.cpu().numpy(), Y2.cpu().numpy()))
        op.close()
    except Exception as e:
        q.put((rank, None, repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo")])
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("n", [4, 64])
def test_iterative_row_blocks_cuda_vs_oracle(world, backend, kind, n):
    scale = 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_iter_worker, args=(r, world, port, backend, scale, kind, n, 1, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r, bounds, y1, y2 = q.get(timeout=300)
        assert bounds is not None, f"rank {r} failed: {y1}"
        res[r] = (bounds, y1, y2)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    p, val, _ = _case(scale, kind, n)
    X = synth.dense(p.m, n, 3000 + scale, kind)
    ref = oracle.spmm(kind, p.m, p.k, n, p.row_offsets, p.col_indices, val, X)
    bounds = res[0][0]
    for r in range(world):
        r0, r1 = bounds[r], bounds[r + 1]
        blk = (ref[0][r0:r1], ref[1][r0:r1]) if kind == "f32_plus_times" else ref[r0:r1]
        _check(kind, res[r][1], blk)
        _check(kind, res[r][2], blk)


def _fused_worker(rank, world, port, backend, scale, kind, n, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    kw = {"device_id": dev} if backend == "nccl" else {}
    dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    try:
        from paper_1803_08601_b200 import dist as D
        p, val, B = _case(scale, kind, n)
        sr = "plus_times" if kind.endswith("plus_times") else "min_plus"
        op = D.RowBlockSpmm(p.row_offsets, p.col_indices, val, p.k, mode=mode, device=dev)
        op.plan(n, "auto", sr)
        Bd = op.broadcast_B(B.to(dev) if rank == 0 else None)
        Cf = op.enable_fused_gather()
        Cf.fill_(float("nan") if kind.startswith("f32") else -(2**31))
        out1 = op.execute_gather(Bd).cpu().numpy()
        dist.barrier()
        Cf.fill_(float("nan") if kind.startswith("f32") else -(2**31))  # every call rewrites every row
        dist.barrier()
        out2 = op.execute_gather(Bd).cpu().numpy()
        q.put((rank, op.bounds, out1, out2))
        op.close()
    except Exception as e:
        q.put((rank, None, repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo")])
@pytest.mark.parametrize("kind", KINDS)
@pytest.mark.parametrize("n", [8, 64])
def test_fused_gather_cuda_vs_oracle(world, backend, kind, n):
    """Each rank's kernels store its finished C rows into its own full C and, through CUDA IPC
    mappings, into every other rank's full C (two processes on one GPU here; NVLink peers on a node):
    after execute_gather every rank holds all of C, equal to the oracle."""
    scale = 13
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_worker, args=(r, world, port, backend, scale, kind, n, 1, q))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r, bounds, c1, c2 = q.get(timeout=300)
        assert bounds is not None, f"rank {r} failed: {c1}"
        res[r] = (bounds, c1, c2)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    p, val, B = _case(scale, kind, n)
    ref = oracle.spmm(kind, p.m, p.k, n, p.row_offsets, p.col_indices, val, B)
    for r in range(world):
        _check(kind, res[r][1], ref)
        _check(kind, res[r][2], ref)
