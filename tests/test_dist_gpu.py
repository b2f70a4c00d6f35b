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
