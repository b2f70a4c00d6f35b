"""Multi-process host logic of the multi-GPU path (north_star), on CPU with the gloo
backend, world_size 2: row-block partition through the C ABI, CSR slicing with rebased offsets,
broadcast of B from rank 0, optional all-gather of C.  The per-rank SpMM is injected (the CPU oracle
here; the CUDA path on GPUs), so these tests cover exactly the exchange and bookkeeping steps."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1803_08601_b200 import dist as D
from paper_1803_08601_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_local(kind):
    """Per-rank SpMM stand-in for the CPU tests: the oracle behind the RowBlockSpmm local interface."""
    class OracleLocal:
        def __init__(self, ro, col, val, k):
            self.ro, self.col, self.val, self.k = ro, col, val, k

        def plan(self, n, algo="auto", semiring="plus_times", **kw):
            self.n = n
            return algo

        def execute(self, B, C=None):
            m = self.ro.numel() - 1
            out = oracle.spmm(kind, m, self.k, self.n, self.ro, self.col, self.val, B)
            out = torch.from_numpy(out[0].astype(np.float32) if kind == "f32_plus_times" else out)
            if C is not None:
                C.copy_(out)
                return C
            return out

        def info(self):
            return {}

        def close(self):
            pass
    return OracleLocal


def _worker(rank, world, port, kind, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = synth.rmat(10, 8, 77)
        val = synth.values(p.nnz, 5, kind)
        n = 33
        B = synth.dense(p.k, n, 6, kind) if rank == 0 else torch.empty(0)
        C_local, bounds = D.distributed_spmm(p.row_offsets, p.col_indices, val, B, p.k, n, mode=mode,
                                             gather=False, local_factory=_oracle_local(kind),
                                             device=torch.device("cpu"))
        C_full, bounds2 = D.distributed_spmm(p.row_offsets, p.col_indices, val, B, p.k, n, mode=mode,
                                             gather=True, local_factory=_oracle_local(kind),
                                             device=torch.device("cpu"))
        q.put((rank, bounds, C_local.numpy(), C_full.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["f32_plus_times", "i32_min_plus"])
@pytest.mark.parametrize("mode", [0, 1])
def test_distributed_spmm_gloo_world2(kind, mode):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, mode, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r, bounds, cl, cf = q.get(timeout=120)
        res[r] = (bounds, cl, cf)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = synth.rmat(10, 8, 77)
    val = synth.values(p.nnz, 5, kind)
    B = synth.dense(p.k, 33, 6, kind)
    ref = oracle.spmm(kind, p.m, p.k, 33, p.row_offsets, p.col_indices, val, B)
    ref = ref[0].astype(np.float32) if kind == "f32_plus_times" else ref
    bounds = res[0][0]
    assert res[1][0] == bounds and bounds[0] == 0 and bounds[-1] == p.m
    # each rank's block equals the matching rows of the single-process result (bit-exact: same per-row order)
    for r in range(world):
        assert np.array_equal(res[r][1], ref[bounds[r]:bounds[r + 1]])
        assert np.array_equal(res[r][2], ref)  # all-gathered C on every rank


def test_partition_balances_nnz_and_items():
    p = synth.rmat(12, 16, 3)
    ro = p.row_offsets.numpy().astype(np.int64)
    for parts in (2, 4, 8):
        b0 = D.partition_rows(p.row_offsets, parts, 0)
        b1 = D.partition_rows(p.row_offsets, parts, 1)
        nnz_blocks = [ro[b0[i + 1]] - ro[b0[i]] for i in range(parts)]
        items = [(b1[i + 1] - b1[i]) + ro[b1[i + 1]] - ro[b1[i]] for i in range(parts)]
        maxrow = int(np.diff(ro).max())
        assert max(nnz_blocks) - min(nnz_blocks) <= 2 * maxrow + 2  # rows are never split
        assert max(items) - min(items) <= 2 * maxrow + 2
    sl = D.slice_rows(p.row_offsets, p.col_indices, synth.values(p.nnz, 1, "f32_plus_times"), 5, 9)
    assert sl[0][0] == 0 and sl[0].numel() == 5 and sl[1].numel() == int(ro[9] - ro[5])
