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

        def execute(self, B, C=None, accumulate=False):
            m = self.ro.numel() - 1
            out = oracle.spmm(kind, m, self.k, self.n, self.ro, self.col, self.val, B)
            out = torch.from_numpy(out[0].astype(np.float32) if kind == "f32_plus_times" else out)
            if accumulate:  # C (+)= A B in the semiring
                out = torch.minimum(C, out) if kind.endswith("min_plus") else C + out
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


def _split_numpy(ro, col, val, c0, c1):
    """CPU stand-in for spmm_csr_split_columns: per row, entries with column in [c0, c1) (rebased) and
    the others, storage order kept."""
    ro_n, col_n, val_n = ro.numpy(), col.numpy(), val.numpy()
    parts = ([0], [], [], [0], [], [])
    for r in range(len(ro_n) - 1):
        c = col_n[ro_n[r]:ro_n[r + 1]]
        v = val_n[ro_n[r]:ro_n[r + 1]]
        inside = (c >= c0) & (c < c1)
        parts[1].extend((c[inside] - c0).tolist())
        parts[2].extend(v[inside].tolist())
        parts[0].append(len(parts[1]))
        parts[4].extend(c[~inside].tolist())
        parts[5].extend(v[~inside].tolist())
        parts[3].append(len(parts[4]))
    t = lambda x, dt: torch.tensor(x, dtype=dt)  # noqa: E731
    return ((t(parts[0], torch.int32), t(parts[1], torch.int32), t(parts[2], val.dtype)),
            (t(parts[3], torch.int32), t(parts[4], torch.int32), t(parts[5], val.dtype)))


def _iter_worker(rank, world, port, kind, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = synth.rmat(9, 8, 78)
        val = synth.values(p.nnz, 15, kind)
        n = 5
        X = synth.dense(p.m, n, 16, kind)
        op = D.IterativeRowBlockSpmm(p.row_offsets, p.col_indices, val, mode=mode, device=torch.device("cpu"),
                                     local_factory=_oracle_local(kind), split_fn=_split_numpy)
        op.plan(n, "auto", "plus_times" if kind.endswith("plus_times") else "min_plus")
        r0, r1 = op.bounds[rank], op.bounds[rank + 1]
        Y = op.step(X[r0:r1].clone())
        q.put((rank, op.bounds, Y.numpy(), op.nnz_diag, op.nnz_off))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["f32_plus_times", "i32_plus_times", "i32_min_plus"])
@pytest.mark.parametrize("mode", [0, 1])
def test_iterative_row_blocks_gloo_world2(kind, mode):
    """NEXT-3 host logic: split of each row block into diagonal / off-diagonal parts, all-gather of the
    row-distributed X, diagonal product then accumulated off-diagonal product, against the oracle."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_iter_worker, args=(r, world, port, kind, mode, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r, bounds, Y, zd, zo = q.get(timeout=120)
        res[r] = (bounds, Y, zd, zo)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = synth.rmat(9, 8, 78)
    val = synth.values(p.nnz, 15, kind)
    X = synth.dense(p.m, 5, 16, kind)
    ref = oracle.spmm(kind, p.m, p.k, 5, p.row_offsets, p.col_indices, val, X)
    bounds = res[0][0]
    assert sum(res[r][2] + res[r][3] for r in range(world)) == p.nnz
    assert all(res[r][3] > 0 for r in range(world))  # both ranks really use the gathered X
    for r in range(world):
        r0, r1 = bounds[r], bounds[r + 1]
        if kind == "f32_plus_times":
            ok, worst, _ = oracle.check_f32(res[r][1], ref[0][r0:r1], ref[1][r0:r1], 1e-5)
            assert ok, worst
        else:
            assert np.array_equal(res[r][1], ref[r0:r1])
