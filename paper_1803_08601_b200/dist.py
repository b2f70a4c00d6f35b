"""Multi-GPU CSR SpMM (north_star): one process per GPU (torch.distributed, NCCL on
B200), A split into 1-D row blocks, B replicated by a broadcast from rank 0, each rank writes its own
C rows; an optional all-gather of C.  The paper itself is single-GPU; rows of C are
independent, so the only exchange steps are the B broadcast and the optional C gather.

This module is the ONE multi-GPU code path: `bench.py` and the tests drive `RowBlockSpmm`
(partition -> slice -> broadcast B -> local execute -> gather C); `distributed_spmm` is the one-shot
form of the same object.

The row partition is computed by the C ABI (spmm_partition_rows, host code in libspmm.so):
  mode 0  nnz-balanced: bounds[p] = lower_bound(ro, p*nnz/P)                      (north_star)
  mode 1  merge-path balanced (rows + nnz), which also charges each row's C write
A row is never split across ranks.

The C gather moves exactly the rows each rank owns (no padding to the largest block): NCCL's
all_gather over row-block views of uneven sizes runs as grouped broadcasts; on gloo
the same broadcasts are issued one by one.

`local_factory` is injectable so the host logic (partition, slicing, collectives) can also be tested
with the gloo backend on CPU; the product default is the CUDA path (paper_1803_08601_b200.spmm).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch


def partition_rows(row_offsets, parts: int, mode: int = 1) -> list[int]:
    """Row bounds (parts+1 ints) via the C ABI's spmm_partition_rows (host-only, no GPU needed)."""
    from . import spmm as S
    ro = np.ascontiguousarray(row_offsets.cpu().numpy() if hasattr(row_offsets, "cpu") else row_offsets,
                              dtype=np.int32)
    bounds = (ctypes.c_int64 * (parts + 1))()
    st = S.spmm_partition_rows(ro.ctypes.data, len(ro) - 1, parts, mode, bounds)
    if st != S.SPMM_OK:
        raise S.SpmmError(st, S.spmm_status_string(st))
    return list(bounds)


def slice_rows(row_offsets, col_indices, values, r0: int, r1: int):
    """Rows [r0, r1) as a standalone CSR with rebased offsets (views for col/values)."""
    ro = row_offsets[r0:r1 + 1]
    z0, z1 = int(ro[0]), int(ro[-1])
    return (ro - z0).contiguous(), col_indices[z0:z1], values[z0:z1]


class CudaLocal:
    """The per-rank SpMM: the CUDA path through the C ABI (CsrSpmm), planned once, executed often."""

    def __init__(self, ro, col, val, k):
        from . import spmm as S
        self.op = S.CsrSpmm(ro, col, val, k)

    def plan(self, n, algo="auto", semiring="plus_times", **kw):
        return self.op.plan(n, algo, semiring, **kw)

    def execute(self, B, C=None, **kw):
        return self.op.execute(B, C, **kw)

    def info(self):
        return self.op.info()

    def close(self):
        self.op.close()


def _backend(group):
    import torch.distributed as dist
    return dist.get_backend(group)


def _bcast(t, src: int, group):
    """Broadcast `t` in place; on gloo, device tensors are staged through host memory."""
    import torch.distributed as dist
    if t.is_cuda and _backend(group) != "nccl":
        h = t.cpu()
        dist.broadcast(h, src=src, group=group)
        t.copy_(h)
    else:
        dist.broadcast(t, src=src, group=group)


class RowBlockSpmm:
    """C = A (x) B over all ranks of `group` with A in 1-D row blocks.

    Every rank passes the full CSR offsets (only its own rows' col/val are read; they may live on any
    device and are copied to `device`).  `bounds` may be given (e.g. weak scaling, where each rank
    already holds only its block: pass row_offsets/col/val of the block and bounds=None, local=True).
    """

    def __init__(self, row_offsets, col_indices, values, k: int, *, group=None, mode: int = 1, device=None,
                 local: bool = False, local_factory=None):
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device or (values.device if values is not None else torch.device("cpu"))
        self.k = int(k)
        if local:
            # this rank's block is given; learn every rank's row count (for the C gather)
            m_loc = torch.tensor([row_offsets.numel() - 1], dtype=torch.int64, device=self._comm_device())
            rows = [torch.empty_like(m_loc) for _ in range(self.world)]
            dist.all_gather(rows, m_loc, group=group)
            counts = [int(r.item()) for r in rows]
            self.bounds = [0]
            for c in counts:
                self.bounds.append(self.bounds[-1] + c)
            ro, col, val = row_offsets, col_indices, values
        else:
            self.bounds = partition_rows(row_offsets, self.world, mode)
            r0, r1 = self.bounds[self.rank], self.bounds[self.rank + 1]
            ro, col, val = slice_rows(row_offsets, col_indices, values, r0, r1)
        self.ro = ro.to(self.device).contiguous()
        self.col = col.to(self.device).contiguous()
        self.val = val.to(self.device).contiguous()
        self.m_local = self.ro.numel() - 1
        self.m = self.bounds[-1]
        self.local = (local_factory or CudaLocal)(self.ro, self.col, self.val, self.k)
        self.n = None

    def _comm_device(self):
        return self.device if _backend(self.group) == "nccl" else torch.device("cpu")

    def plan(self, n: int, algo: str = "auto", semiring: str = "plus_times", **kw) -> str:
        self.n = n
        return self.local.plan(n, algo, semiring, **kw)

    def broadcast_B(self, B_root=None, out=None):
        """Exchange step 1: replicate B (k x n) from rank 0 to every rank; returns this rank's copy."""
        import torch.distributed as dist
        dtype = self.val.dtype
        if out is None:
            out = torch.empty(self.k, self.n, dtype=dtype, device=self.device)
        if self.rank == 0 and B_root is not None and B_root.data_ptr() != out.data_ptr():
            out.copy_(B_root)
        _bcast(out, 0, self.group)
        return out

    def execute(self, B, C_local=None, **kw):
        """Local step: this rank's C rows = A_block (x) B (B replicated, k x n)."""
        if C_local is None:
            C_local = torch.empty(self.m_local, self.n, dtype=B.dtype, device=self.device)
        return self.local.execute(B, C_local, **kw)

    def gather_C(self, C_local, out=None):
        """Exchange step 2 (optional): every rank receives all of C (m x n).  Each rank's rows are
        broadcast from their owner into a row-block view of `out`: exactly m*n elements move, no
        padding (uneven blocks)."""
        import torch.distributed as dist
        if out is None:
            out = torch.empty(self.m, self.n, dtype=C_local.dtype, device=self.device)
        views = [out[self.bounds[i]:self.bounds[i + 1]] for i in range(self.world)]
        if _backend(self.group) == "nccl":
            # uneven output sizes: ProcessGroupNCCL runs this as grouped (coalesced) broadcasts
            dist.all_gather(views, C_local.contiguous(), group=self.group)
        else:
            views[self.rank].copy_(C_local)
            for i in range(self.world):
                if views[i].numel():
                    _bcast(views[i], i, self.group)
        return out

    def info(self):
        return self.local.info()

    def close(self):
        self.local.close()


def distributed_spmm(row_offsets, col_indices, values, B_root, k: int, n: int, *, group=None, mode: int = 1,
                     gather: bool = False, algo: str = "auto", semiring: str = "plus_times", local_factory=None,
                     device=None):
    """One-shot C = A*B over all ranks of `group` (RowBlockSpmm: partition, broadcast B, execute,
    optional gather).  B_root is the k x n B on rank 0 (ignored elsewhere).  Returns (C_local, bounds)
    or, with gather=True, (C_full, bounds)."""
    op = RowBlockSpmm(row_offsets, col_indices, values, k, group=group, mode=mode, device=device,
                      local_factory=local_factory)
    try:
        op.plan(n, algo, semiring)
        B = op.broadcast_B(B_root if op.rank == 0 else None)
        C_local = op.execute(B)
        if not gather:
            return C_local, op.bounds
        return op.gather_C(C_local), op.bounds
    finally:
        op.close()
