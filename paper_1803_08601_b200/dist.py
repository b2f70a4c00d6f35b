"""Multi-GPU CSR SpMM (north_star): one process per GPU (torch.distributed, NCCL on
B200), A split into 1-D row blocks, B replicated by a broadcast from rank 0, each rank writes its own
C rows; an optional all-gather of C.  The paper itself is single-GPU; rows of C are
independent, so the only exchange steps are the B broadcast and the optional C gather.

The row partition is computed by the C ABI (spmm_partition_rows, host code in libspmm.so):
  mode 0  nnz-balanced: bounds[p] = lower_bound(ro, p*nnz/P)
  mode 1  merge-path balanced (rows + nnz), which also charges each row's C write
A row is never split across ranks.

`local_spmm` is injectable so the host logic (partition, slicing, collectives) can be tested with the
gloo backend on CPU; the product default is the CUDA path (paper_1803_08601_b200.spmm).
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


def _cuda_local_spmm(ro, col, val, B, k, n, algo="auto", semiring="plus_times"):
    from . import spmm as S
    op = S.CsrSpmm(ro, col, val, k)
    try:
        op.plan(n, algo, semiring)
        return op.execute(B)
    finally:
        op.close()


def distributed_spmm(row_offsets, col_indices, values, B_root, k: int, n: int, *, group=None, mode: int = 1,
                     gather: bool = False, algo: str = "auto", semiring: str = "plus_times", local_spmm=None,
                     device=None):
    """C = A*B over all ranks of `group`.

    Every rank passes the full CSR (or at least its offsets + its own rows; only rows of its block are
    read).  B_root is the k x n B on rank 0 (ignored elsewhere).  Returns (C_local, bounds) or, with
    gather=True, (C_full, bounds) assembled by an all-gather of padded row blocks.
    """
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    device = device or (values.device if values is not None else torch.device("cpu"))
    bounds = partition_rows(row_offsets, world, mode)
    r0, r1 = bounds[rank], bounds[rank + 1]
    ro, col, val = slice_rows(row_offsets, col_indices, values, r0, r1)
    ro, col, val = ro.to(device), col.to(device), val.to(device)
    # exchange step 1: replicate B (broadcast from rank 0)
    dtype = values.dtype
    B = B_root.to(device).contiguous() if rank == 0 else torch.empty(k, n, dtype=dtype, device=device)
    dist.broadcast(B, src=0, group=group)
    fn = local_spmm or _cuda_local_spmm
    C_local = fn(ro, col, val, B, k, n, algo=algo, semiring=semiring)
    if not gather:
        return C_local, bounds
    # exchange step 2 (optional): all-gather C row blocks, padded to the largest block
    rows = [bounds[i + 1] - bounds[i] for i in range(world)]
    mx = max(rows) if rows else 0
    pad = torch.zeros(mx, n, dtype=C_local.dtype, device=device)
    pad[:C_local.shape[0]] = C_local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    C = torch.cat([parts[i][:rows[i]] for i in range(world)], 0)
    return C, bounds
