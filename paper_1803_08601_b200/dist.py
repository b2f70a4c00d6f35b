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

Two further forms:
  * NEXT-1, the all-gather of C fused into the SpMM (RowBlockSpmm.enable_fused_gather /
    execute_gather): every rank's full C lives in a CUDA IPC buffer that every other rank maps, and
    the kernels store each finished row into the local C AND into every peer's C (over NVLink on a
    multi-GPU node), so the gather overlaps the compute row by row instead of following it.
  * NEXT-3, the iterative distributed SpMM (IterativeRowBlockSpmm): Y = A X with X and Y distributed in
    the same row blocks (LOBPCG / block Lanczos / multi-RHS); each step all-gathers X
    while the diagonal block A_rr X_r is computed, then accumulates the off-diagonal block
    A_r,other X (spmm_csr_execute_ex, accumulate = 1); A_r is split once (spmm_csr_split_columns).

`local_factory` (and `split_fn`) are injectable so the host logic (partition, slicing, collectives) can
also be tested with the gloo backend on CPU; the product default is the CUDA path
(paper_1803_08601_b200.spmm).
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

    def split_columns(self, c0, c1):
        """(ro, col, val) of the entries with column in [c0, c1) (columns rebased) and of the others."""
        return split_columns_cuda(self.op.row_offsets, self.op.col_indices, self.op.values, c0, c1)

    def info(self):
        return self.op.info()

    def close(self):
        self.op.close()


def split_columns_cuda(ro, col, val, c0: int, c1: int):
    """spmm_csr_split_columns through the C ABI (device tensors in, device tensors out)."""
    from . import spmm as S
    m, nnz = ro.numel() - 1, col.numel()
    dev = ro.device
    ro_in = torch.empty(m + 1, dtype=torch.int32, device=dev)
    ro_out = torch.empty(m + 1, dtype=torch.int32, device=dev)
    col_in = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    col_out = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    val_in = torch.empty(max(nnz, 1), dtype=val.dtype, device=dev)
    val_out = torch.empty(max(nnz, 1), dtype=val.dtype, device=dev)
    st, z_in = S.spmm_csr_split_columns(
        ctypes.c_void_p(ro.data_ptr()), ctypes.c_void_p(col.data_ptr() if nnz else 0),
        ctypes.c_void_p(val.data_ptr() if nnz else 0), m, nnz, int(c0), int(c1), S._dtype_code(val),
        ctypes.c_void_p(ro_in.data_ptr()), ctypes.c_void_p(col_in.data_ptr()), ctypes.c_void_p(val_in.data_ptr()),
        ctypes.c_void_p(ro_out.data_ptr()), ctypes.c_void_p(col_out.data_ptr()), ctypes.c_void_p(val_out.data_ptr()),
        S._stream_ptr(None))
    if st != S.SPMM_OK:
        raise S.SpmmError(st, S.spmm_status_string(st))
    z_out = nnz - z_in
    return (ro_in, col_in[:z_in], val_in[:z_in]), (ro_out, col_out[:z_out], val_out[:z_out])


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory (wraps an IPC buffer as a torch tensor)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2, "strides": None}


def _tensor_at(ptr: int, shape, dtype, device):
    typestr = {torch.float32: "<f4", torch.int32: "<i4"}[dtype]
    return torch.as_tensor(_CudaArray(ptr, shape, typestr), device=device)


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

    # ---------------- NEXT-1: the C all-gather fused into the SpMM ----------------
    def enable_fused_gather(self):
        """Collective (every rank): allocate this rank's full C (m x n) as a CUDA IPC buffer, exchange
        the handles, and map every peer's full C.  Afterwards execute_gather() leaves all of C on every
        rank with no separate collective."""
        import torch.distributed as dist
        from . import spmm as S
        if self.n is None:
            raise RuntimeError("plan() first")
        if self.world - 1 > S.SPMM_MAX_PEERS:
            raise ValueError(f"fused gather supports at most {S.SPMM_MAX_PEERS + 1} ranks")
        dtype = self.val.dtype
        nbytes = max(16, self.m * self.n * 4)
        st, ptr, handle = S.spmm_ipc_alloc(nbytes)
        if st != S.SPMM_OK:
            raise S.SpmmError(st, "spmm_ipc_alloc: " + S.spmm_status_string(st))
        self._ipc_ptr = ptr
        self.C_full = _tensor_at(ptr, (self.m, self.n), dtype, self.device)
        handles = [None] * self.world
        dist.all_gather_object(handles, handle, group=self.group)
        self._peer_ptrs = []
        for i, h in enumerate(handles):
            if i == self.rank:
                continue
            st, pp = S.spmm_ipc_open(h)
            if st != S.SPMM_OK:
                raise S.SpmmError(st, f"spmm_ipc_open(rank {i}): " + S.spmm_status_string(st))
            self._peer_ptrs.append(pp)
        dist.barrier(group=self.group)
        return self.C_full

    def execute_gather(self, B, **kw):
        """C = A (x) B with every finished row stored into the local full C and into every peer's full
        C by the kernels themselves (spmm_csr_execute_ex peers); returns this rank's full C, complete
        on return (stream synchronised + barrier: every rank's stores into it have landed)."""
        import torch.distributed as dist
        if getattr(self, "C_full", None) is None:
            raise RuntimeError("enable_fused_gather() first")
        r0, r1 = self.bounds[self.rank], self.bounds[self.rank + 1]
        # every rank's earlier work on its C (reads, refills) is finished before any peer stores into it
        torch.cuda.current_stream(self.device).synchronize()
        dist.barrier(group=self.group)
        self.local.execute(B, self.C_full[r0:r1], peers=self._peer_ptrs, peer_row_offset=r0, **kw)
        torch.cuda.current_stream(self.device).synchronize()
        dist.barrier(group=self.group)
        return self.C_full

    def info(self):
        return self.local.info()

    def close(self):
        from . import spmm as S
        for pp in getattr(self, "_peer_ptrs", []):
            S.spmm_ipc_close(pp)
        self._peer_ptrs = []
        if getattr(self, "_ipc_ptr", None):
            self.C_full = None
            S.spmm_ipc_free(self._ipc_ptr)
            self._ipc_ptr = None
        self.local.close()


class IterativeRowBlockSpmm:
    """NEXT-3: Y = A (x) X for square A with X and Y row-distributed by the same
    bounds -- the iterative use of tall-skinny SpMM (LOBPCG, block Lanczos, multi-RHS),
    where B changes every iteration and so must be exchanged every iteration.

    Rank r holds the row block A_r, split once into the diagonal block A_rr (columns of its own rows,
    rebased) and the rest.  step(X_r): start the all-gather of X (async), compute Y_r = A_rr X_r
    meanwhile (it needs only local data), wait, then Y_r (+)= A_r,rest X (the off-diagonal SpMM with
    accumulate, spmm_csr_execute_ex).  Rows of C are independent, so the result equals the
    single-GPU product (fp32 up to summation order)."""

    def __init__(self, row_offsets, col_indices, values, k: int | None = None, *, group=None, mode: int = 1,
                 device=None, local_factory=None, split_fn=None):
        import torch.distributed as dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device or values.device
        self.m = row_offsets.numel() - 1
        if k is not None and int(k) != self.m:
            raise ValueError(f"iterative SpMM needs a square A (X and Y share the row blocks): m = {self.m}, k = {k}")
        self.bounds = partition_rows(row_offsets, self.world, mode)
        r0, r1 = self.bounds[self.rank], self.bounds[self.rank + 1]
        ro, col, val = slice_rows(row_offsets, col_indices, values, r0, r1)
        ro, col, val = ro.to(self.device).contiguous(), col.to(self.device).contiguous(), val.to(self.device).contiguous()
        (rd, cd, vd), (rx, cx, vx) = (split_fn or split_columns_cuda)(ro, col, val, r0, r1)
        fac = local_factory or CudaLocal
        self.m_local = r1 - r0
        self.nnz_diag, self.nnz_off = cd.numel(), cx.numel()
        self._keep = (rd, cd, vd, rx, cx, vx)
        self.diag = fac(rd, cd, vd, self.m_local)
        self.off = fac(rx, cx, vx, self.m) if self.nnz_off else None
        self.dtype = val.dtype
        self.n = None

    def plan(self, n: int, algo: str = "auto", semiring: str = "plus_times", **kw):
        self.n = n
        self.X_full = torch.empty(self.m, n, dtype=self.dtype, device=self.device)
        picks = [self.diag.plan(n, algo, semiring, **kw)]
        if self.off is not None:
            picks.append(self.off.plan(n, algo, semiring, **kw))
        return picks

    def _gather_X(self, X_local):
        """All-gather of the X row blocks into X_full; returns a waitable (or None when done)."""
        import torch.distributed as dist
        views = [self.X_full[self.bounds[i]:self.bounds[i + 1]] for i in range(self.world)]
        if _backend(self.group) == "nccl":
            return dist.all_gather(views, X_local.contiguous(), group=self.group, async_op=True)
        views[self.rank].copy_(X_local)
        for i in range(self.world):
            if views[i].numel():
                _bcast(views[i], i, self.group)
        return None

    def step(self, X_local, Y_local=None):
        """Y_r = A_r (x) X (X given as this rank's rows X_r); returns Y_r."""
        if Y_local is None:
            Y_local = torch.empty(self.m_local, self.n, dtype=self.dtype, device=self.device)
        work = self._gather_X(X_local)           # exchange of X, in flight ...
        self.diag.execute(X_local, Y_local)      # ... while the diagonal block is computed
        if work is not None:
            work.wait()
        if self.off is not None:
            self.off.execute(self.X_full, Y_local, accumulate=True)
        return Y_local

    def close(self):
        self.diag.close()
        if self.off is not None:
            self.off.close()


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
