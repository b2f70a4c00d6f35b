"""Thin ctypes binding of libspmm.so (include/spmm.h).  Argument marshalling only: every step of the
SpMM path runs in the CUDA kernels of csrc/.  There is no CPU fallback: if the in-tree library is
missing or no CUDA device is present, calls raise.

Low-level functions carry the C names (spmm_csr_create, spmm_csr_plan, spmm_csr_plan_ex,
spmm_csr_execute, spmm_csr_destroy, spmm_csr_get_plan_info, spmm_status_string, spmm_csr_last_error,
spmm_merge_num_ctas, spmm_merge_partition, spmm_partition_rows, spmm_abi_version).  `CsrSpmm` wraps a
handle around torch CUDA tensors (PyTorch is used for device memory and streams only).
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_char_p, c_double, c_int32, c_int64, c_size_t, c_uint32, c_void_p

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libspmm.so")

# enums (include/spmm.h)
SPMM_OK = 0
SPMM_ERR_NULL_POINTER = 1
SPMM_ERR_INVALID_ARG = 2
SPMM_ERR_INVALID_CSR = 3
SPMM_ERR_NOT_PLANNED = 4
SPMM_ERR_WORKSPACE_TOO_SMALL = 5
SPMM_ERR_UNSUPPORTED = 6
SPMM_ERR_CUDA = 7
SPMM_ALGO_AUTO, SPMM_ALGO_ROWSPLIT, SPMM_ALGO_MERGE, SPMM_ALGO_TILED = 0, 1, 2, 3
SPMM_F32, SPMM_I32 = 0, 1
SPMM_PLUS_TIMES, SPMM_MIN_PLUS = 0, 1
SPMM_FLAG_VALIDATE = 1
SPMM_POLICY_AUTO, SPMM_POLICY_PAPER = 0, 1
SPMM_PARTITION_MERGE_PATH, SPMM_PARTITION_NONZERO_SPLIT = 0, 1
SPMM_MERGE_WORKER_AUTO, SPMM_MERGE_WORKER_WARP, SPMM_MERGE_WORKER_FOLDED = 0, 1, 2
MERGE_WORKERS = {"auto": SPMM_MERGE_WORKER_AUTO, "warp": SPMM_MERGE_WORKER_WARP, "folded": SPMM_MERGE_WORKER_FOLDED}

ALGOS = {"auto": SPMM_ALGO_AUTO, "rowsplit": SPMM_ALGO_ROWSPLIT, "merge": SPMM_ALGO_MERGE, "tiled": SPMM_ALGO_TILED}
ALGO_NAMES = {v: k for k, v in ALGOS.items()}
SEMIRINGS = {"plus_times": SPMM_PLUS_TIMES, "min_plus": SPMM_MIN_PLUS}

EXPORTED = ("spmm_csr_create", "spmm_csr_plan", "spmm_csr_plan_ex", "spmm_csr_execute", "spmm_csr_execute_ex",
            "spmm_csr_destroy", "spmm_csr_get_plan_info", "spmm_status_string", "spmm_csr_last_error",
            "spmm_abi_version", "spmm_merge_num_ctas", "spmm_merge_partition", "spmm_partition_rows",
            "spmm_csr_set_timing_events", "spmm_csr_split_columns", "spmm_ipc_alloc", "spmm_ipc_free",
            "spmm_ipc_open", "spmm_ipc_close", "spmm_csr_multiply_host")
SPMM_HOST_SYNC = 1
SPMM_MAX_PEERS = 7
SPMM_IPC_HANDLE_BYTES = 64


class spmm_plan_opts(Structure):
    _fields_ = [("policy", c_int32), ("partition", c_int32), ("items_per_cta", c_int32),
                ("merge_worker", c_int32), ("tasks_per_warp", c_int32), ("reserved", c_int32 * 3)]


class spmm_plan_info(Structure):
    _fields_ = [("m", c_int64), ("k", c_int64), ("nnz", c_int64), ("n", c_int32), ("chosen", c_int32),
                ("semiring", c_int32), ("dtype", c_int32), ("policy", c_int32), ("partition", c_int32),
                ("mean_row_length", c_double), ("max_row_length", c_int64), ("threshold", c_double),
                ("num_ctas", c_int32), ("items_per_cta", c_int32), ("launches_per_execute", c_int32),
                ("compute_launch", c_int32), ("workspace_bytes", c_size_t), ("b_staging", c_int32),
                ("rows_per_tile", c_int32), ("bspan_compact", c_double), ("merge_worker_lanes", c_int32),
                ("tasks_per_warp", c_int32)]


class spmm_exec_opts(Structure):
    _fields_ = [("accumulate", c_int32), ("num_peers", c_int32), ("peer_row_offset", c_int64), ("peer_ldc", c_int64),
                ("peer_C", c_void_p * SPMM_MAX_PEERS), ("reserved", c_int32 * 4)]


class SpmmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} (status {status})")
        self.status = status


_lib = None


def load(path: str | None = None):
    """Load the in-tree libspmm.so (built by paper_1803_08601_b200.build / __graft_entry__.build()).
    SPMM_LIB=<path> selects an alternative in-tree build (tuning experiments only)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("SPMM_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"libspmm.so not found at {path}: run `python -m paper_1803_08601_b200.build` "
                           "(the CUDA path has no fallback)")
    lib = ctypes.CDLL(path)
    lib.spmm_csr_create.argtypes = [POINTER(c_void_p), c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                    c_int32, c_uint32, c_void_p]
    lib.spmm_csr_plan.argtypes = [c_void_p, c_int32, c_int32, c_int32, c_double, c_void_p, POINTER(c_size_t),
                                  POINTER(c_int32)]
    lib.spmm_csr_plan_ex.argtypes = [c_void_p, c_int32, c_int32, c_int32, c_double, POINTER(spmm_plan_opts),
                                     c_void_p, POINTER(c_size_t), POINTER(c_int32)]
    lib.spmm_csr_execute.argtypes = [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_int32, c_void_p, c_size_t,
                                     c_void_p]
    lib.spmm_csr_execute_ex.argtypes = [c_void_p, c_void_p, c_int64, c_void_p, c_int64, c_int32, c_void_p, c_size_t,
                                        POINTER(spmm_exec_opts), c_void_p]
    lib.spmm_csr_split_columns.argtypes = [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_int32, c_int32, c_int32,
                                           c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                           POINTER(c_int64), c_void_p]
    lib.spmm_csr_multiply_host.argtypes = [c_int64, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_int32, c_void_p,
                                           c_int64, c_void_p, c_int64, c_int32, c_int32, c_int32, c_uint32, c_void_p]
    lib.spmm_ipc_alloc.argtypes = [c_size_t, POINTER(c_void_p), c_void_p]
    lib.spmm_ipc_free.argtypes = [c_void_p]
    lib.spmm_ipc_open.argtypes = [c_void_p, POINTER(c_void_p)]
    lib.spmm_ipc_close.argtypes = [c_void_p]
    lib.spmm_csr_destroy.argtypes = [c_void_p]
    lib.spmm_csr_get_plan_info.argtypes = [c_void_p, POINTER(spmm_plan_info)]
    lib.spmm_status_string.argtypes = [c_int32]
    lib.spmm_status_string.restype = c_char_p
    lib.spmm_csr_last_error.argtypes = [c_void_p]
    lib.spmm_csr_last_error.restype = c_char_p
    lib.spmm_abi_version.restype = c_int32
    lib.spmm_merge_num_ctas.argtypes = [c_int64, c_int64, c_int32, c_int32]
    lib.spmm_merge_num_ctas.restype = c_int64
    lib.spmm_merge_partition.argtypes = [c_void_p, c_int64, c_int64, c_int32, c_int32, c_int64, c_void_p, c_void_p]
    lib.spmm_partition_rows.argtypes = [c_void_p, c_int64, c_int32, c_int32, POINTER(c_int64)]
    lib.spmm_csr_set_timing_events.argtypes = [c_void_p, POINTER(c_void_p), c_int32]
    for name in EXPORTED:
        if name not in ("spmm_status_string", "spmm_csr_last_error", "spmm_abi_version", "spmm_merge_num_ctas"):
            getattr(lib, name).restype = c_int32
    _lib = lib
    return lib


# ------------------------------------------------------------------------------------------------
# C-named wrappers (plain ints / pointers in, status out)
# ------------------------------------------------------------------------------------------------
def spmm_status_string(s: int) -> str:
    return load().spmm_status_string(s).decode()


def spmm_abi_version() -> int:
    return int(load().spmm_abi_version())


def spmm_csr_last_error(h) -> str:
    return load().spmm_csr_last_error(h).decode()


def _check(status: int, h=None):
    if status != SPMM_OK:
        detail = spmm_csr_last_error(h) if h else ""
        raise SpmmError(status, f"{spmm_status_string(status)} {detail}".strip())


def spmm_csr_create(m, k, nnz, row_offsets_ptr, col_indices_ptr, values_ptr, dtype, flags=0, stream=None):
    h = c_void_p()
    st = load().spmm_csr_create(ctypes.byref(h), m, k, nnz, row_offsets_ptr, col_indices_ptr, values_ptr, dtype,
                                flags, stream)
    return st, h


def spmm_csr_plan(h, n, algo, semiring, threshold=0.0, stream=None):
    ws = c_size_t(0)
    chosen = c_int32(0)
    st = load().spmm_csr_plan(h, n, algo, semiring, threshold, stream, ctypes.byref(ws), ctypes.byref(chosen))
    return st, ws.value, chosen.value


def spmm_csr_plan_ex(h, n, algo, semiring, threshold=0.0, policy=0, partition=0, items_per_cta=0, stream=None,
                     merge_worker=0, tasks_per_warp=0):
    o = spmm_plan_opts(policy, partition, items_per_cta, merge_worker, tasks_per_warp)
    ws = c_size_t(0)
    chosen = c_int32(0)
    st = load().spmm_csr_plan_ex(h, n, algo, semiring, threshold, ctypes.byref(o), stream, ctypes.byref(ws),
                                 ctypes.byref(chosen))
    return st, ws.value, chosen.value


def spmm_csr_execute(h, B_ptr, ldb, C_ptr, ldc, n, ws_ptr, ws_bytes, stream=None) -> int:
    return load().spmm_csr_execute(h, B_ptr, ldb, C_ptr, ldc, n, ws_ptr, ws_bytes, stream)


def spmm_csr_execute_ex(h, B_ptr, ldb, C_ptr, ldc, n, ws_ptr, ws_bytes, opts, stream=None) -> int:
    return load().spmm_csr_execute_ex(h, B_ptr, ldb, C_ptr, ldc, n, ws_ptr, ws_bytes,
                                      ctypes.byref(opts) if opts is not None else None, stream)


def spmm_csr_split_columns(ro_ptr, col_ptr, val_ptr, m, nnz, c0, c1, dtype, ro_in, col_in, val_in, ro_out, col_out,
                           val_out, stream=None):
    nnz_in = c_int64(0)
    st = load().spmm_csr_split_columns(ro_ptr, col_ptr, val_ptr, m, nnz, c0, c1, dtype, ro_in, col_in, val_in, ro_out,
                                       col_out, val_out, ctypes.byref(nnz_in), stream)
    return st, nnz_in.value


def spmm_csr_multiply_host(m, k, nnz, ro_ptr, col_ptr, val_ptr, dtype, B_ptr, ldb, C_ptr, ldc, n, algo, semiring,
                           flags=0, stream=None) -> int:
    return load().spmm_csr_multiply_host(m, k, nnz, ro_ptr, col_ptr, val_ptr, dtype, B_ptr, ldb, C_ptr, ldc, n, algo,
                                         semiring, flags, stream)


def multiply_host(row_offsets, col_indices, values, k, B, C=None, algo="auto", semiring="plus_times", stream=None,
                  sync=True):
    """C = A (x) B with every array in (preferably pinned) HOST memory, through spmm_csr_multiply_host:
    the library copies in, plans, executes and copies C back on `stream`."""
    import torch
    for t in (row_offsets, col_indices, values, B):
        if t.is_cuda or not t.is_contiguous():
            raise ValueError("multiply_host takes contiguous host tensors")
    m, nnz, n = row_offsets.numel() - 1, col_indices.numel(), B.shape[1]
    if C is None:
        C = torch.empty(m, n, dtype=B.dtype, pin_memory=True)
    st = spmm_csr_multiply_host(m, k, nnz, c_void_p(row_offsets.data_ptr()), c_void_p(col_indices.data_ptr()),
                                c_void_p(values.data_ptr()), _dtype_code(values), c_void_p(B.data_ptr()), B.stride(0),
                                c_void_p(C.data_ptr()), C.stride(0), n, ALGOS[algo], SEMIRINGS[semiring],
                                SPMM_HOST_SYNC if sync else 0, _stream_ptr(stream))
    _check(st)
    return C


def spmm_ipc_alloc(nbytes):
    ptr = c_void_p()
    handle = ctypes.create_string_buffer(SPMM_IPC_HANDLE_BYTES)
    st = load().spmm_ipc_alloc(nbytes, ctypes.byref(ptr), handle)
    return st, ptr.value, handle.raw


def spmm_ipc_free(ptr) -> int:
    return load().spmm_ipc_free(ptr)


def spmm_ipc_open(handle: bytes):
    ptr = c_void_p()
    buf = ctypes.create_string_buffer(bytes(handle), SPMM_IPC_HANDLE_BYTES)
    st = load().spmm_ipc_open(buf, ctypes.byref(ptr))
    return st, ptr.value


def spmm_ipc_close(ptr) -> int:
    return load().spmm_ipc_close(ptr)


def spmm_csr_destroy(h) -> int:
    return load().spmm_csr_destroy(h)


def spmm_csr_get_plan_info(h):
    info = spmm_plan_info()
    st = load().spmm_csr_get_plan_info(h, ctypes.byref(info))
    return st, info


def spmm_csr_set_timing_events(h, event_handles) -> int:
    arr = (c_void_p * max(1, len(event_handles)))(*[c_void_p(e) for e in event_handles])
    return load().spmm_csr_set_timing_events(h, arr, len(event_handles))


def spmm_merge_num_ctas(m, nnz, items_per_cta, partition) -> int:
    return int(load().spmm_merge_num_ctas(m, nnz, items_per_cta, partition))


def spmm_merge_partition(ro_ptr, m, nnz, items_per_cta, partition, num_ctas, states_ptr, stream=None) -> int:
    return load().spmm_merge_partition(ro_ptr, m, nnz, items_per_cta, partition, num_ctas, states_ptr, stream)


def spmm_partition_rows(host_ro_ptr, m, parts, mode, bounds_array) -> int:
    return load().spmm_partition_rows(host_ro_ptr, m, parts, mode, bounds_array)


# ------------------------------------------------------------------------------------------------
# torch-facing convenience layer
# ------------------------------------------------------------------------------------------------
def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return c_void_p(stream.cuda_stream)


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float32:
        return SPMM_F32
    if t.dtype == torch.int32:
        return SPMM_I32
    raise TypeError(f"values must be float32 or int32, got {t.dtype}")


class CsrSpmm:
    """C = A (x) B for a CSR matrix A held in torch CUDA tensors (borrowed, never copied).

    One workspace per plan: executes of one CsrSpmm must not overlap on different streams (they share
    the merge kernel's partition / carry arrays and the row-split tile queue).  Use one CsrSpmm per
    stream for concurrent executes."""

    def __init__(self, row_offsets, col_indices, values, k: int, validate: bool = False, stream=None):
        import torch
        for t, name in ((row_offsets, "row_offsets"), (col_indices, "col_indices"), (values, "values")):
            if not t.is_cuda:
                raise ValueError(f"{name} must be a CUDA tensor (no CPU path)")
            if not t.is_contiguous():
                raise ValueError(f"{name} must be contiguous")
        if row_offsets.dtype != torch.int32 or col_indices.dtype != torch.int32:
            raise TypeError("row_offsets and col_indices must be int32")
        self.row_offsets, self.col_indices, self.values = row_offsets, col_indices, values
        self.m = row_offsets.numel() - 1
        self.k = int(k)
        self.nnz = col_indices.numel()
        self.dtype = _dtype_code(values)
        self._h = None
        st, h = spmm_csr_create(self.m, self.k, self.nnz, c_void_p(row_offsets.data_ptr()),
                                c_void_p(col_indices.data_ptr() if self.nnz else 0),
                                c_void_p(values.data_ptr() if self.nnz else 0), self.dtype,
                                SPMM_FLAG_VALIDATE if validate else 0, _stream_ptr(stream))
        _check(st)
        self._h = h
        self.n = None
        self.workspace = None
        self.chosen = None

    def plan(self, n: int, algo: str = "auto", semiring: str = "plus_times", threshold: float = 0.0,
             policy: str = "auto", partition: str = "merge_path", items_per_cta: int = 0, stream=None,
             merge_worker: str = "auto", tasks_per_warp: int = 0) -> str:
        import torch
        st, ws, chosen = spmm_csr_plan_ex(self._h, n, ALGOS[algo], SEMIRINGS[semiring], threshold,
                                          {"auto": SPMM_POLICY_AUTO, "paper": SPMM_POLICY_PAPER}[policy],
                                          {"merge_path": SPMM_PARTITION_MERGE_PATH,
                                           "nonzero_split": SPMM_PARTITION_NONZERO_SPLIT}[partition],
                                          items_per_cta, _stream_ptr(stream), MERGE_WORKERS[merge_worker], tasks_per_warp)
        _check(st, self._h)
        self.n = n
        self.workspace = torch.empty(max(ws, 16), dtype=torch.uint8, device=self.row_offsets.device)
        self.ws_bytes = ws
        self.chosen = ALGO_NAMES[chosen]
        return self.chosen

    def info(self) -> dict:
        st, inf = spmm_csr_get_plan_info(self._h)
        _check(st, self._h)
        return {f: getattr(inf, f) for f, _ in spmm_plan_info._fields_}

    def execute(self, B, C=None, stream=None, accumulate: bool = False, peers=None, peer_row_offset: int = 0):
        """C[:m, :n] = A (x) B.  B: k' x ldb row-major CUDA tensor with k' >= k rows and >= n columns
        (only columns [0, n) are read); C (optional): m x >= n row-major, overwritten in [0, n).
        accumulate=True: C = C (+) A (x) B.  peers: device pointers (ints) of up to 7 other copies of
        C with the same leading dimension; every finished row r is also stored at row
        r + peer_row_offset of each (spmm_csr_execute_ex)."""
        import torch
        if self.n is None:
            raise RuntimeError("plan() first")
        dev = self.row_offsets.device
        if not B.is_cuda or B.dim() != 2 or B.stride(1) != 1:
            raise ValueError("B must be a 2-D CUDA tensor with unit column stride (row-major)")
        if B.device != dev:
            raise ValueError(f"B is on {B.device}, A on {dev}")
        if B.dtype != self.values.dtype:
            raise TypeError("B dtype must match values")
        if B.shape[0] < self.k or B.shape[1] < self.n:
            raise ValueError(f"B is {tuple(B.shape)}, needs at least {self.k} x {self.n}")
        if C is None:
            C = torch.empty(self.m, self.n, dtype=B.dtype, device=dev)
        if C.dim() != 2 or C.stride(1) != 1 or C.dtype != B.dtype:
            raise ValueError("C must be a 2-D row-major tensor of B's dtype")
        if C.device != dev:
            raise ValueError(f"C is on {C.device}, A on {dev}")
        if C.shape[0] != self.m or C.shape[1] < self.n:
            raise ValueError(f"C is {tuple(C.shape)}, needs {self.m} rows and at least {self.n} columns")
        ldb = B.stride(0) if B.shape[0] > 1 else max(B.shape[1], self.n)
        ldc = C.stride(0) if C.shape[0] > 1 else max(C.shape[1], self.n)
        if not accumulate and not peers:
            st = spmm_csr_execute(self._h, c_void_p(B.data_ptr()), ldb, c_void_p(C.data_ptr()), ldc, self.n,
                                  c_void_p(self.workspace.data_ptr()), self.workspace.numel(), _stream_ptr(stream))
        else:
            peers = list(peers or [])
            if len(peers) > SPMM_MAX_PEERS:
                raise ValueError(f"at most {SPMM_MAX_PEERS} peers")
            o = spmm_exec_opts()
            o.accumulate = 1 if accumulate else 0
            o.num_peers = len(peers)
            o.peer_row_offset = peer_row_offset
            o.peer_ldc = ldc
            for i, p in enumerate(peers):
                o.peer_C[i] = p
            st = spmm_csr_execute_ex(self._h, c_void_p(B.data_ptr()), ldb, c_void_p(C.data_ptr()), ldc, self.n,
                                     c_void_p(self.workspace.data_ptr()), self.workspace.numel(), o,
                                     _stream_ptr(stream))
        _check(st, self._h)
        return C

    def set_timing_events(self, events):
        """events: list of torch.cuda.Event(enable_timing=True); see spmm_csr_set_timing_events.
        torch creates the underlying cudaEvent_t lazily: record each event once before passing it."""
        self._events = list(events)  # keep alive
        if any(e.cuda_event == 0 for e in self._events):
            raise ValueError("torch.cuda.Event not created yet: call .record() once first")
        _check(spmm_csr_set_timing_events(self._h, [e.cuda_event for e in self._events]), self._h)

    def close(self):
        if self._h is not None:
            spmm_csr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def spmm(row_offsets, col_indices, values, B, k=None, algo="auto", semiring="plus_times", **plan_kw):
    """One-shot C = A (x) B (creates, plans, executes, destroys)."""
    k = B.shape[0] if k is None else k
    op = CsrSpmm(row_offsets, col_indices, values, k)
    try:
        op.plan(B.shape[1], algo, semiring, **plan_kw)
        return op.execute(B)
    finally:
        op.close()
