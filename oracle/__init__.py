"""oracle -- TEST INFRASTRUCTURE ONLY (plain CPU oracle for arXiv 1803.08601's CSR SpMM).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may import
this package.  It never imports the product package (paper_1803_08601_b200) and the product never
imports it; the only code both sides use is the seeded input generator module
paper_1803_08601_b200/synth.py, which holds none of the method's arithmetic.

Functions and the passages they follow:
  spmm(...)              C = A*B, the definition (§1; CSR PAPER.md:35 §2.2; row-major B/C
                         PAPER.md:37,103), in the four semiring/dtype combinations (PAPER.md:13 GrB_mxm).
                         See spmm_oracle.c for the exact arithmetic of each.
  merge_path_walk(...)   brute-force walk of the merge path (§4(2b), Fig. 2(c)).
  nonzero_split(...)     Baxter's 1-D nonzero split start rows (§4(2a)).
  heuristic(...)         §5.4 rule: merge-based iff mean row length d = nnz/m < 9.35,
                         reading "d = nnz/n" as nnz/m per the prose (SURVEY.md §8(c) ambiguity 1/2).
Parity pins for all of these live in tests/test_oracle.py (-m "not gpu").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spmm_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

PAPER_THRESHOLD = 9.35


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc -O2 -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                               "-std=c11", "-o", _LIB_PATH, _SRC, "-lm"])
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        for name in ("oracle_spmm_f32_plus_times", "oracle_spmm_i32_plus_times",
                     "oracle_spmm_f32_min_plus", "oracle_spmm_i32_min_plus",
                     "oracle_merge_path_walk", "oracle_nonzero_split"):
            getattr(_lib, name).restype = ctypes.c_int
    return _lib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _np(x, dtype):
    """Accept torch tensors or numpy arrays; return a C-contiguous numpy array of dtype."""
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(x), dtype=dtype)


def set_threads(n: int) -> None:
    os.environ["OMP_NUM_THREADS"] = str(n)


def spmm(kind: str, m: int, k: int, n: int, row_offsets, col_indices, values, B, ldb: int | None = None,
         rows=None):
    """C = A*B per SURVEY.md §8(c).  `B` is k x ldb row-major (only columns [0,n) are read).

    Returns (C, bound) for kind == 'f32_plus_times' (both float64, nrows x n), else C alone
    (int32 / float32).  rows: optional int64 list of row ids to compute (sampled parity); C row r then
    holds A's row rows[r]."""
    lib = _load()
    ro = _np(row_offsets, np.int32)
    ci = _np(col_indices, np.int32)
    Bn = _np(B, np.float32 if kind.startswith("f32") else np.int32)
    if ldb is None:
        ldb = Bn.shape[1] if Bn.ndim == 2 else n
    Bn = Bn.reshape(-1)
    assert ro.shape[0] == m + 1
    rws = None if rows is None else _np(rows, np.int64)
    nrows = m if rws is None else rws.shape[0]
    args_head = (ctypes.c_int64(m), ctypes.c_int64(k), ctypes.c_int64(n), _p(ro), _p(ci))
    tail_rows = (_p(rws), ctypes.c_int64(nrows))
    if kind == "f32_plus_times":
        v = _np(values, np.float32)
        C = np.zeros((nrows, n), np.float64)
        bound = np.zeros((nrows, n), np.float64)
        rc = lib.oracle_spmm_f32_plus_times(*args_head, _p(v), _p(Bn), ctypes.c_int64(ldb), *tail_rows,
                                            _p(C), _p(bound))
        assert rc == 0
        return C, bound
    if kind == "i32_plus_times":
        v = _np(values, np.int32)
        C = np.zeros((nrows, n), np.int32)
        rc = lib.oracle_spmm_i32_plus_times(*args_head, _p(v), _p(Bn), ctypes.c_int64(ldb), *tail_rows, _p(C))
    elif kind == "f32_min_plus":
        v = _np(values, np.float32)
        C = np.zeros((nrows, n), np.float32)
        rc = lib.oracle_spmm_f32_min_plus(*args_head, _p(v), _p(Bn), ctypes.c_int64(ldb), *tail_rows, _p(C))
    elif kind == "i32_min_plus":
        v = _np(values, np.int32)
        C = np.zeros((nrows, n), np.int32)
        rc = lib.oracle_spmm_i32_min_plus(*args_head, _p(v), _p(Bn), ctypes.c_int64(ldb), *tail_rows, _p(C))
    else:
        raise ValueError(kind)
    assert rc == 0
    return C


def merge_path_walk(row_offsets, diags):
    """States (i, j) reached after each diagonal d in `diags` (ascending) on the merge path."""
    lib = _load()
    ro = _np(row_offsets, np.int32)
    m = ro.shape[0] - 1
    nnz = int(ro[-1])
    d = _np(diags, np.int64)
    oi = np.zeros(d.shape[0], np.int64)
    oj = np.zeros(d.shape[0], np.int64)
    rc = lib.oracle_merge_path_walk(_p(ro), ctypes.c_int64(m), ctypes.c_int64(nnz), _p(d),
                                    ctypes.c_int64(d.shape[0]), _p(oi), _p(oj))
    assert rc == 0, "diagonals must be ascending and within [0, m+nnz]"
    return oi, oj


def nonzero_split(row_offsets, G: int, nblocks: int):
    """Start row of each of `nblocks` blocks of G nonzeros (Baxter's 1-D split)."""
    lib = _load()
    ro = _np(row_offsets, np.int32)
    m = ro.shape[0] - 1
    out = np.zeros(nblocks, np.int64)
    rc = lib.oracle_nonzero_split(_p(ro), ctypes.c_int64(m), ctypes.c_int64(G), ctypes.c_int64(nblocks), _p(out))
    assert rc == 0
    return out


def mean_row_length(nnz: int, m: int) -> float:
    """d of §5.4: "computing the average row length"."""
    return nnz / m


def heuristic(d: float, threshold: float = PAPER_THRESHOLD) -> str:
    """"use merge-based on datasets whose mean row length is less than 9.35, and row
    split otherwise" -> 'merge' iff d < threshold, else 'rowsplit'."""
    return "merge" if d < threshold else "rowsplit"


def check_f32(C_gpu, C_ref, bound, rel: float = 1e-5):
    """north_star tolerance: |C_gpu - C_ref| <= rel * (|A|.|B|)_ij elementwise; bound 0 forces exact 0.
    Returns (ok, worst_ratio, index_of_worst)."""
    Cg = np.asarray(C_gpu, np.float64)
    err = np.abs(Cg - C_ref)
    ok_mask = err <= rel * bound
    ok_mask &= np.isfinite(Cg)
    ratio = np.where(bound > 0, err / np.where(bound > 0, bound, 1.0), np.where(err > 0, np.inf, 0.0))
    worst = int(np.argmax(ratio)) if ratio.size else 0
    return bool(ok_mask.all()), (float(ratio.reshape(-1)[worst]) if ratio.size else 0.0), worst
