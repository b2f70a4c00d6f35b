"""CPU-side checks of the C ABI (-m "not gpu"): the library builds/loads, exports every symbol
include/spmm.h declares, rejects bad arguments before touching the GPU, and the host-only entry points
(status strings, merge CTA count, multi-GPU row partition) behave as documented."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1803_08601_b200 import build as spmm_build
from paper_1803_08601_b200 import spmm as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    spmm_build.build()
    return S.load()


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "spmm.h")).read()
    return sorted(set(re.findall(r"SPMM_API\s+[\w\s\*]+?\b(spmm_\w+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared_functions()
    for must in ("spmm_csr_create", "spmm_csr_plan", "spmm_csr_execute", "spmm_csr_destroy",
                 "spmm_status_string", "spmm_csr_last_error", "spmm_partition_rows"):
        assert must in names
    assert set(names) == set(S.EXPORTED)


def test_library_exports_every_declared_symbol(lib):
    out = os.popen(f"nm -D --defined-only {S.LIB_PATH}").read()
    exported = set(re.findall(r" T (spmm_\w+)", out))
    assert set(_declared_functions()) <= exported
    # nothing else leaks out of the .so (hidden visibility)
    assert all(e.startswith("spmm_") for e in exported)


def test_library_is_sm100a_only(lib):
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {S.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", ""))


def test_status_strings_and_version(lib):
    assert S.spmm_abi_version() == 4
    for s in range(8):
        assert S.spmm_status_string(s).startswith("SPMM_")
    assert "unknown" in S.spmm_status_string(99)


def test_argument_errors_without_gpu(lib):
    # rejected before any CUDA call
    st, h = S.spmm_csr_create(-1, 4, 0, None, None, None, S.SPMM_F32)
    assert st == S.SPMM_ERR_INVALID_ARG and not h.value
    st, h = S.spmm_csr_create(4, 4, 3, None, None, None, S.SPMM_F32)
    assert st == S.SPMM_ERR_NULL_POINTER
    st, h = S.spmm_csr_create(4, 0, 3, 8, 8, 8, S.SPMM_F32)
    assert st == S.SPMM_ERR_INVALID_ARG  # k == 0 requires nnz == 0
    st, h = S.spmm_csr_create(4, 4, 3, 8, 8, 8, 5)
    assert st == S.SPMM_ERR_INVALID_ARG  # bad dtype
    st, h = S.spmm_csr_create(4, 4, 3, 8, 8, 8, S.SPMM_F32, 0x80)
    assert st == S.SPMM_ERR_INVALID_ARG  # unknown flag
    assert lib.spmm_csr_create(None, 1, 1, 0, None, None, None, 0, 0, None) == S.SPMM_ERR_NULL_POINTER
    st, ws, ch = S.spmm_csr_plan(None, 64, 0, 0)
    assert st == S.SPMM_ERR_NULL_POINTER
    assert S.spmm_csr_execute(None, None, 64, None, 64, 64, None, 0) == S.SPMM_ERR_NULL_POINTER
    assert S.spmm_csr_destroy(None) == S.SPMM_OK
    assert S.spmm_csr_last_error(None) == "null handle"


def test_merge_num_ctas(lib):
    assert S.spmm_merge_num_ctas(0, 0, 2048, 0) == 0
    assert S.spmm_merge_num_ctas(4, 6, 2048, 0) == 1
    assert S.spmm_merge_num_ctas(1 << 20, 16 << 20, 2048, 0) == ((17 << 20) + 2047) // 2048
    assert S.spmm_merge_num_ctas(100, 0, 256, 1) == 1  # nonzero split with no nonzeros: one CTA
    assert S.spmm_merge_num_ctas(1, 10000, 128, 1) == 79
    assert S.spmm_merge_num_ctas(5, 5, 0, 0) == -1


def _bounds(ro, parts, mode):
    ro = np.ascontiguousarray(ro, np.int32)
    b = (ctypes.c_int64 * (parts + 1))()
    st = S.spmm_partition_rows(ro.ctypes.data, len(ro) - 1, parts, mode, b)
    assert st == S.SPMM_OK
    return list(b)


def test_partition_rows_nnz_balanced_and_merge_path(lib):
    ro = [0, 2, 2, 5, 6]
    assert _bounds(ro, 3, 0) == [0, 1, 3, 4]
    rng = np.random.default_rng(0)
    for _ in range(200):
        m = int(rng.integers(1, 60))
        lens = rng.integers(0, 20, m)
        lens[rng.random(m) < 0.4] = 0
        ro = np.zeros(m + 1, np.int64)
        ro[1:] = np.cumsum(lens)
        parts = int(rng.integers(1, 9))
        nnz = int(ro[-1])
        for mode in (0, 1):
            b = _bounds(ro, parts, mode)
            assert b[0] == 0 and b[-1] == m and all(x <= y for x, y in zip(b, b[1:]))
            if mode == 0:  # definition: lower_bound(ro, p*nnz/parts)
                for p in range(1, parts):
                    t = nnz * p / parts
                    assert b[p] == int(np.searchsorted(ro, t, side="left"))
            else:  # merge-path row of diagonal p*(m+nnz)/parts (closed form: #row ends before D)
                for p in range(1, parts):
                    D = (m + nnz) * p // parts
                    assert b[p] == sum(1 for r in range(m) if r + ro[r + 1] < D)


def test_partition_rows_errors(lib):
    b = (ctypes.c_int64 * 3)()
    assert S.spmm_partition_rows(None, 4, 2, 0, b) == S.SPMM_ERR_NULL_POINTER
    ro = np.array([0, 1], np.int32)
    assert S.spmm_partition_rows(ro.ctypes.data, 1, 0, 0, b) == S.SPMM_ERR_INVALID_ARG
    assert S.spmm_partition_rows(ro.ctypes.data, 1, 2, 7, b) == S.SPMM_ERR_INVALID_ARG


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle, and CsrSpmm refuses CPU tensors."""
    import torch
    pkg = os.path.join(ROOT, "paper_1803_08601_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert "import oracle" not in src and "from oracle" not in src, f
    with pytest.raises(ValueError):
        S.CsrSpmm(torch.zeros(2, dtype=torch.int32), torch.zeros(0, dtype=torch.int32),
                  torch.zeros(0), 1)


def test_source_identity_of_the_build():
    # the build's identity for evidence files (profiles/ncu_traffic.json): a hash of the sources, headers
    # and flags -- stable across calls, sensitive to extra defines (nvcc .so files are not bit-reproducible)
    a = spmm_build.source_sha16()
    assert a == spmm_build.source_sha16() and len(a) == 16
    assert spmm_build.source_sha16(defines=("MW_U=4",)) != a
    assert os.path.join(spmm_build.ROOT, "include", "spmm.h") in spmm_build.DEPS
