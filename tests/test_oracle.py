"""Pins for the CPU oracle (-m "not gpu").  Each pin ties the oracle to something other than itself:
a library routine on a special case (dense numpy GEMM / min-plus over the densified matrix), closed
forms (identity, permutation, all-ones row sums), invariants (empty rows, row sampling, padding),
values printed in the paper / SPEC worked examples (tests/golden/), and brute force on tiny inputs.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
from paper_1803_08601_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand_csr(rng, m, k, density, dups=False, empty_frac=0.2):
    rows = []
    for i in range(m):
        if rng.random() < empty_frac:
            rows.append([])
            continue
        L = rng.binomial(k, density)
        if dups:
            rows.append(list(rng.integers(0, k, size=L)))  # unsorted, with duplicates
        else:
            rows.append(sorted(rng.choice(k, size=min(L, k), replace=False).tolist()))
    ro = np.zeros(m + 1, np.int32)
    ro[1:] = np.cumsum([len(r) for r in rows])
    col = np.array([c for r in rows for c in r], np.int32)
    return ro, col


def _densify(m, k, ro, col, val):
    A = np.zeros((m, k), np.float64 if val.dtype.kind == "f" else np.int64)
    rows = np.repeat(np.arange(m), np.diff(ro))
    np.add.at(A, (rows, col.astype(np.int64)), val)
    return A


def _present(m, k, ro, col):
    P = np.zeros((m, k), bool)
    rows = np.repeat(np.arange(m), np.diff(ro))
    P[rows, col] = True
    return P


# ------------------------------------------------------------------------------------------------
# plus-times vs dense GEMM (special case that reduces to a library routine)
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dups", [False, True])
@pytest.mark.parametrize("shape", [(1, 1, 1), (7, 13, 5), (64, 48, 33), (200, 256, 64)])
def test_f32_plus_times_equals_dense_gemm(shape, dups):
    m, k, n = shape
    rng = np.random.default_rng(m * 1000 + k + n + dups)
    ro, col = _rand_csr(rng, m, k, 0.2, dups=dups)
    val = rng.uniform(-1, 1, col.shape[0]).astype(np.float32)
    B = rng.uniform(-1, 1, (k, n)).astype(np.float32)
    C, bound = oracle.spmm("f32_plus_times", m, k, n, ro, col, val, B)
    A = _densify(m, k, ro, col, val.astype(np.float64))
    ref = A @ B.astype(np.float64)
    # fp64 sums in a different order: agree to fp64 rounding
    assert np.allclose(C, ref, rtol=0, atol=1e-12 * max(1.0, np.abs(A).sum(1).max()))
    # bound = |A|.|B| (exact identity for sums of |a||b|; duplicates add up in |A| only if same sign,
    # so compare against the per-entry definition instead)
    Aabs = np.zeros((m, k))
    rows = np.repeat(np.arange(m), np.diff(ro))
    np.add.at(Aabs, (rows, col.astype(np.int64)), np.abs(val.astype(np.float64)))
    assert np.allclose(bound, Aabs @ np.abs(B.astype(np.float64)), rtol=1e-12, atol=1e-300)


def test_f32_plus_times_catches_transpose_and_index_mistakes():
    """A non-symmetric 2x3 case with distinct entries: a transposed operand or an off-by-one index
    would change at least one entry."""
    ro = np.array([0, 2, 3], np.int32)
    col = np.array([0, 2, 1], np.int32)
    val = np.array([2.0, -3.0, 5.0], np.float32)
    B = np.array([[1.0, 10.0], [100.0, 1000.0], [0.5, 0.25]], np.float32)
    C, _ = oracle.spmm("f32_plus_times", 2, 3, 2, ro, col, val, B)
    assert C.tolist() == [[2.0 - 1.5, 20.0 - 0.75], [500.0, 5000.0]]


@pytest.mark.parametrize("shape", [(5, 5, 3), (64, 100, 33), (150, 90, 64)])
def test_i32_plus_times_wraps_like_int64_mod_2_32(shape):
    m, k, n = shape
    rng = np.random.default_rng(k + n)
    ro, col = _rand_csr(rng, m, k, 0.3)
    val = rng.integers(-(2**20), 2**20, col.shape[0]).astype(np.int32)  # products up to 2^40: wraps
    B = rng.integers(-(2**20), 2**20, (k, n)).astype(np.int32)
    C = oracle.spmm("i32_plus_times", m, k, n, ro, col, val, B)
    A = _densify(m, k, ro, col, val.astype(np.int64))
    ref = (A.astype(object) @ B.astype(object)) if m * k * n < 5000 else None
    full = (A @ B.astype(np.int64))  # int64 wraps mod 2^64; low 32 bits are exact
    exp = (full & 0xFFFFFFFF).astype(np.uint32).view(np.int32)
    assert np.array_equal(C, exp)
    if ref is not None:
        exp2 = np.vectorize(lambda x: ((int(x) + 2**31) % 2**32) - 2**31)(ref).astype(np.int32)
        assert np.array_equal(C, exp2)


@pytest.mark.parametrize("kind", ["f32_min_plus", "i32_min_plus"])
@pytest.mark.parametrize("shape", [(6, 4, 3), (50, 70, 33), (128, 40, 64)])
def test_min_plus_equals_dense_min_reduction(kind, shape):
    m, k, n = shape
    rng = np.random.default_rng(m + 7 * k + n)
    ro, col = _rand_csr(rng, m, k, 0.25)
    if kind == "f32_min_plus":
        val = rng.uniform(1, 1000, col.shape[0]).astype(np.float32)
        B = rng.uniform(1, 1000, (k, n)).astype(np.float32)
    else:
        val = rng.integers(1, 1000, col.shape[0]).astype(np.int32)
        B = rng.integers(1, 1000, (k, n)).astype(np.int32)
    C = oracle.spmm(kind, m, k, n, ro, col, val, B)
    P = _present(m, k, ro, col)
    A = np.zeros((m, k), val.dtype)
    rows = np.repeat(np.arange(m), np.diff(ro))
    A[rows, col] = val
    S = A[:, :, None] + B[None, :, :]  # fp32 add in numpy float32 (one rounding) / int32
    if kind == "f32_min_plus":
        S = np.where(P[:, :, None], S, np.float32(np.inf))
        exp = S.min(axis=1).astype(np.float32)
    else:
        S = np.where(P[:, :, None], S, np.int32(2**31 - 1))
        exp = S.min(axis=1).astype(np.int32)
    assert np.array_equal(C, exp)


# ------------------------------------------------------------------------------------------------
# closed forms and invariants
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("kind", synth.KINDS)
def test_identity_gives_B(kind):
    k = n = 37
    ro = np.arange(k + 1, dtype=np.int32)
    col = np.arange(k, dtype=np.int32)
    one = 0 if kind.endswith("min_plus") else 1
    val = np.full(k, one, np.float32 if kind.startswith("f32") else np.int32)
    B = synth.dense(k, n, 5, kind).numpy()
    out = oracle.spmm(kind, k, k, n, ro, col, val, B)
    C = out[0] if kind == "f32_plus_times" else out
    assert np.array_equal(C.astype(B.dtype), B)


@pytest.mark.parametrize("kind", synth.KINDS)
def test_permutation_gives_PB(kind):
    k = n = 41
    perm = np.random.default_rng(3).permutation(k).astype(np.int32)
    ro = np.arange(k + 1, dtype=np.int32)
    one = 0 if kind.endswith("min_plus") else 1
    val = np.full(k, one, np.float32 if kind.startswith("f32") else np.int32)
    B = synth.dense(k, n, 6, kind).numpy()
    out = oracle.spmm(kind, k, k, n, ro, perm, val, B)
    C = out[0] if kind == "f32_plus_times" else out
    assert np.array_equal(C.astype(B.dtype), B[perm])


def test_all_ones_dense_pattern_gives_column_sums_of_B():
    m, k, n = 9, 300, 17
    ro = (np.arange(m + 1) * k).astype(np.int32)
    col = np.tile(np.arange(k, dtype=np.int32), m)
    val = np.ones(m * k, np.float32)
    rng = np.random.default_rng(0)
    B = rng.integers(-(2**24) // k, (2**24) // k, (k, n)).astype(np.float32)  # sums exact in fp32
    C, _ = oracle.spmm("f32_plus_times", m, k, n, ro, col, val, B)
    s = B.astype(np.int64).sum(axis=0)
    assert np.array_equal(C, np.broadcast_to(s.astype(np.float64), (m, n)))


@pytest.mark.parametrize("kind", synth.KINDS)
def test_empty_rows_give_identity(kind):
    m, k, n = 6, 5, 4
    ro = np.array([0, 0, 2, 2, 2, 3, 3], np.int32)
    col = np.array([1, 4, 0], np.int32)
    val = synth.values(3, 1, kind).numpy()
    B = synth.dense(k, n, 2, kind).numpy()
    out = oracle.spmm(kind, m, k, n, ro, col, val, B)
    C = out[0] if kind == "f32_plus_times" else out
    ident = synth.identity_value(kind)
    for r in (0, 2, 3, 5):
        assert np.all(C[r] == ident)
    assert not np.any(C[1] == ident) or kind.endswith("plus_times")


@pytest.mark.parametrize("kind", synth.KINDS)
def test_row_sampling_and_padding_invariants(kind):
    p = synth.uniform_rows(300, 200, 7, 11)
    val = synth.values(p.nnz, 12, kind)
    B = synth.dense(200, 33, 13, kind, ld=40)  # NaN / INT32_MIN poison in cols 33..39
    full = oracle.spmm(kind, p.m, p.k, 33, p.row_offsets, p.col_indices, val, B, ldb=40)
    tight = oracle.spmm(kind, p.m, p.k, 33, p.row_offsets, p.col_indices, val, B[:, :33].contiguous(), ldb=33)
    rows = np.array([299, 0, 17, 17, 150], np.int64)
    samp = oracle.spmm(kind, p.m, p.k, 33, p.row_offsets, p.col_indices, val, B, ldb=40, rows=rows)
    if kind == "f32_plus_times":
        full, tight, samp = full[0], tight[0], samp[0]
        assert np.all(np.isfinite(full))
    assert np.array_equal(full, tight)
    assert np.array_equal(samp, full[rows])


def test_spec_worked_examples():
    g = json.load(open(os.path.join(GOLDEN, "spec_spmm_examples.json")))
    for c in g["cases"]:
        B = np.array(c["B"], np.float32)
        C, _ = oracle.spmm("f32_plus_times", c["m"], c["k"], B.shape[1], np.array(c["row_offsets"], np.int32),
                           np.array(c["col_indices"], np.int32), np.array(c["values"], np.float32), B)
        assert C.tolist() == c["C"], c["name"]


def test_thread_count_invariance():
    p = synth.uniform_rows(500, 500, 9, 4)
    val = synth.values(p.nnz, 1, "f32_plus_times")
    B = synth.dense(500, 16, 2, "f32_plus_times")
    a, _ = oracle.spmm("f32_plus_times", p.m, p.k, 16, p.row_offsets, p.col_indices, val, B)
    b, _ = oracle.spmm("f32_plus_times", p.m, p.k, 16, p.row_offsets, p.col_indices, val, B, rows=np.arange(p.m))
    assert np.array_equal(a, b)


# ------------------------------------------------------------------------------------------------
# partition oracles
# ------------------------------------------------------------------------------------------------
def _valid_states(ro, d):
    """Closed-form characterisation of merge-path states on diagonal d: (i, j) with i + j = d,
    ro[i] <= j <= ro[i+1] for i < m, and j == nnz for i == m (the path is a monotone staircase that
    takes row end i only once all of row i's nonzeros are consumed)."""
    m = len(ro) - 1
    nnz = ro[-1]
    out = []
    for i in range(max(0, d - nnz), min(d, m) + 1):
        j = d - i
        if i < m and ro[i] <= j <= ro[i + 1]:
            out.append((i, j))
        elif i == m and j == nnz:
            out.append((i, j))
    return out


def _rand_offsets(rng, m, maxlen):
    lens = rng.integers(0, maxlen + 1, m)
    lens[rng.random(m) < 0.3] = 0  # runs of empty rows
    ro = np.zeros(m + 1, np.int32)
    ro[1:] = np.cumsum(lens)
    return ro


def test_merge_walk_matches_closed_form_and_row_end_count():
    rng = np.random.default_rng(81)
    cases = [np.array([0, 2, 2, 5, 6], np.int32), np.array([0], np.int32), np.array([0, 0, 0], np.int32),
             np.array([0, 5], np.int32)]
    cases += [_rand_offsets(rng, int(rng.integers(1, 40)), int(rng.integers(0, 9))) for _ in range(300)]
    for ro in cases:
        m = len(ro) - 1
        nnz = int(ro[-1])
        diags = np.arange(m + nnz + 1)
        wi, wj = oracle.merge_path_walk(ro, diags)
        for d in diags:
            st = _valid_states(ro, int(d))
            assert st == [(int(wi[d]), int(wj[d]))], (ro.tolist(), d, st)
            # row end of row r sits at path position r + ro[r+1]
            assert wi[d] == sum(1 for r in range(m) if r + ro[r + 1] < d)


def test_merge_walk_small_example_fig2c_shape():
    # ro = [0,2,2,5,6]: items in path order are n0 n1 R0 R1 n2 n3 n4 R2 n5 R3
    ro = np.array([0, 2, 2, 5, 6], np.int32)
    wi, wj = oracle.merge_path_walk(ro, np.arange(11))
    assert list(zip(wi.tolist(), wj.tolist())) == [(0, 0), (0, 1), (0, 2), (1, 2), (2, 2), (2, 3), (2, 4),
                                                   (2, 5), (3, 5), (3, 6), (4, 6)]


def test_nonzero_split_golden_and_definition():
    g = json.load(open(os.path.join(GOLDEN, "nonzero_split_spec.json")))
    c0 = g["cases"][0]
    ro = np.array(c0["row_offsets"], np.int32)
    nb = -(-int(ro[-1]) // c0["G"])
    assert oracle.nonzero_split(ro, c0["G"], nb).tolist() == c0["start_rows"]
    c1 = g["cases"][1]
    ro = np.array(c1["row_offsets"], np.int32)
    nb = -(-int(ro[-1]) // c1["G"])
    assert nb == c1["nblocks"]
    assert set(oracle.nonzero_split(ro, c1["G"], nb).tolist()) == {c1["start_rows_all"]}
    rng = np.random.default_rng(5)
    for _ in range(200):
        ro = _rand_offsets(rng, int(rng.integers(1, 30)), 6)
        nnz = int(ro[-1])
        if nnz == 0:
            continue
        G = int(rng.integers(1, 9))
        nb = -(-nnz // G)
        rows = oracle.nonzero_split(ro, G, nb)
        m = len(ro) - 1
        for c in range(1, nb):
            r = rows[c]
            t = c * G
            assert ro[r] <= t and (r == m or ro[r + 1] > t)  # largest r with ro[r] <= t
        assert rows[0] == 0


def test_heuristic_paper_values():
    g = json.load(open(os.path.join(GOLDEN, "heuristic_paper.json")))
    for c in g["cases"]:
        assert oracle.heuristic(c["d"], g["threshold"]) == c["expect"], c["cite"]
    # monotone in d
    ds = np.linspace(0, 40, 401)
    picks = [oracle.heuristic(d) for d in ds]
    first_rs = picks.index("rowsplit")
    assert all(p == "rowsplit" for p in picks[first_rs:])
    assert oracle.mean_row_length(16_777_216, 1 << 20) == 16.0


def test_check_f32_tolerance_rule():
    ref = np.array([1.0, 0.0, 2.0])
    bound = np.array([1.0, 0.0, 4.0])
    ok, _, _ = oracle.check_f32(np.array([1.0 + 5e-6, 0.0, 2.0 - 3.9e-5], np.float32), ref, bound)
    assert ok
    ok, _, _ = oracle.check_f32(np.array([1.0, 1e-30, 2.0], np.float32), ref, bound)  # bound 0 -> exact
    assert not ok
    ok, _, _ = oracle.check_f32(np.array([1.0 + 2e-5, 0.0, 2.0], np.float32), ref, bound)
    assert not ok


def test_synth_generators_are_canonical_and_device_independent():
    for p in (synth.uniform_rows(100, 80, 10, 3), synth.banded(64), synth.rmat(9, 8, 4),
              synth.lognormal_rows(200, 150, 7.92, 5), synth.aspect(256, 16)):
        ro = p.row_offsets.numpy().astype(np.int64)
        col = p.col_indices.numpy()
        assert ro[0] == 0 and np.all(np.diff(ro) >= 0) and ro[-1] == len(col)
        assert np.all((col >= 0) & (col < p.k))
        for i in range(p.m):
            seg = col[ro[i]:ro[i + 1]]
            assert np.all(np.diff(seg) > 0)
    u = synth.uniform_rows(50, 1000, 16, 9)
    assert np.all(np.diff(u.row_offsets.numpy()) == 16)
    b = synth.banded(1000)
    assert np.all(np.diff(b.row_offsets.numpy()) == 16)
    # R-MAT 16 statistics in line with the survey's trend table (scale 18: 43% empty rows)
    r = synth.rmat(14, 16, 1805)
    lens = np.diff(r.row_offsets.numpy())
    assert 0.30 < (lens == 0).mean() < 0.50 and lens.max() > 20 * lens.mean()
    # hash is a pure function of (seed, stream, idx)
    h1 = synth.counter_u32(1, 2, torch.arange(10, dtype=torch.int64))
    h2 = synth.counter_u32(1, 2, torch.arange(10, dtype=torch.int64))
    assert torch.equal(h1, h2) and int(h1.max()) < 2**32 and int(h1.min()) >= 0
