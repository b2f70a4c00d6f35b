"""GPU parity (-m gpu): the CUDA path, called through the C ABI (ctypes binding), against the CPU
oracle on the same seeded inputs.  Bar (north_star / SURVEY.md §8(c)): bit-exact for int32
plus-times and both min-plus semirings; |C - C_ref| <= 1e-5 * (|A|.|B|)_ij for fp32 plus-times.
Integer-valued partition outputs are compared bit-exactly with the oracle's brute-force walk."""
import numpy as np
import pytest
import torch

import oracle
from paper_1803_08601_b200 import spmm as S
from paper_1803_08601_b200 import synth

pytestmark = pytest.mark.gpu

DEV = "cuda"
TOL = 1e-5


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    S.load()


def make_inputs(p: synth.CsrPattern, kind: str, n: int, seed: int = 7, ldb=None, ldc=None, b_offset=0):
    val = synth.values(p.nnz, seed + 100, kind)
    Bh = synth.dense(p.k, n, seed + 200, kind, ld=ldb)
    ld_b = Bh.shape[1]
    ro = p.row_offsets.to(DEV)
    ci = p.col_indices.to(DEV)
    vd = val.to(DEV)
    if b_offset:  # misaligned B: shift the base pointer by b_offset elements
        flat = torch.empty(Bh.numel() + b_offset, dtype=Bh.dtype, device=DEV)
        flat[b_offset:] = Bh.reshape(-1).to(DEV)
        Bd = flat[b_offset:].view(p.k, ld_b)
    else:
        Bd = Bh.to(DEV)
    ld_c = n if ldc is None else ldc
    poison = float("nan") if kind.startswith("f32") else -(2**31)
    Cd = torch.full((p.m, ld_c), poison, dtype=Bh.dtype, device=DEV)
    return val, Bh, ro, ci, vd, Bd, Cd


def run_gpu(p, kind, n, algo, ro, ci, vd, Bd, Cd, **plan_kw):
    sr = "plus_times" if kind.endswith("plus_times") else "min_plus"
    op = S.CsrSpmm(ro, ci, vd, p.k)
    chosen = op.plan(n, algo, sr, **plan_kw)
    Cview = Cd[:, :n] if Cd.shape[1] > n else Cd
    op.execute(Bd[:, :n] if Bd.shape[1] > n else Bd, Cview)
    torch.cuda.synchronize()
    info = op.info()
    op.close()
    return chosen, info


def check(p, kind, n, val, Bh, Cd, rows=None, ldb=None):
    C = Cd[:, :n].cpu().numpy()
    if rows is not None:
        C = C[np.asarray(rows)]
    ref = oracle.spmm(kind, p.m, p.k, n, p.row_offsets, p.col_indices, val, Bh, ldb=Bh.shape[1], rows=rows)
    if kind == "f32_plus_times":
        Cref, bound = ref
        ok, worst, idx = oracle.check_f32(C, Cref, bound, TOL)
        assert ok, f"fp32 tolerance violated: worst |err|/bound = {worst} at flat index {idx}"
    else:
        if not np.array_equal(C, ref):
            bad = np.argwhere(C != ref)
            r, c = bad[0]
            raise AssertionError(f"{len(bad)} mismatches, first at ({r},{c}): gpu {C[r, c]} ref {ref[r, c]}")
    if Cd.shape[1] > n:  # columns [n, ldc) untouched
        tail = Cd[:, n:].cpu()
        if kind.startswith("f32"):
            assert torch.isnan(tail).all()
        else:
            assert (tail == -(2**31)).all()


ALGOS = ["rowsplit", "merge", "auto"]


# ------------------------------------------------------------------------------------------------
# config 0 (tiny uniform) across semirings, n and both kernels
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("kind", synth.KINDS)
@pytest.mark.parametrize("n", [1, 2, 3, 4, 7, 8, 16, 31, 32, 33, 48, 64, 65, 100, 127, 128])
@pytest.mark.parametrize("algo", ALGOS)
def test_config0_parity(kind, n, algo):
    p = synth.config_pattern(0)
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
    run_gpu(p, kind, n, algo, ro, ci, vd, Bd, Cd)
    check(p, kind, n, val, Bh, Cd)


@pytest.mark.parametrize("partition", ["merge_path", "nonzero_split"])
@pytest.mark.parametrize("items", [32, 96, 256, 512, 2048, 4096])
@pytest.mark.parametrize("kind", ["f32_plus_times", "i32_min_plus"])
def test_merge_partitions_and_tile_sizes(partition, items, kind):
    p = synth.lognormal_rows(3000, 2000, 7.92, 17)  # ragged rows, empty rows, several CTAs
    n = 64
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
    run_gpu(p, kind, n, "merge", ro, ci, vd, Bd, Cd, partition=partition, items_per_cta=items)
    check(p, kind, n, val, Bh, Cd)


# ------------------------------------------------------------------------------------------------
# adversarial families (SPEC.md:457 / SURVEY.md §4)
# ------------------------------------------------------------------------------------------------
def _families():
    fam = {}
    fam["all_empty"] = synth.from_rows(50, 40, [[] for _ in range(50)])
    fam["one_giant_row"] = synth.explicit_lengths(1, 200_000, [100_000], seed=3)
    fam["giant_row_plus_singletons"] = synth.explicit_lengths(1001, 150_000, [100_000] + [1] * 1000, seed=4)
    fam["lengths_1_31_32_33"] = synth.explicit_lengths(400, 300, [1, 31, 32, 33] * 100, seed=5)
    lens = [0] * 997 + [5, 0, 0, 64]
    fam["many_empty_rows"] = synth.explicit_lengths(len(lens), 100, lens, seed=6)
    fam["leading_trailing_empty"] = synth.explicit_lengths(12, 10, [0, 0, 0, 3, 0, 10, 1, 0, 0, 2, 0, 0], seed=7)
    fam["unsorted_duplicates"] = synth.from_lengths_unsorted(300, 50, [int(x) for x in (np.arange(300) % 13)],
                                                             seed=8, allow_dups=True)
    fam["rmat12"] = synth.rmat(12, 16, 99)
    fam["aspect_short_wide"] = synth.aspect(1 << 16, 4)      # 4 rows x 16384 nnz
    fam["aspect_tall"] = synth.aspect(1 << 16, 1 << 15)      # 32768 rows x 2
    fam["single_row_single_nnz"] = synth.from_rows(1, 1, [[0]])
    return fam


FAMILY_NAMES = ["all_empty", "one_giant_row", "giant_row_plus_singletons", "lengths_1_31_32_33", "many_empty_rows",
                "leading_trailing_empty", "unsorted_duplicates", "rmat12", "aspect_short_wide", "aspect_tall",
                "single_row_single_nnz"]
_FAM_CACHE = {}


def family(name):
    if not _FAM_CACHE:
        _FAM_CACHE.update(_families())
    return _FAM_CACHE[name]


@pytest.mark.parametrize("fam", FAMILY_NAMES)
@pytest.mark.parametrize("kind", ["f32_plus_times", "i32_plus_times", "f32_min_plus"])
@pytest.mark.parametrize("n", [1, 16, 33, 64, 128])
@pytest.mark.parametrize("algo", ["rowsplit", "merge"])
def test_adversarial_parity(fam, kind, n, algo):
    p = family(fam)
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
    run_gpu(p, kind, n, algo, ro, ci, vd, Bd, Cd)
    check(p, kind, n, val, Bh, Cd)


@pytest.mark.parametrize("algo", ["rowsplit", "merge"])
@pytest.mark.parametrize("kind", synth.KINDS)
def test_padding_and_misalignment(algo, kind):
    """ldb/ldc > n (poisoned padding must not be read or written) and a B base pointer that is
    only 4-byte aligned (forces the scalar path)."""
    p = synth.uniform_rows(700, 500, 9, 21)
    for n, ldb, ldc, off in ((64, 70, 72, 0), (64, 64, 64, 1), (17, 20, 19, 3), (128, 131, 128, 1), (1, 3, 2, 0)):
        val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n, ldb=ldb, ldc=ldc, b_offset=off)
        run_gpu(p, kind, n, algo, ro, ci, vd, Bd, Cd)
        check(p, kind, n, val, Bh, Cd)


def test_integer_and_minplus_bit_identical_across_kernels():
    """Order-independent semirings: every kernel / partition / tile size gives the same bits."""
    p = synth.rmat(13, 8, 5)
    for kind in ("i32_plus_times", "i32_min_plus", "f32_min_plus"):
        outs = []
        for algo, kw in (("rowsplit", {}), ("merge", {}), ("merge", {"partition": "nonzero_split"}),
                         ("merge", {"items_per_cta": 256}), ("auto", {})):
            val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, 64)
            run_gpu(p, kind, 64, algo, ro, ci, vd, Bd, Cd, **kw)
            outs.append(Cd.cpu())
        for o in outs[1:]:
            assert torch.equal(o, outs[0])


def test_fp32_deterministic_run_to_run():
    p = synth.rmat(12, 16, 8)
    for algo in ("rowsplit", "merge"):
        res = []
        for _ in range(2):
            val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, "f32_plus_times", 64)
            run_gpu(p, "f32_plus_times", 64, algo, ro, ci, vd, Bd, Cd)
            res.append(Cd.cpu())
        assert torch.equal(res[0], res[1])


def test_row_permutation_equivariance_and_power_of_two_scaling():
    p = synth.uniform_rows(513, 400, 11, 33)
    kind, n = "f32_plus_times", 32
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
    run_gpu(p, kind, n, "rowsplit", ro, ci, vd, Bd, Cd)
    base = Cd.cpu()
    perm = torch.randperm(p.m, generator=torch.Generator().manual_seed(1))
    lens = (p.row_offsets[1:] - p.row_offsets[:-1]).long()
    starts = p.row_offsets[:-1].long()
    new_ro = torch.zeros(p.m + 1, dtype=torch.int64)
    new_ro[1:] = torch.cumsum(lens[perm], 0)
    idx = torch.cat([torch.arange(starts[r], starts[r] + lens[r]) for r in perm.tolist()])
    Cd2 = torch.empty_like(Cd)
    op = S.CsrSpmm(new_ro.to(torch.int32).to(DEV), p.col_indices[idx].to(DEV), (val[idx] * 8.0).to(DEV), p.k)
    op.plan(n, "rowsplit")
    op.execute(Bd, Cd2)
    torch.cuda.synchronize()
    assert torch.equal(Cd2.cpu(), base[perm] * 8.0)


# ------------------------------------------------------------------------------------------------
# partition kernel (Alg. 1 line 2) vs the oracle's brute-force walk / linear scan, bit-exact
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("mode", [0, 1])
def test_partition_kernel_matches_oracle(mode):
    rng = np.random.default_rng(40 + mode)
    cases = [np.array([0, 2, 2, 5, 6], np.int32), np.array([0, 0, 0, 0], np.int32)]
    for _ in range(60):
        m = int(rng.integers(1, 3000))
        lens = rng.integers(0, 12, m)
        lens[rng.random(m) < 0.5] = 0
        if rng.random() < 0.2:
            lens[int(rng.integers(0, m))] = int(rng.integers(100, 5000))
        ro = np.zeros(m + 1, np.int32)
        ro[1:] = np.cumsum(lens)
        cases.append(ro)
    for ro in cases:
        m, nnz = len(ro) - 1, int(ro[-1])
        for items in (1, 3, 7, 256, 2048):
            nc = S.spmm_merge_num_ctas(m, nnz, items, mode)
            if nc <= 0:
                continue
            states = torch.empty(2 * (nc + 1), dtype=torch.int32, device=DEV)
            rod = torch.from_numpy(ro).to(DEV)
            st = S.spmm_merge_partition(rod.data_ptr(), m, nnz, items, mode, nc, states.data_ptr())
            assert st == S.SPMM_OK
            torch.cuda.synchronize()
            got = states.cpu().numpy().reshape(-1, 2)
            if mode == 0:
                diags = np.minimum(np.arange(nc + 1, dtype=np.int64) * items, m + nnz)
                wi, wj = oracle.merge_path_walk(ro, diags)
                assert np.array_equal(got[:, 0], wi) and np.array_equal(got[:, 1], wj)
            else:
                rows = oracle.nonzero_split(ro, items, nc)
                assert np.array_equal(got[:nc, 0], rows)
                assert np.array_equal(got[:nc, 1], np.arange(nc) * items)
                assert tuple(got[nc]) == (m, nnz)
    # SPEC.md:284 worked example through the kernel
    ro = torch.tensor([0, 2, 2, 5, 6], dtype=torch.int32, device=DEV)
    states = torch.empty(2 * 3, dtype=torch.int32, device=DEV)
    assert S.spmm_merge_partition(ro.data_ptr(), 4, 6, 3, 1, 2, states.data_ptr()) == S.SPMM_OK
    assert states.cpu().view(-1, 2)[:, 0].tolist() == [0, 2, 4]


# ------------------------------------------------------------------------------------------------
# heuristic (§5.4) and the ABI's error behaviour on a live device
# ------------------------------------------------------------------------------------------------
def test_heuristic_choice_matches_oracle_rule():
    for d in (1, 2, 7, 9, 10, 16, 62):
        p = synth.uniform_rows(2000, 4000, d, d)
        vd = synth.values(p.nnz, 1, "f32_plus_times").to(DEV)
        op = S.CsrSpmm(p.row_offsets.to(DEV), p.col_indices.to(DEV), vd, p.k)
        chosen = op.plan(64, "auto", policy="paper")
        assert chosen == oracle.heuristic(oracle.mean_row_length(p.nnz, p.m))
        op.close()
    # skew guard (AUTO policy): R-MAT has d >= 9.35 but a row far above the per-warp fair share
    r = synth.rmat(16, 16, 1805)
    vd = synth.values(r.nnz, 1, "f32_plus_times").to(DEV)
    op = S.CsrSpmm(r.row_offsets.to(DEV), r.col_indices.to(DEV), vd, r.k)
    assert op.plan(64, "auto", policy="paper") == "rowsplit"
    assert op.plan(64, "auto", policy="auto") == "merge"
    assert op.info()["max_row_length"] == int((r.row_offsets[1:] - r.row_offsets[:-1]).max())
    op.close()


def test_auto_few_rows_guard_needs_enough_work():
    # few rows + large work (aspect 1024 x 16384) -> merge; few rows + tiny work (config 0) -> row split
    for pat, want in ((synth.aspect(1 << 24, 1 << 10), "merge"), (synth.config_pattern(0), "rowsplit")):
        vd = synth.values(pat.nnz, 1, "f32_plus_times").to(DEV)
        op = S.CsrSpmm(pat.row_offsets.to(DEV), pat.col_indices.to(DEV), vd, pat.k)
        assert op.plan(64, "auto") == want
        op.close()


@pytest.mark.parametrize("kind", synth.KINDS)
@pytest.mark.parametrize("n", [8, 64, 128])
def test_rowsplit_tile_queue_for_irregular_rows(kind, n):
    # lognormal rows (max row >> mean): row split under the AUTO policy takes the row tiles from a
    # queue in the workspace (256 bytes); results unchanged
    p = synth.lognormal_rows(20000, 9000, 7.92, 77)
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
    sr = "plus_times" if kind.endswith("plus_times") else "min_plus"
    op = S.CsrSpmm(ro, ci, vd, p.k)
    assert op.plan(n, "rowsplit", sr) == "rowsplit"
    info = op.info()
    assert info["workspace_bytes"] == 256 and info["launches_per_execute"] == 2 and info["compute_launch"] == 1
    op.execute(Bd, Cd)
    torch.cuda.synchronize()
    check(p, kind, n, val, Bh, Cd)
    # a second execute on the SAME op and workspace, C re-poisoned: the queue must be re-zeroed, or
    # every tile would be skipped and the poison would survive
    Cd.fill_(float("nan") if kind.startswith("f32") else -(2**31))
    op.execute(Bd, Cd)
    torch.cuda.synchronize()
    op.close()
    check(p, kind, n, val, Bh, Cd)


def test_auto_refit_guards():
    """Round-2 refit of AUTO (profiles/r02_config3_summary.txt): mildly skewed rows with n >= 16 and very
    short rows with wide B go to merge; banded short rows and narrow B stay on row split."""
    cases = ((synth.lognormal_rows(1 << 16, 1 << 16, 7.92, 87), 64, "merge"),
             (synth.lognormal_rows(1 << 16, 1 << 16, 7.92, 87), 4, "rowsplit"),
             (synth.uniform_rows(1 << 16, 1 << 16, 1, 5), 64, "merge"),
             (synth.uniform_rows(1 << 16, 1 << 16, 1, 5), 16, "rowsplit"),
             (synth.uniform_rows(1 << 16, 1 << 16, 2, 5), 128, "merge"),
             # d = 4 at n = 128 went back to row split with the 8-lane x 4-block row groups (session 3)
             (synth.uniform_rows(1 << 16, 1 << 16, 4, 5), 128, "rowsplit"),
             (synth.banded(1 << 16, 2, 2), 64, "rowsplit"))
    for pat, n, want in cases:
        vd = synth.values(pat.nnz, 1, "f32_plus_times").to(DEV)
        op = S.CsrSpmm(pat.row_offsets.to(DEV), pat.col_indices.to(DEV), vd, pat.k)
        got = op.plan(n, "auto")
        inf = op.info()
        op.close()
        assert got == want, (pat.name, n, inf["mean_row_length"], inf["max_row_length"])


def test_auto_picks_merge_for_rows_too_long_to_stage():
    # 1.2 x 16 x d > 8192 <=> d > 426: a 16-row tile no longer fits the staged slice
    for d, want in ((400, "rowsplit"), (450, "merge")):
        p = synth.uniform_rows(40000, 20000, d, d)
        vd = synth.values(p.nnz, 1, "f32_plus_times").to(DEV)
        op = S.CsrSpmm(p.row_offsets.to(DEV), p.col_indices.to(DEV), vd, p.k)
        assert op.plan(64, "auto") == want
        op.close()


def test_abi_errors_on_device():
    p = synth.uniform_rows(100, 100, 4, 2)
    vd = synth.values(p.nnz, 1, "f32_plus_times").to(DEV)
    op = S.CsrSpmm(p.row_offsets.to(DEV), p.col_indices.to(DEV), vd, p.k)
    with pytest.raises(S.SpmmError) as e:
        op.plan(129)
    assert e.value.status == S.SPMM_ERR_UNSUPPORTED
    st = S.spmm_csr_execute(op._h, None, 8, None, 8, 8, None, 0)
    assert st == S.SPMM_ERR_NOT_PLANNED
    op.plan(8, "merge")
    B = torch.zeros(100, 8, device=DEV)
    C = torch.zeros(100, 8, device=DEV)
    assert S.spmm_csr_execute(op._h, B.data_ptr(), 8, C.data_ptr(), 8, 9, None, 0) == S.SPMM_ERR_INVALID_ARG
    assert S.spmm_csr_execute(op._h, B.data_ptr(), 8, C.data_ptr(), 8, 8, op.workspace.data_ptr(), 0) == \
        S.SPMM_ERR_WORKSPACE_TOO_SMALL
    assert S.spmm_csr_execute(op._h, B.data_ptr(), 4, C.data_ptr(), 8, 8, op.workspace.data_ptr(),
                              op.ws_bytes) == S.SPMM_ERR_INVALID_ARG
    assert "workspace" in S.spmm_csr_last_error(op._h) or "ld" in S.spmm_csr_last_error(op._h)
    op.close()
    # validation catches broken CSR invariants
    bad_ro = torch.tensor([0, 3, 2, 4], dtype=torch.int32, device=DEV)
    col = torch.tensor([0, 1, 2, 3], dtype=torch.int32, device=DEV)
    with pytest.raises(S.SpmmError) as e:
        S.CsrSpmm(bad_ro, col, torch.ones(4, device=DEV), 4, validate=True)
    assert e.value.status == S.SPMM_ERR_INVALID_CSR
    good_ro = torch.tensor([0, 1, 2, 4], dtype=torch.int32, device=DEV)
    with pytest.raises(S.SpmmError):
        S.CsrSpmm(good_ro, torch.tensor([0, 1, 2, 9], dtype=torch.int32, device=DEV), torch.ones(4, device=DEV), 4,
                  validate=True)
    S.CsrSpmm(good_ro, col, torch.ones(4, device=DEV), 4, validate=True).close()


def test_empty_and_degenerate_shapes():
    # m = 0: no-op
    ro = torch.zeros(1, dtype=torch.int32, device=DEV)
    op = S.CsrSpmm(ro, torch.zeros(0, dtype=torch.int32, device=DEV), torch.zeros(0, device=DEV), 5)
    op.plan(4)
    op.execute(torch.zeros(5, 4, device=DEV), torch.zeros(0, 4, device=DEV))
    op.close()
    # nnz = 0: identity everywhere, for every semiring and both kernels
    for kind in synth.KINDS:
        p = synth.from_rows(9, 3, [[]] * 9)
        for algo in ("rowsplit", "merge"):
            val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, 5)
            run_gpu(p, kind, 5, algo, ro, ci, vd, Bd, Cd)
            check(p, kind, 5, val, Bh, Cd)


# ------------------------------------------------------------------------------------------------
# BASELINE.json full sizes, in the launch configuration bench.py times, sampled rows
# ------------------------------------------------------------------------------------------------
def _sample_rows(p, extra_rows=(), seed=0):
    lens = (p.row_offsets[1:] - p.row_offsets[:-1]).to(torch.int64)
    longest = torch.topk(lens, min(256, p.m)).indices
    rng = torch.Generator().manual_seed(seed)
    rand = torch.randint(0, p.m, (4096,), generator=rng)
    edge = torch.tensor([0, 1, p.m - 2, p.m - 1] + list(extra_rows), dtype=torch.int64).clamp(0, p.m - 1)
    return torch.unique(torch.cat([longest.cpu(), rand, edge])).numpy()


@pytest.mark.parametrize("cfg", [1, 2])
@pytest.mark.parametrize("algo", ["auto", "rowsplit", "merge"])
def test_full_size_configs_sampled(cfg, algo):
    p = synth.config_pattern(cfg, device=DEV).to("cpu")
    kind, n = "f32_plus_times", 64
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n, seed=synth.STRUCT_SEED + cfg)
    chosen, info = run_gpu(p, kind, n, algo, ro, ci, vd, Bd, Cd)
    rows = _sample_rows(p)
    check(p, kind, n, val, Bh, Cd, rows=rows)
    # every row was written (no poison left anywhere)
    assert not torch.isnan(Cd).any()


# ------------------------------------------------------------------------------------------------
# B staging of the row-split kernel (compact B row spans copied to shared memory by TMA)
# ------------------------------------------------------------------------------------------------
def _banded_with_far_entries(m: int, every: int, seed: int = 3):
    """Band of 9 plus, in every `every`-th row, one far column: tiles holding such a row have a
    scattered B span and keep the global gathers; the others are staged."""
    cols, ro = [], [0]
    for i in range(m):
        row = sorted({(i + o) % m for o in range(-4, 5)} | ({(i * 7919 + seed * 104729) % m} if i % every == 0 else set()))
        cols += row
        ro.append(len(cols))
    return synth.CsrPattern(m, m, torch.tensor(ro, dtype=torch.int32), torch.tensor(cols, dtype=torch.int32),
                            f"band_far{every}")


@pytest.mark.parametrize("kind", synth.KINDS)
@pytest.mark.parametrize("n", [1, 3, 8, 16, 31, 64, 100, 128])
@pytest.mark.parametrize("case", ["aligned", "ldb_pad", "misaligned", "mixed_tiles"])
def test_b_staging_parity(kind, n, case):
    p = _banded_with_far_entries(4099, 700) if case == "mixed_tiles" else synth.banded(4099, lo=5, hi=9)
    ldb = n + 4 if case == "ldb_pad" else None
    off = 1 if case == "misaligned" else 0
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n, ldb=ldb, b_offset=off)
    chosen, info = run_gpu(p, kind, n, "rowsplit", ro, ci, vd, Bd, Cd)
    assert chosen == "rowsplit"
    # staged when B rows are whole 16-byte granules (TMA bulk copy) of at least 256 bytes
    staged = n % 4 == 0 and n >= 64
    assert info["b_staging"] == (1 if staged else 0)
    if staged:
        assert info["bspan_compact"] >= 0.5
    check(p, kind, n, val, Bh, Cd)


def test_b_staging_plan_decision():
    """Compact (banded) spans are staged; uniform-random columns are not."""
    for pat, want in ((synth.banded(1 << 14), 1), (synth.uniform_rows(1 << 14, 1 << 14, 16, 5), 0)):
        vd = synth.values(pat.nnz, 1, "f32_plus_times").to(DEV)
        op = S.CsrSpmm(pat.row_offsets.to(DEV), pat.col_indices.to(DEV), vd, pat.k)
        assert op.plan(64, "rowsplit") == "rowsplit"
        inf = op.info()
        assert inf["b_staging"] == want, inf
        assert (inf["bspan_compact"] > 0.9) == bool(want)
        op.close()


# ------------------------------------------------------------------------------------------------
# randomized shapes: every path against the oracle on seeded random CSR / n / ld / algo / partition
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("case", range(48))
def test_randomized_parity(case):
    rng = np.random.default_rng(9000 + case)
    m = int(rng.integers(1, 5000))
    k = int(rng.integers(1, 5000))
    shape = case % 4
    if shape == 0:    # uniform short rows
        lens = rng.integers(0, 24, m)
    elif shape == 1:  # skewed: a few long rows, many empty
        lens = np.where(rng.random(m) < 0.6, 0, rng.integers(1, 8, m))
        lens[rng.integers(0, m, 3)] = rng.integers(500, 4000, 3)
    elif shape == 2:  # banded around the diagonal (compact B spans)
        lens = None
    else:             # lognormal
        lens = np.minimum(np.round(rng.lognormal(1.5, 1.0, m)).astype(np.int64), 2000)
    if lens is None:
        w = int(rng.integers(1, 20))
        p = synth.banded(m, lo=w // 2, hi=w - w // 2 - 1)
    else:
        lens = np.minimum(lens, k)
        p = synth.explicit_lengths(m, k, [int(x) for x in lens], seed=case)
    n = int(rng.choice([1, 2, 3, 4, 5, 8, 12, 16, 24, 32, 40, 48, 63, 64, 96, 127, 128]))
    kind = synth.KINDS[case % len(synth.KINDS)]
    algo = ["rowsplit", "merge", "auto"][(case // 4) % 3]
    kw = {}
    if algo == "merge":
        kw = {"partition": ["merge_path", "nonzero_split"][case % 2],
              "items_per_cta": int(rng.choice([256, 512, 1024, 2048, 4096]))}
    ldb = n + int(rng.choice([0, 0, 4, 7])) if case % 5 else None
    ldc = n + int(rng.choice([0, 3])) if case % 3 else None
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n, seed=case, ldb=ldb, ldc=ldc)
    run_gpu(p, kind, n, algo, ro, ci, vd, Bd, Cd, **kw)
    check(p, kind, n, val, Bh, Cd)


# ------------------------------------------------------------------------------------------------
# CSR arrays that are views at arbitrary 4-byte offsets (row blocks sliced out of a larger matrix, as
# the multi-GPU partition does): the TMA staging must align by address, and values whose 16-byte
# phase differs from the column indices' are copied by the producer warp
# ------------------------------------------------------------------------------------------------
def _offset_view(t, off):
    buf = torch.empty(t.numel() + 4, dtype=t.dtype, device=DEV)
    buf[off:off + t.numel()] = t
    return buf[off:off + t.numel()]


@pytest.mark.parametrize("offs", [(0, 1, 1), (0, 2, 2), (0, 3, 3), (1, 1, 2), (3, 2, 0), (2, 0, 3)])
@pytest.mark.parametrize("algo", ["rowsplit", "merge"])
@pytest.mark.parametrize("pat", ["banded", "lognormal"])
@pytest.mark.parametrize("kind", ["f32_plus_times", "i32_min_plus"])
def test_misaligned_csr_views(offs, algo, pat, kind):
    p = synth.banded(3001) if pat == "banded" else synth.lognormal_rows(3001, 2000, 7.92, 19)
    n = 64
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
    o_ro, o_ci, o_v = offs
    ro2, ci2, vd2 = _offset_view(ro, o_ro), _offset_view(ci, o_ci), _offset_view(vd, o_v)
    assert ci2.data_ptr() % 16 == 4 * o_ci
    run_gpu(p, kind, n, algo, ro2, ci2, vd2, Bd, Cd)
    check(p, kind, n, val, Bh, Cd)


def test_row_block_slices_match_full_matrix():
    """The multi-GPU local step: row blocks sliced (views, offsets not multiples of 4) out of one CSR,
    each multiplied on its own, reassemble C of the whole matrix bit-exactly for an exact semiring."""
    from paper_1803_08601_b200 import dist as D
    p = synth.rmat(13, 8, 21)
    kind, n = "i32_plus_times", 48
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
    run_gpu(p, kind, n, "auto", ro, ci, vd, Bd, Cd)
    full = Cd.cpu()
    for parts, mode in ((3, 0), (5, 1), (8, 1)):
        bounds = D.partition_rows(p.row_offsets, parts, mode)
        for r in range(parts):
            r0, r1 = bounds[r], bounds[r + 1]
            bro, bci, bvd = D.slice_rows(ro, ci, vd, r0, r1)
            for algo in ("rowsplit", "merge"):
                op = S.CsrSpmm(bro, bci, bvd, p.k)
                op.plan(n, algo, "plus_times")
                C = op.execute(Bd)
                torch.cuda.synchronize()
                op.close()
                assert torch.equal(C.cpu(), full[r0:r1]), (parts, mode, r, algo)


# ------------------------------------------------------------------------------------------------
# BASELINE configs 1 and 2 at full size, EVERY row against the oracle (SURVEY.md §8(d) parity
# coverage), in the launch configuration bench.py times (AUTO) and with each kernel forced
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("cfg", [1, 2])
@pytest.mark.parametrize("algo", ["auto", "rowsplit", "merge"])
def test_full_size_configs_every_row(cfg, algo):
    p = synth.config_pattern(cfg, device=DEV).to("cpu")
    kind, n = "f32_plus_times", 64
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n, seed=synth.STRUCT_SEED + cfg)
    run_gpu(p, kind, n, algo, ro, ci, vd, Bd, Cd)
    check(p, kind, n, val, Bh, Cd)


def test_config4_rmat26_sampled_rows():
    """BASELINE configs[4] (R-MAT scale 26, ~1.06e9 nonzeros, n = 64) in the bench launch configuration:
    the 1,024 longest rows, the rows around every merge-CTA boundary of a deterministic subset, and 2^20
    seeded random rows, against the oracle (SURVEY.md §8(d) config 5 sample)."""
    p = synth.config_pattern(4, device=DEV)
    kind, n = "f32_plus_times", 64
    seed = synth.STRUCT_SEED + 4
    vd = synth.values(p.nnz, seed + 100, kind, device=DEV)
    Bd = synth.dense(p.k, n, seed + 200, kind, device=DEV)
    Cd = torch.full((p.m, n), float("nan"), device=DEV)
    op = S.CsrSpmm(p.row_offsets, p.col_indices, vd, p.k)
    chosen = op.plan(n, "auto")
    info = op.info()
    op.execute(Bd, Cd)
    torch.cuda.synchronize()
    op.close()
    assert chosen == "merge" and not torch.isnan(Cd).any()
    lens = (p.row_offsets[1:] - p.row_offsets[:-1]).to(torch.int64)
    longest = torch.topk(lens, 1024).indices.cpu()
    g = torch.Generator().manual_seed(4)
    rand = torch.randint(0, p.m, (1 << 20,), generator=g)
    # rows at merge-path CTA boundaries (items_per_cta = 2048): diagonal c*2048 -> row ~ searchsorted
    items = info["items_per_cta"]
    diag = torch.arange(0, p.m + p.nnz, items * 997, dtype=torch.int64)
    ro64 = p.row_offsets.to(torch.int64).cpu()
    brow = torch.searchsorted(ro64 + torch.arange(p.m + 1), diag).clamp(0, p.m - 1)
    rows = torch.unique(torch.cat([longest, rand, brow, (brow + 1).clamp(max=p.m - 1), (brow - 1).clamp(min=0)]))
    pc = p.to("cpu")
    Cref, bound = oracle.spmm(kind, p.m, p.k, n, pc.row_offsets, pc.col_indices, vd.cpu(), Bd.cpu(), rows=rows.numpy())
    C = Cd.cpu().numpy()[rows.numpy()]
    ok, worst, idx = oracle.check_f32(C, Cref, bound, TOL)
    assert ok, f"worst |err|/bound {worst} at {idx}"


# ------------------------------------------------------------------------------------------------
# merge workers: whole warp (k_merge_w) vs lane-folded slots (k_merge_f, n <= 16), static tasks vs
# the task queue (tasks_per_warp > 1)
# ------------------------------------------------------------------------------------------------
def _worker_patterns():
    return {"rmat12": synth.rmat(12, 16, 99), "lognormal": synth.lognormal_rows(3000, 2000, 7.92, 17),
            "many_empty_rows": family("many_empty_rows"), "giant_row_plus_singletons": family("giant_row_plus_singletons"),
            "leading_trailing_empty": family("leading_trailing_empty"), "unsorted_duplicates": family("unsorted_duplicates")}


_WP = {}


@pytest.mark.parametrize("pat", ["rmat12", "lognormal", "many_empty_rows", "giant_row_plus_singletons",
                                 "leading_trailing_empty", "unsorted_duplicates"])
@pytest.mark.parametrize("kind", synth.KINDS)
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 6, 8, 10, 12, 13, 14, 16])
@pytest.mark.parametrize("worker,tpw", [("folded", 1), ("folded", 4), ("warp", 4)])
def test_merge_worker_parity(pat, kind, n, worker, tpw):
    if not _WP:
        _WP.update(_worker_patterns())
    p = _WP[pat]
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
    _, info = run_gpu(p, kind, n, "merge", ro, ci, vd, Bd, Cd, merge_worker=worker, tasks_per_warp=tpw)
    assert (info["merge_worker_lanes"] < 32) == (worker == "folded")
    check(p, kind, n, val, Bh, Cd)


@pytest.mark.parametrize("partition", ["merge_path", "nonzero_split"])
@pytest.mark.parametrize("items", [32, 96, 256, 2048])
@pytest.mark.parametrize("kind", ["f32_plus_times", "i32_plus_times", "f32_min_plus"])
@pytest.mark.parametrize("n", [1, 4, 16])
def test_folded_merge_partitions_and_task_sizes(partition, items, kind, n):
    # tasks shorter than a chunk, tasks that cut long rows, both partitions
    p = synth.lognormal_rows(3000, 2000, 7.92, 17)
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
    run_gpu(p, kind, n, "merge", ro, ci, vd, Bd, Cd, partition=partition, items_per_cta=items, merge_worker="folded")
    check(p, kind, n, val, Bh, Cd)


@pytest.mark.parametrize("kind", synth.KINDS)
def test_folded_merge_padding_and_misalignment(kind):
    """ldb/ldc padding (poisoned) and a misaligned B base: the folded kernel's scalar path (VEC = 1,
    G up to 16 lanes per slot) and its float2 path on 8-byte aligned rows (VEC = 2)."""
    p = synth.rmat(11, 8, 41)
    for n, ldb, ldc, off in ((16, 16, 16, 1), (16, 20, 17, 0), (12, 12, 12, 3), (9, 11, 10, 0), (1, 3, 2, 1),
                             (8, 8, 8, 2), (4, 4, 4, 1), (2, 6, 4, 2), (10, 12, 10, 0), (6, 6, 8, 2)):
        val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n, ldb=ldb, ldc=ldc, b_offset=off)
        run_gpu(p, kind, n, "merge", ro, ci, vd, Bd, Cd, merge_worker="folded")
        check(p, kind, n, val, Bh, Cd)


def test_merge_workers_bit_identical_in_exact_semirings():
    p = synth.rmat(13, 8, 5)
    for kind in ("i32_plus_times", "i32_min_plus", "f32_min_plus"):
        for n in (1, 4, 16):
            outs = []
            for kw in ({"merge_worker": "warp"}, {"merge_worker": "folded"}, {"merge_worker": "folded", "tasks_per_warp": 8},
                       {"merge_worker": "folded", "partition": "nonzero_split"}, {"merge_worker": "folded", "items_per_cta": 64}):
                val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
                run_gpu(p, kind, n, "merge", ro, ci, vd, Bd, Cd, **kw)
                outs.append(Cd.cpu())
            val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
            run_gpu(p, kind, n, "rowsplit", ro, ci, vd, Bd, Cd)
            outs.append(Cd.cpu())
            for o in outs[1:]:
                assert torch.equal(o, outs[0])


@pytest.mark.parametrize("worker", ["warp", "folded"])
def test_merge_task_queue_rezeroed_every_execute(worker):
    # tasks from the queue: a second execute on the SAME op and workspace (C re-poisoned) must redo
    # every task, so the partition kernel must have reset the queue
    p = synth.rmat(12, 16, 99)
    kind, n = "f32_plus_times", 8
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
    op = S.CsrSpmm(ro, ci, vd, p.k)
    op.plan(n, "merge", merge_worker=worker, tasks_per_warp=4)
    for _ in range(2):
        Cd.fill_(float("nan"))
        op.execute(Bd, Cd)
        torch.cuda.synchronize()
        check(p, kind, n, val, Bh, Cd)
    op.close()


def test_folded_merge_rejects_wide_b():
    p = synth.uniform_rows(100, 100, 4, 2)
    vd = synth.values(p.nnz, 1, "f32_plus_times").to(DEV)
    op = S.CsrSpmm(p.row_offsets.to(DEV), p.col_indices.to(DEV), vd, p.k)
    with pytest.raises(S.SpmmError) as e:
        op.plan(17, "merge", merge_worker="folded")
    assert e.value.status == S.SPMM_ERR_UNSUPPORTED
    op.close()


# ------------------------------------------------------------------------------------------------
# execute epilogue (spmm_csr_execute_ex): accumulate, peer copies of C; column split (NEXT-1/3 set-up)
# ------------------------------------------------------------------------------------------------
def _combine_ref(kind, C0, ref):
    if kind.endswith("min_plus"):
        return np.minimum(C0, ref)
    if kind == "i32_plus_times":
        return (C0.astype(np.int64) + ref.astype(np.int64)).astype(np.uint32).astype(np.int32)
    return C0.astype(np.float64) + ref


@pytest.mark.parametrize("kind", synth.KINDS)
@pytest.mark.parametrize("algo,worker", [("rowsplit", "auto"), ("merge", "warp"), ("merge", "folded")])
@pytest.mark.parametrize("n", [4, 16, 64])
def test_execute_accumulate_and_peers(kind, algo, worker, n):
    if worker == "folded" and n > 16:
        pytest.skip("folded merge is for n <= 16")
    p = synth.lognormal_rows(2500, 1800, 7.92, 23)  # ragged rows with empty rows, several tasks
    val, Bh, ro, ci, vd, Bd, _ = make_inputs(p, kind, n)
    C0 = synth.dense(p.m, n, 31, kind)
    Cd = C0.to(DEV).clone()
    off = 37  # this C is rows [37, 37 + m) of the peer copies
    peers = [torch.full((p.m + 50, n), -7, dtype=C0.dtype, device=DEV) for _ in range(3)]
    sr = "plus_times" if kind.endswith("plus_times") else "min_plus"
    op = S.CsrSpmm(ro, ci, vd, p.k)
    op.plan(n, algo, sr, merge_worker=worker)
    op.execute(Bd, Cd, accumulate=True, peers=[t.data_ptr() for t in peers], peer_row_offset=off)
    torch.cuda.synchronize()
    op.close()
    ref = oracle.spmm(kind, p.m, p.k, n, p.row_offsets, p.col_indices, val, Bh)
    C = Cd.cpu().numpy()
    if kind == "f32_plus_times":
        want = _combine_ref(kind, C0.numpy(), ref[0])
        err = np.abs(C.astype(np.float64) - want)
        assert (err <= 1e-5 * ref[1] + 2.0 ** -22 * np.abs(want) + 1e-30).all(), float(err.max())
    else:
        assert np.array_equal(C, _combine_ref(kind, C0.numpy(), ref))
    for t in peers:  # the peer copies hold the final rows, bit for bit; rows outside are untouched
        tc = t.cpu()
        assert torch.equal(tc[off:off + p.m], Cd.cpu())
        assert (tc[:off] == -7).all() and (tc[off + p.m:] == -7).all()


def test_execute_ex_argument_errors():
    p = synth.uniform_rows(100, 100, 4, 2)
    vd = synth.values(p.nnz, 1, "f32_plus_times").to(DEV)
    op = S.CsrSpmm(p.row_offsets.to(DEV), p.col_indices.to(DEV), vd, p.k)
    op.plan(8, "merge")
    B = torch.zeros(100, 8, device=DEV)
    C = torch.zeros(100, 8, device=DEV)
    D = torch.zeros(200, 8, device=DEV)
    args = (op._h, B.data_ptr(), 8, C.data_ptr(), 8, 8, op.workspace.data_ptr(), op.workspace.numel())

    def ex(**f):
        o = S.spmm_exec_opts()
        for k, v in f.items():
            if k == "peer_C":
                for i, x in enumerate(v):
                    o.peer_C[i] = x
            else:
                setattr(o, k, v)
        return S.spmm_csr_execute_ex(*args, o)
    assert ex(accumulate=2) == S.SPMM_ERR_INVALID_ARG
    assert ex(num_peers=8, peer_ldc=8) == S.SPMM_ERR_INVALID_ARG
    assert ex(num_peers=1, peer_ldc=9, peer_C=[D.data_ptr()]) == S.SPMM_ERR_INVALID_ARG
    assert ex(num_peers=1, peer_ldc=8) == S.SPMM_ERR_NULL_POINTER
    assert ex(num_peers=1, peer_ldc=8, peer_C=[D.data_ptr() + 4]) == S.SPMM_ERR_INVALID_ARG
    assert ex(num_peers=1, peer_ldc=8, peer_row_offset=-1, peer_C=[D.data_ptr()]) == S.SPMM_ERR_INVALID_ARG
    assert ex(num_peers=1, peer_ldc=8, peer_row_offset=100, peer_C=[D.data_ptr()]) == S.SPMM_OK
    torch.cuda.synchronize()
    assert torch.equal(D[100:].cpu(), C.cpu())
    op.close()


@pytest.mark.parametrize("pat", ["rmat12", "unsorted_duplicates", "all_empty", "lognormal"])
def test_split_columns_kernel(pat):
    from paper_1803_08601_b200 import dist as D
    p = synth.lognormal_rows(3000, 2000, 7.92, 17) if pat == "lognormal" else family(pat)
    val = synth.values(p.nnz, 3, "i32_plus_times")
    ro, col = p.row_offsets.numpy(), p.col_indices.numpy()
    for c0, c1 in ((0, p.k // 3), (p.k // 3, 2 * p.k // 3), (0, p.k), (5, 5)):
        (ri, ci_, vi), (rx, cx, vx) = D.split_columns_cuda(p.row_offsets.to(DEV), p.col_indices.to(DEV), val.to(DEV),
                                                           c0, c1)
        ri, ci_, vi, rx, cx, vx = (t.cpu().numpy() for t in (ri, ci_, vi, rx, cx, vx))
        vn = val.numpy()
        for r in range(p.m):
            c = col[ro[r]:ro[r + 1]]
            v = vn[ro[r]:ro[r + 1]]
            ins = (c >= c0) & (c < c1)
            assert np.array_equal(ci_[ri[r]:ri[r + 1]], c[ins] - c0) and np.array_equal(vi[ri[r]:ri[r + 1]], v[ins])
            assert np.array_equal(cx[rx[r]:rx[r + 1]], c[~ins]) and np.array_equal(vx[rx[r]:rx[r + 1]], v[~ins])


# ------------------------------------------------------------------------------------------------
# A/B-tiled kernel (NEXT-4): dense-ish rows, B streamed through shared memory in column blocks
# ------------------------------------------------------------------------------------------------
@pytest.mark.parametrize("kind", synth.KINDS)
@pytest.mark.parametrize("n", [32, 36, 64, 96, 128])
def test_tiled_parity(kind, n):
    # rows of 0 / short / very long lengths (many B blocks per row, blocks with no entries)
    lens = [0, 1, 7, 300, 2500, 0, 64] * 40 + [4000, 3]
    p = synth.explicit_lengths(len(lens), 9000, lens, seed=9)
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
    chosen, info = run_gpu(p, kind, n, "tiled", ro, ci, vd, Bd, Cd)
    assert chosen == "tiled" and info["launches_per_execute"] == 1
    check(p, kind, n, val, Bh, Cd)


@pytest.mark.parametrize("kind", ["f32_plus_times", "i32_min_plus"])
def test_tiled_padding_misalignment_and_epilogue(kind):
    p = synth.uniform_rows(700, 3000, 400, 5)
    for n, ldb, ldc, off in ((64, 70, 68, 0), (64, 64, 64, 1), (32, 33, 35, 3), (128, 128, 131, 2)):
        val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n, ldb=ldb, ldc=ldc, b_offset=off)
        run_gpu(p, kind, n, "tiled", ro, ci, vd, Bd, Cd)
        check(p, kind, n, val, Bh, Cd)
    # accumulate + a peer copy
    n = 64
    val, Bh, ro, ci, vd, Bd, _ = make_inputs(p, kind, n)
    C0 = synth.dense(p.m, n, 41, kind)
    Cd = C0.to(DEV).clone()
    peer = torch.zeros(p.m + 5, n, dtype=C0.dtype, device=DEV)
    op = S.CsrSpmm(ro, ci, vd, p.k)
    op.plan(n, "tiled", "plus_times" if kind.endswith("plus_times") else "min_plus")
    op.execute(Bd, Cd, accumulate=True, peers=[peer.data_ptr()], peer_row_offset=5)
    torch.cuda.synchronize()
    op.close()
    ref = oracle.spmm(kind, p.m, p.k, n, p.row_offsets, p.col_indices, val, Bh)
    if kind == "f32_plus_times":
        want = _combine_ref(kind, C0.numpy(), ref[0])
        err = np.abs(Cd.cpu().numpy().astype(np.float64) - want)
        assert (err <= 1e-5 * ref[1] + 2.0 ** -22 * np.abs(want) + 1e-30).all()
    else:
        assert np.array_equal(Cd.cpu().numpy(), _combine_ref(kind, C0.numpy(), ref))
    assert torch.equal(peer[5:].cpu(), Cd.cpu())


def test_tiled_bit_identical_and_preconditions():
    p = synth.uniform_rows(900, 5000, 600, 8)
    for kind in ("i32_plus_times", "f32_min_plus"):
        outs = []
        for algo in ("tiled", "merge", "rowsplit"):
            val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, 64)
            run_gpu(p, kind, 64, algo, ro, ci, vd, Bd, Cd)
            outs.append(Cd.cpu())
        assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    vd = synth.values(p.nnz, 1, "f32_plus_times").to(DEV)
    op = S.CsrSpmm(p.row_offsets.to(DEV), p.col_indices.to(DEV), vd, p.k)
    for bad_n in (30, 16, 132):
        with pytest.raises(S.SpmmError) as e:
            op.plan(bad_n, "tiled")
        assert e.value.status == S.SPMM_ERR_UNSUPPORTED
    op.close()
    u = family("unsorted_duplicates")  # columns not sorted within rows: tiled must refuse
    vu = synth.values(u.nnz, 1, "f32_plus_times").to(DEV)
    op = S.CsrSpmm(u.row_offsets.to(DEV), u.col_indices.to(DEV), vu, u.k)
    with pytest.raises(S.SpmmError) as e:
        op.plan(64, "tiled")
    assert e.value.status == S.SPMM_ERR_UNSUPPORTED
    op.close()


@pytest.mark.parametrize("algo", ["rowsplit", "merge", "tiled"])
def test_execute_is_cuda_graph_capturable(algo):
    """execute() enqueues only kernels / memsets on the given stream (no host sync, no allocation), so a
    planned SpMM can be captured once in a CUDA graph and replayed on new B contents."""
    p = synth.lognormal_rows(3000, 2000, 7.92, 17) if algo != "tiled" else synth.uniform_rows(800, 3000, 300, 4)
    kind, n = "f32_plus_times", 64
    val, Bh, ro, ci, vd, Bd, Cd = make_inputs(p, kind, n)
    op = S.CsrSpmm(ro, ci, vd, p.k)
    op.plan(n, algo)
    op.execute(Bd, Cd)  # first launch outside the capture (kernel attributes, occupancy caches)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        op.execute(Bd, Cd)
    for seed in (301, 302):
        Bh2 = synth.dense(p.k, n, seed, kind)
        Bd.copy_(Bh2.to(DEV))
        Cd.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        check(p, kind, n, val, Bh2, Cd)
    op.close()


@pytest.mark.parametrize("kind", synth.KINDS)
@pytest.mark.parametrize("algo", ["auto", "rowsplit", "merge"])
def test_multiply_host_buffers(kind, algo):
    """spmm_csr_multiply_host: the whole path behind one C call on host buffers (pinned and pageable),
    padding columns of the host C untouched."""
    p = synth.lognormal_rows(3000, 2000, 7.92, 17)
    n, ldb, ldc = 33, 37, 40
    val = synth.values(p.nnz, 311, kind)
    Bh = synth.dense(p.k, n, 312, kind, ld=ldb)
    poison = float("nan") if kind.startswith("f32") else -(2**31)
    for pinned in (True, False):
        Ch = torch.full((p.m, ldc), poison, dtype=Bh.dtype)
        args = [p.row_offsets.contiguous(), p.col_indices.contiguous(), val.contiguous(), Bh, Ch]
        if pinned:
            args = [t.pin_memory() for t in args]
        sr = "plus_times" if kind.endswith("plus_times") else "min_plus"
        st = S.spmm_csr_multiply_host(p.m, p.k, p.nnz, *[a.data_ptr() for a in args[:3]], S._dtype_code(val),
                                      args[3].data_ptr(), ldb, args[4].data_ptr(), ldc, n, S.ALGOS[algo],
                                      S.SEMIRINGS[sr], S.SPMM_HOST_SYNC, None)
        assert st == S.SPMM_OK
        check(p, kind, n, val, Bh, args[4])
    C2 = S.multiply_host(p.row_offsets, p.col_indices, val, p.k, Bh[:, :n].contiguous(), algo=algo,
                         semiring="plus_times" if kind.endswith("plus_times") else "min_plus")
    check(p, kind, n, val, Bh, C2)
