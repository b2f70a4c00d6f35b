"""Seeded synthetic inputs for the CSR SpMM hot path (shared by the CUDA path, the oracle and the bench).

This module holds NONE of the method's arithmetic: it only draws sparsity patterns and values.
Every random number comes from a counter-based 32-bit hash evaluated with exact int64 torch ops,
so the same (seed, stream, index) gives bit-identical matrices on CPU and on CUDA.  That lets the
bench build R-MAT 22 on the GPU in milliseconds while the oracle sees the very same matrix on the host.

Workload shapes follow the paper and SURVEY.md §8(d):
  * uniform fixed-length rows: "making a fixed percentage of elements in each row nonzero by sampling
    indices ... without replacement" (§6 / Fig. 7);
  * banded (circulant band of 16): the regular long-row regime (§5.2);
  * R-MAT (Graph500 a,b,c,d = .57,.19,.19,.05): the scale-free end of the corpus, "small-degree
    large-diameter (road network) to scale-free";
  * aspect matrices: dense rows stored as CSR, Fig. 1 / Fig. 4;
  * lognormal row lengths with the corpus means 7.92 and 62.5.
All generators emit canonical CSR: int32 row_offsets[m+1], int32 col_indices[nnz] sorted and unique
within each row (SURVEY.md §8(c) ambiguity 12).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

M32 = 0xFFFFFFFF

# semiring/dtype "kinds" used across tests and bench
KINDS = ("f32_plus_times", "i32_plus_times", "f32_min_plus", "i32_min_plus")


# ----------------------------------------------------------------------------------------------
# counter-based hash (Wellons' lowbias32), exact in int64 on any device
# ----------------------------------------------------------------------------------------------
def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for x in [0, 2^32) held in int64, with no intermediate above 2^49."""
    lo = x & 0xFFFF
    hi = x >> 16
    return (lo * c + (((hi * c) & 0xFFFF) << 16)) & M32


def _hash32(x: torch.Tensor) -> torch.Tensor:
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _hash32_int(x: int) -> int:
    x &= M32
    x ^= x >> 16
    x = (x * 0x7FEB352D) & M32
    x ^= x >> 15
    x = (x * 0x846CA68B) & M32
    x ^= x >> 16
    return x


def counter_u32(seed: int, stream: int, idx: torch.Tensor) -> torch.Tensor:
    """Uniform 32-bit integers (held in int64) for counters `idx` (int64 >= 0)."""
    s1 = _hash32_int(_hash32_int(seed) ^ (stream * 0x9E3779B1))
    s2 = _hash32_int(s1 ^ 0x5BD1E995)
    h = _hash32((idx & M32) ^ s1)
    h = _hash32(h ^ (idx >> 32) ^ s2)
    return h


def _arange(n: int, device) -> torch.Tensor:
    return torch.arange(n, dtype=torch.int64, device=device)


# ----------------------------------------------------------------------------------------------
# CSR container
# ----------------------------------------------------------------------------------------------
@dataclass
class CsrPattern:
    m: int
    k: int
    row_offsets: torch.Tensor  # int32 [m+1]
    col_indices: torch.Tensor  # int32 [nnz]
    name: str = ""

    @property
    def nnz(self) -> int:
        return int(self.col_indices.numel())

    def to(self, device) -> "CsrPattern":
        return CsrPattern(self.m, self.k, self.row_offsets.to(device), self.col_indices.to(device), self.name)


def _csr_from_sorted_keys(keys: torch.Tensor, m: int, k: int, name: str) -> CsrPattern:
    """keys = row*k + col, sorted ascending and unique."""
    rows = keys // k
    cols = (keys - rows * k).to(torch.int32)
    counts = torch.bincount(rows, minlength=m)
    ro = torch.zeros(m + 1, dtype=torch.int64, device=keys.device)
    ro[1:] = torch.cumsum(counts, 0)
    assert int(ro[-1]) < 2**31, "int32 offsets (SURVEY.md §8(c) ambiguity 13)"
    return CsrPattern(m, k, ro.to(torch.int32), cols.contiguous(), name)


def from_rows(m: int, k: int, rows: list[list[int]], name: str = "explicit") -> CsrPattern:
    """Small hand-built pattern; each row's columns are sorted + deduplicated."""
    assert len(rows) == m
    ro = [0]
    cols: list[int] = []
    for r in rows:
        rr = sorted(set(r))
        assert all(0 <= c < k for c in rr)
        cols.extend(rr)
        ro.append(len(cols))
    return CsrPattern(m, k, torch.tensor(ro, dtype=torch.int32), torch.tensor(cols, dtype=torch.int32), name)


def from_lengths_unsorted(m: int, k: int, lengths: list[int], seed: int, allow_dups: bool = False,
                          name: str = "lengths", device="cpu") -> CsrPattern:
    """Rows with exactly the given lengths (distinct columns drawn without replacement).

    With allow_dups=True the columns are drawn WITH replacement and left unsorted: a non-canonical
    CSR that the kernels must still handle (SURVEY.md §8(c) ambiguity 12)."""
    assert len(lengths) == m
    if not allow_dups:
        assert all(0 <= L <= k for L in lengths)
    ro = torch.zeros(m + 1, dtype=torch.int64)
    ro[1:] = torch.cumsum(torch.tensor(lengths, dtype=torch.int64), 0)
    nnz = int(ro[-1])
    if allow_dups:
        h = counter_u32(seed, 7, _arange(nnz, "cpu"))
        cols = ((h * k) >> 32).to(torch.int32)
        return CsrPattern(m, k, ro.to(torch.int32).to(device), cols.to(device), name)
    out = []
    for i, L in enumerate(lengths):
        if L == 0:
            continue
        if L * 2 >= k:  # dense-ish row: random permutation prefix via hash keys
            keys = counter_u32(seed, 8, i * k + _arange(k, "cpu"))
            sel = torch.argsort(keys * k + _arange(k, "cpu"))[:L]
            out.append(torch.sort(sel)[0])
        else:  # draw candidates in batches, keep first occurrences in draw order
            got: list[int] = []
            seen = set()
            t = 0
            while len(got) < L:
                cand = ((counter_u32(seed, 9, i * 1_000_003 + t + _arange(4 * L, "cpu")) * k) >> 32).tolist()
                t += 4 * L
                for c in cand:
                    if c not in seen:
                        seen.add(c)
                        got.append(c)
                        if len(got) == L:
                            break
            out.append(torch.tensor(sorted(got), dtype=torch.int64))
    cols = torch.cat(out).to(torch.int32) if out else torch.zeros(0, dtype=torch.int32)
    return CsrPattern(m, k, ro.to(torch.int32).to(device), cols.to(device), name)


# ----------------------------------------------------------------------------------------------
# structure generators
# ----------------------------------------------------------------------------------------------
def banded(m: int, lo: int = 8, hi: int = 7, device="cpu", row_begin: int = 0, row_end: int | None = None
           ) -> CsrPattern:
    """Circulant band: row i has columns {(i+o) mod m : o in [-lo, hi]}, sorted (SURVEY.md §8(d) cfg 2).
    row_begin/row_end select a row block (rows keep their global column indices; k stays m)."""
    w = lo + hi + 1
    assert w <= m
    row_end = m if row_end is None else row_end
    i = _arange(row_end - row_begin, device) + row_begin
    offs = torch.arange(-lo, hi + 1, dtype=torch.int64, device=device)
    cols = torch.remainder(i[:, None] + offs[None, :], m)
    cols = torch.sort(cols, dim=1)[0]
    rows = row_end - row_begin
    ro = (_arange(rows + 1, device) * w).to(torch.int32)
    return CsrPattern(rows, m, ro, cols.reshape(-1).to(torch.int32).contiguous(), f"banded_m{m}_w{w}")


def uniform_rows(m: int, k: int, d: int, seed: int, device="cpu") -> CsrPattern:
    """Each row has exactly d distinct columns drawn uniformly without replacement."""
    assert 0 <= d <= k
    if d == 0 or m == 0:
        return CsrPattern(m, k, torch.zeros(m + 1, dtype=torch.int32, device=device),
                          torch.zeros(0, dtype=torch.int32, device=device), f"uniform_m{m}_d{d}")
    if 4 * d >= k:  # dense-ish: rank random keys over all k columns
        out = []
        chunk = max(1, (1 << 24) // k)
        for r0 in range(0, m, chunk):
            r1 = min(m, r0 + chunk)
            idx = (_arange(r1 - r0, device)[:, None] + r0) * k + _arange(k, device)[None, :]
            keys = counter_u32(seed, 1, idx) * k + _arange(k, device)[None, :]
            sel = torch.topk(keys, d, dim=1, largest=False, sorted=False)[1]
            out.append(torch.sort(sel, dim=1)[0])
        cols = torch.cat(out, 0)
    else:
        c = 2 * d + 8
        out = []
        chunk = max(1, (1 << 24) // c)
        for r0 in range(0, m, chunk):
            r1 = min(m, r0 + chunk)
            rows = r1 - r0
            idx = (_arange(rows, device)[:, None] + r0) * c + _arange(c, device)[None, :]
            cand = (counter_u32(seed, 2, idx) * k) >> 32
            sv, si = torch.sort(cand, dim=1, stable=True)
            dup_sorted = torch.zeros_like(sv, dtype=torch.bool)
            dup_sorted[:, 1:] = sv[:, 1:] == sv[:, :-1]
            dup = torch.empty_like(dup_sorted)
            dup.scatter_(1, si, dup_sorted)
            keep = ~dup
            rank = torch.cumsum(keep.to(torch.int32), dim=1)
            sel = keep & (rank <= d)
            assert bool((sel.sum(1) == d).all()), "too many duplicate draws; raise candidate count"
            cols_c = cand[sel].view(rows, d)
            out.append(torch.sort(cols_c, dim=1)[0])
        cols = torch.cat(out, 0)
    ro = (_arange(m + 1, device) * d).to(torch.int32)
    return CsrPattern(m, k, ro, cols.reshape(-1).to(torch.int32).contiguous(), f"uniform_m{m}_k{k}_d{d}")


def rmat(scale: int, edge_factor: int, seed: int, abcd=(0.57, 0.19, 0.19, 0.05), device="cpu",
         chunk_edges: int = 1 << 26) -> CsrPattern:
    """Graph500-style R-MAT: 2^scale vertices, edge_factor*2^scale generated edges, no permutation,
    self-loops kept, duplicates merged (SURVEY.md §8(d) cfg 3/5).  Quadrant choice per level is an
    integer compare of a 32-bit counter hash against floor(p*2^32), so CPU and GPU agree exactly."""
    a, b, c, _ = abcd
    n = 1 << scale
    E = edge_factor * n
    ta = int(a * 2**32)
    tab = int((a + b) * 2**32)
    tabc = int((a + b + c) * 2**32)
    uniq = []
    for e0 in range(0, E, chunk_edges):
        e1 = min(E, e0 + chunk_edges)
        e = _arange(e1 - e0, device) + e0
        row = torch.zeros_like(e)
        col = torch.zeros_like(e)
        for lvl in range(scale):
            h = counter_u32(seed, 100 + lvl, e)
            rb = (h >= tab).to(torch.int64)
            cb = (((h >= ta) & (h < tab)) | (h >= tabc)).to(torch.int64)
            row = (row << 1) | rb
            col = (col << 1) | cb
        del e
        uniq.append(torch.unique(row * n + col, sorted=True))
        del row, col
    keys = torch.unique(torch.cat(uniq), sorted=True) if len(uniq) > 1 else uniq[0]
    return _csr_from_sorted_keys(keys, n, n, f"rmat{scale}_ef{edge_factor}")


def aspect(total_nnz: int, m: int, device="cpu") -> CsrPattern:
    """Dense m x (total_nnz/m) matrix stored as CSR (Fig. 1 / Fig. 4 microbenchmark)."""
    assert total_nnz % m == 0
    d = total_nnz // m
    cols = _arange(d, device).repeat(m).to(torch.int32)
    ro = (_arange(m + 1, device) * d).to(torch.int32)
    return CsrPattern(m, d, ro, cols, f"aspect_m{m}_d{d}")


def _lognormal_thresholds(mean: float, sigma: float, lmax: int) -> list[int]:
    """uint32 thresholds t_L = floor(P(len <= L) * 2^32) for a discretised lognormal with the given
    mean (len = round(X), X lognormal).  Computed on the host in Python -> device-independent."""
    mu = math.log(mean) - 0.5 * sigma * sigma
    th = []
    for L in range(lmax):
        x = L + 0.5
        p = 0.5 * (1.0 + math.erf((math.log(x) - mu) / (sigma * math.sqrt(2.0))))
        th.append(min(M32, int(p * 2**32)))
    return th


def lognormal_rows(m: int, k: int, mean: float, seed: int, sigma: float = 1.0, device="cpu") -> CsrPattern:
    """Row lengths ~ round(lognormal) with the given mean (corpus means 7.92 / 62.5);
    columns drawn uniformly with replacement then merged, so a row may come out slightly shorter."""
    lmax = min(k, int(mean * 200) + 1)
    th = torch.tensor(_lognormal_thresholds(mean, sigma, lmax), dtype=torch.int64, device=device)
    h = counter_u32(seed, 20, _arange(m, device))
    lens = torch.searchsorted(th, h, right=True).clamp_(max=lmax)
    E = int(lens.sum())
    rows = torch.repeat_interleave(_arange(m, device), lens)
    cols = (counter_u32(seed, 21, _arange(E, device)) * k) >> 32
    keys = torch.unique(rows * k + cols, sorted=True)
    return _csr_from_sorted_keys(keys, m, k, f"lognormal_m{m}_mean{mean}")


def explicit_lengths(m: int, k: int, lengths, seed: int = 0, device="cpu", name="lengths") -> CsrPattern:
    return from_lengths_unsorted(m, k, list(lengths), seed, name=name, device=device)


# ----------------------------------------------------------------------------------------------
# values
# ----------------------------------------------------------------------------------------------
def _vals(kind: str, h: torch.Tensor) -> torch.Tensor:
    """Map uniform u32 draws to the value recipe of SURVEY.md §8(d):
    f32 plus-times U[-1,1) (multiples of 2^-23, exact); i32 plus-times U{-4..4};
    f32 min-plus U[1,1000); i32 min-plus U{1..999}."""
    if kind == "f32_plus_times":
        return ((h >> 8) - (1 << 23)).to(torch.float32) * (2.0 ** -23)
    if kind == "i32_plus_times":
        return (torch.remainder(h, 9) - 4).to(torch.int32)
    if kind == "f32_min_plus":
        return (h >> 8).to(torch.float32) * (999.0 / 16777216.0) + 1.0
    if kind == "i32_min_plus":
        return (torch.remainder(h, 999) + 1).to(torch.int32)
    raise ValueError(kind)


def values(nnz: int, seed: int, kind: str, device="cpu", offset: int = 0) -> torch.Tensor:
    """Values of nonzeros offset .. offset+nnz-1 (offset = global position of a row block)."""
    return _vals(kind, counter_u32(seed, 30, _arange(nnz, device) + offset))


def dense(rows: int, n: int, seed: int, kind: str, ld: int | None = None, device="cpu",
          pad_value=None) -> torch.Tensor:
    """rows x ld row-major matrix; columns [n, ld) hold a poison value (NaN / INT32_MIN) so that a
    kernel reading outside [0, n) shows up in parity."""
    ld = n if ld is None else ld
    assert ld >= n
    out = torch.empty(rows, ld, dtype=torch.float32 if kind.startswith("f32") else torch.int32, device=device)
    chunk = max(1, (1 << 26) // max(1, n))
    for r0 in range(0, rows, chunk):
        r1 = min(rows, r0 + chunk)
        idx = (_arange(r1 - r0, device)[:, None] + r0) * n + _arange(n, device)[None, :]
        out[r0:r1, :n] = _vals(kind, counter_u32(seed, 40, idx))
    if ld > n:
        if pad_value is None:
            pad_value = float("nan") if kind.startswith("f32") else -(2**31)
        out[:, n:] = pad_value
    return out


def identity_value(kind: str):
    """Additive identity of the semiring (the value of an empty row, SURVEY.md §8(c) ambiguity 11)."""
    if kind.endswith("plus_times"):
        return 0
    return float("inf") if kind.startswith("f32") else 2**31 - 1


# ----------------------------------------------------------------------------------------------
# BASELINE.json configs
# ----------------------------------------------------------------------------------------------
STRUCT_SEED = 1803


def config_pattern(idx: int, device="cpu", scale: int | None = None) -> CsrPattern:
    """configs[idx] of BASELINE.json (0-based):
    0 tiny uniform m=k=1024, 16/row; 1 banded m=k=2^20, 16/row; 2 R-MAT 22 ef 16; 4 R-MAT 26 ef 16."""
    seed = STRUCT_SEED + idx
    if idx == 0:
        return uniform_rows(1024, 1024, 16, seed, device)
    if idx == 1:
        return banded(1 << 20, device=device)
    if idx == 2:
        return rmat(22 if scale is None else scale, 16, seed, device=device)
    if idx == 4:
        return rmat(26 if scale is None else scale, 16, seed, device=device)
    raise ValueError(idx)


def config4_mix(device="cpu", small: bool = False):
    """The n-sweep matrix mix of SURVEY.md §8(d) cfg 4 (26 matrices).  small=True shrinks every
    matrix ~64x for quick runs."""
    s = 6 if small else 0
    mats = []
    seed = STRUCT_SEED + 3
    M = 1 << (20 - s)
    for d in (1, 2, 4, 8, 9, 10, 12, 16, 32, 64):
        mats.append(uniform_rows(M, M, d, seed + d, device))
    for d in (3, 5, 7, 27):
        lo = d // 2
        mats.append(banded(M, lo, d - lo - 1, device))
    for lm in (10, 12, 14, 16, 18, 20, 22):
        lm2 = lm - s if small else lm
        mats.append(aspect(1 << (24 - s), 1 << max(1, lm2), device))
    for ef in (4, 8, 16, 32):
        mats.append(rmat(20 - s, ef, seed + 50 + ef, device=device))
    for mean in (7.92, 62.5):
        mats.append(lognormal_rows(M, M, mean, seed + 80 + int(mean), device=device))
    return mats
