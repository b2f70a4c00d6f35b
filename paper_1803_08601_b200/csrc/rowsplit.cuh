// rowsplit.cuh -- Algorithm I, row-splitting SpMM (§4.1, Fig. 3, Table 1), sm_100a.
//
// Paper design (K40c): one warp per row (§4.1 decision 1); lanes map to columns of
// row-major B so every B-row gather is coalesced (decision 2); each lane loads one
// (col, val) per 32-nonzero chunk and the warp runs 32 `__shfl` broadcast rounds, each an independent
// B-row load (decision 3; Table 1 "Read B: 0 < L <= 32").
//
// B200 redesign:
//   * a "row group" of G lanes owns one row; G = ceil(n/VEC) rounded to a power of two, so the
//     group's lanes cover the n columns with VEC-wide (float4/float2) gathers; a warp therefore runs
//     S = 32/G rows at once.  n = 64 -> float4, G = 16, two rows per warp; n = 128 -> G = 32 (the
//     paper's warp per row); n = 1 -> G = 1, thread per row (the paper's own suggestion for short rows,
//     PAPER.md:99).  This replaces the paper's 32-column C tiles that re-read A per tile.
//   * chunk = max(G, U) nonzeros: each lane loads K = chunk/G (col, val) pairs (streaming, no L1
//     allocation), then `__shfl_sync(.., width=G)` broadcasts them and U B-row gathers are issued
//     back to back before any FMA (ILP).
//   * no dummy column-0 loads: lanes past the row end are predicated off, so 0*Inf and
//     the min-plus identity are never touched (SURVEY.md §8(c) ambiguity 10).
//   * two interleaved accumulators per column (shorter fp32 dependency chains, smaller error growth).
//   * software pipeline across the rows a group owns: the row offsets two rows ahead and the first
//     A chunk one row ahead are loaded while the current row's B gathers are in flight, so a short
//     row costs one exposed memory round trip instead of three.
//   * a CTA owns a contiguous block of rows, interleaved over its warps, so concurrently running
//     rows share B rows through L1 (banded / locally clustered matrices).
#pragma once
#include "common.cuh"

namespace spmm {

template <typename T, int SR, int VEC, int G, int NV, int U>
__global__ void __launch_bounds__(THREADS)
k_rowsplit(int m, int n, const int* __restrict__ ro, const int* __restrict__ col, const T* __restrict__ val,
           const T* __restrict__ B, long long ldb, T* __restrict__ C, long long ldc, int rounds) {
    using R = Ring<T, SR>;
    constexpr int S = 32 / G;                 // rows per warp at a time
    constexpr int CH = (G > U) ? G : U;       // nonzeros per chunk
    constexpr int K = CH / G;                 // (col,val) pairs per lane per chunk
    constexpr int UU = (CH < U) ? CH : U;     // gathers in flight per batch
    static_assert(G >= 1 && G <= 32 && (32 % G) == 0, "G must divide 32");
    static_assert(CH % UU == 0, "batch must divide chunk");

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int slot = lane / G;
    const int gl = lane - slot * G;
    const int stride = WARPS_PER_CTA * S;     // rows between two rounds of the same group
    const long long rows_per_cta = (long long)stride * rounds;
    const long long cta_row0 = (long long)blockIdx.x * rows_per_cta;
    const long long cta_row_end = min((long long)m, cta_row0 + rows_per_cta);
    long long r = cta_row0 + warp * S + slot;

    // columns of this lane: c = gl*VEC + v*G*VEC + e, v < NV, e < VEC
    bool colok[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) colok[v] = (gl * VEC + v * G * VEC) < n;

    auto load_ro = [&](long long row, int& s, int& e) {
        if (row < cta_row_end) {
            s = ld_stream(ro + row);
            e = ld_stream(ro + row + 1);
        } else {
            s = 0;
            e = 0;
        }
    };
    auto load_chunk = [&](int s, int e, int base, int (&c)[K], unsigned (&a)[K]) {
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
            const int q = s + base + gl + kk * G;
            if (q < e) {
                c[kk] = ld_stream(col + q);
                a[kk] = ld_stream_u(val + q);
            } else {
                c[kk] = 0;
                a[kk] = 0u;
            }
        }
    };

    int s0, e0, s1, e1;
    load_ro(r, s0, e0);
    load_ro(r + stride, s1, e1);
    int c0[K];
    unsigned a0[K];
    load_chunk(s0, e0, 0, c0, a0);

    for (int t = 0; t < rounds; ++t, r += stride) {
        if (cta_row0 + (long long)t * stride >= cta_row_end) break;  // warp-uniform
        const bool active = r < cta_row_end;
        int s2, e2;
        load_ro(r + 2 * stride, s2, e2);
        int c1[K];
        unsigned a1[K];
        load_chunk(s1, e1, 0, c1, a1);

        T acc[2][NV][VEC];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int x = 0; x < VEC; ++x) acc[h][v][x] = R::id();

        const int len = active ? (e0 - s0) : 0;
        const int maxlen = __reduce_max_sync(FULL, len);
        for (int base = 0; base < maxlen; base += CH) {
            int c[K];
            unsigned a[K];
            if (base == 0) {
#pragma unroll
                for (int kk = 0; kk < K; ++kk) { c[kk] = c0[kk]; a[kk] = a0[kk]; }
            } else {
                load_chunk(s0, e0, base, c, a);
            }
            const int cnt = len - base;                 // this group's nonzeros left (may be <= 0)
            const int maxcnt = min(CH, maxlen - base);  // warp-uniform
#pragma unroll
            for (int j0 = 0; j0 < CH; j0 += UU) {
                if (j0 >= maxcnt) break;
                unsigned bv[UU][NV][VEC];
                unsigned av[UU];
#pragma unroll
                for (int u = 0; u < UU; ++u) {
                    const int j = j0 + u;             // nonzero index within the chunk
                    const int kk = j / G;             // which of the lane's pairs
                    const int src = j - kk * G;       // source lane within the group
                    int cj;
                    if (G == 1) {
                        cj = c[kk];
                        av[u] = a[kk];
                    } else {
                        cj = __shfl_sync(FULL, c[kk], src, G);
                        av[u] = __shfl_sync(FULL, a[kk], src, G);
                    }
                    if (j < cnt) {
                        const T* brow = B + (long long)cj * ldb + gl * VEC;
#pragma unroll
                        for (int v = 0; v < NV; ++v)
                            if (colok[v]) ldg_vec<VEC>(bv[u][v], brow + v * G * VEC);
                    }
                }
#pragma unroll
                for (int u = 0; u < UU; ++u) {
                    const int j = j0 + u;
                    if (j < cnt) {
                        const T aval = from_bits<T>(av[u]);
#pragma unroll
                        for (int v = 0; v < NV; ++v)
#pragma unroll
                            for (int x = 0; x < VEC; ++x)
                                acc[u & 1][v][x] = R::mac(acc[u & 1][v][x], aval, from_bits<T>(bv[u][v][x]));
                    }
                }
            }
        }
        if (active) {
            T* crow = C + r * ldc + gl * VEC;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (colok[v]) {
                    unsigned o[VEC];
#pragma unroll
                    for (int x = 0; x < VEC; ++x) o[x] = to_bits<T>(R::add(acc[0][v][x], acc[1][v][x]));
                    st_vec<VEC>(crow + v * G * VEC, o);
                }
            }
        }
        s0 = s1; e0 = e1; s1 = s2; e1 = e2;
#pragma unroll
        for (int kk = 0; kk < K; ++kk) { c0[kk] = c1[kk]; a0[kk] = a1[kk]; }
    }
}

}  // namespace spmm
