// merge.cuh -- Algorithm II, merge-based SpMM (§4.2, Algorithm 1), sm_100a.
//
// Phase 1, PartitionSpmm (Alg. 1 line 2): k_partition writes the merge-path state
//   (row, nonzero) at which every CTA starts.  2-D merge path (Fig. 2(c)): CTA c starts on
//   diagonal c*I of the merge of row-end offsets with nonzero indices (rows first on ties), so every
//   CTA gets I items = rows + nonzeros, which also charges the C write of empty rows.
//   1-D nonzero split (PAPER.md:80, the paper's own choice, :89): CTA c starts at nonzero c*I in the
//   largest row r with ro[r] <= c*I.  One warp per boundary, 32-ary search (~6 dependent probes).
// Phase 2 (Alg. 1 lines 3-23): k_merge.  Per CTA:
//   GlobalToShared (line 5): the CTA's row-end slice and its (col, val) slice are staged into shared
//     memory with coalesced 16-byte loads.
//   Each warp is a "worker": it finds its own equal share of the CTA's items with a second merge-path
//     search in shared memory, then streams them: (col, val) are read from shared memory as warp
//     broadcasts (the paper's 32 `Broadcast` rounds, lines 14-17, without registers new_ind/new_val),
//     U B-row gathers are issued back to back (lanes over columns, float4/float2, line 18), and each
//     row-end item flushes the running row into C (identity for empty rows).  Because every lane of a
//     worker sees the same row id, the paper's valB[32] + PrepareSpmm (CSR->COO, line 21) +
//     ReduceToGlobalSpmm segmented reduction (line 22) collapse into a running accumulator that is
//     written on each row end; this removes the T = 1 register limit.
//   Carry-outs (line 22): a worker whose range ends inside a row keeps its partial;
//     partials whose row is finished inside the same CTA are added into C by warp 0 after a CTA
//     barrier (ascending worker order); the CTA's final open row becomes the CTA's carry-out.
// Phase 3, FixCarryOut (Alg. 1 line 24): k_fixup adds each run of consecutive CTA
//   carry-outs that share a row into C[row], in ascending CTA order (deterministic, no atomics).
// Ownership (SURVEY.md §8(c) ambiguity 20): the worker that consumes a row's end item writes the row;
//   every earlier partial is added afterwards, in order.
#pragma once
#include "common.cuh"

namespace spmm {

// merge-path predicate: row end of row x (at path position x + ro[x+1]) lies before diagonal D
struct MergePred {
    const int* ro;
    long long D;
    __device__ __forceinline__ bool operator()(long long x) const {
        return (long long)ld_stream(ro + x + 1) > D - x - 1;
    }
};
struct NzPred {  // first r with ro[r] > t
    const int* ro;
    long long t;
    __device__ __forceinline__ bool operator()(long long x) const { return (long long)ld_stream(ro + x) > t; }
};

// states[2c] = row, states[2c+1] = nonzero, c in [0, num_ctas]
__global__ void __launch_bounds__(THREADS)
k_partition(const int* __restrict__ ro, int m, int nnz, int items, int mode, int num_ctas, int* __restrict__ states) {
    const int lane = threadIdx.x & 31;
    const long long c = (long long)blockIdx.x * WARPS_PER_CTA + (threadIdx.x >> 5);
    if (c > num_ctas) return;
    long long row, nz;
    if (mode == 0) {
        const long long D = min(c * items, (long long)m + nnz);
        const long long lo = max(0LL, D - nnz), hi = min(D, (long long)m);
        row = warp_search_first(lo, hi, MergePred{ro, D});
        nz = D - row;
    } else {
        if (c == 0) {
            row = 0; nz = 0;
        } else if (c == num_ctas) {
            row = m; nz = nnz;
        } else {
            const long long t = c * items;  // < nnz
            row = warp_search_first(0, (long long)m + 1, NzPred{ro, t}) - 1;
            nz = t;
        }
    }
    if (lane == 0) {
        states[2 * c] = (int)row;
        states[2 * c + 1] = (int)nz;
    }
}

// shared-memory layout of k_merge (bytes, 16-aligned pieces)
__host__ __device__ constexpr size_t merge_smem_bytes(int items, int n, int elem) {
    return (size_t)((items + 4 + 3) / 4 * 4) * 4              // E: row ends, items + 1 (+pad)
           + (size_t)items * 8                                // AV: (col, val bits) pairs
           + (size_t)(WARPS_PER_CTA + 1) * n * elem           // carries of the workers + carry-in
           + (size_t)(WARPS_PER_CTA + 1) * 16                 // carry rows/flags
           + 64;                                              // sub-tile state
}

template <typename T, int SR, int VEC, int NV, int U>
__global__ void __launch_bounds__(THREADS)
k_merge(int m, int n, int nnz, const int* __restrict__ ro, const int* __restrict__ col, const T* __restrict__ val,
        const T* __restrict__ B, long long ldb, T* __restrict__ C, long long ldc, const int* __restrict__ states,
        int items, int* __restrict__ carry_row, int* __restrict__ carry_flag, T* __restrict__ carry_val) {
    using R = Ring<T, SR>;
    extern __shared__ __align__(16) unsigned char smem[];
    int* E = reinterpret_cast<int*>(smem);                                       // ro[rs+1+t]
    int2* AV = reinterpret_cast<int2*>(smem + (size_t)((items + 4 + 3) / 4 * 4) * 4);
    T* Cw = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(AV) + (size_t)items * 8);  // [W+1][n]
    int* Crow = reinterpret_cast<int*>(Cw + (size_t)(WARPS_PER_CTA + 1) * n);     // [W+1]
    int* Cflag = Crow + (WARPS_PER_CTA + 1);                                      // [W+1]
    int* Tst = Cflag + (WARPS_PER_CTA + 1) + 2 * WARPS_PER_CTA;                   // sub-tile end state

    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int cta = blockIdx.x;
    const long long cta_rs = states[2 * cta], cta_zs = states[2 * cta + 1];
    const long long cta_re = states[2 * cta + 2], cta_ze = states[2 * cta + 3];
    const long long L = (cta_re - cta_rs) + (cta_ze - cta_zs);

    bool colok[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) colok[v] = (lane * VEC + v * 32 * VEC) < n;

    // carry-in slot (index WARPS_PER_CTA): running partial of the open row between sub-tiles
    if (threadIdx.x == 0) { Crow[WARPS_PER_CTA] = -1; Cflag[WARPS_PER_CTA] = 0; }

    long long rs = cta_rs, zs = cta_zs;
    for (long long done = 0; done < L; ) {
        const long long Ls = min((long long)items, L - done);
        long long re, ze;
        if (done + Ls == L) {
            re = cta_re; ze = cta_ze;
        } else {  // 1-D split with more items than one tile: find the sub-tile end on the path
            if (warp == 0) {
                const long long D = rs + zs + Ls;
                const long long lo = max(rs, D - cta_ze), hi = min(D - zs, cta_re);
                const long long i = warp_search_first(lo, hi, MergePred{ro, D});
                if (lane == 0) { Tst[0] = (int)i; Tst[1] = (int)(D - i); }
            }
            __syncthreads();
            re = Tst[0]; ze = Tst[1];
        }
        // ---- GlobalToShared (Alg. 1 line 5): row ends of rows rs..min(re, m-1), (col,val) of zs..ze-1
        const int nE = (int)(min(re, (long long)m - 1) - rs + 1);
        const int nA = (int)(ze - zs);
        for (int t = threadIdx.x; t < nE; t += THREADS) E[t] = ld_stream(ro + rs + 1 + t);
        for (int t = threadIdx.x; t < nA; t += THREADS) {
            AV[t] = make_int2(ld_stream(col + zs + t), (int)ld_stream_u(val + zs + t));
        }
        __syncthreads();

        // ---- worker sub-range: equal share of the Ls items, second merge-path search in smem
        const long long per = (Ls + WARPS_PER_CTA - 1) / WARPS_PER_CTA;
        auto search = [&](long long d) -> long long {  // row coordinate of diagonal rs+zs+d
            const long long D = rs + zs + d;
            long long lo = max(rs, D - ze), hi = min(D - zs, re);
            while (lo < hi) {
                const long long mid = (lo + hi) >> 1;
                if ((long long)E[mid - rs] <= D - mid - 1) lo = mid + 1; else hi = mid;
            }
            return lo;
        };
        const long long d0 = min((long long)warp * per, Ls), d1 = min((long long)(warp + 1) * per, Ls);
        const long long ia = search(d0), ja = rs + zs + d0 - ia;
        const long long ib = search(d1), jb = rs + zs + d1 - ib;

        T acc[NV][VEC];
        bool dirty = false;
        if (warp == 0 && Cflag[WARPS_PER_CTA]) {  // continue the previous sub-tile's open row
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int x = 0; x < VEC; ++x) {
                    const int cc = lane * VEC + v * 32 * VEC + x;
                    acc[v][x] = colok[v] ? Cw[WARPS_PER_CTA * n + cc] : R::id();
                }
            dirty = true;
        } else {
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int x = 0; x < VEC; ++x) acc[v][x] = R::id();
        }

        long long r = ia;
        long long q = ja;
        long long e = (r < m) ? (long long)E[r - rs] : 0x7fffffffffffLL;
        auto flush = [&]() {
            T* crow = C + r * ldc + lane * VEC;
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (colok[v]) {
                    unsigned o[VEC];
#pragma unroll
                    for (int x = 0; x < VEC; ++x) o[x] = to_bits<T>(acc[v][x]);
                    st_vec<VEC>(crow + v * 32 * VEC, o);
                }
#pragma unroll
                for (int x = 0; x < VEC; ++x) acc[v][x] = R::id();
            }
            dirty = false;
            ++r;
            e = (r < m) ? (long long)E[r - rs] : 0x7fffffffffffLL;
        };

        while (q < jb) {
            const int cnt = (int)min((long long)U, jb - q);
            unsigned bv[U][NV][VEC];
            unsigned av[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (u < cnt) {
                    const int2 p = AV[q + u - zs];
                    av[u] = (unsigned)p.y;
                    const T* brow = B + (long long)p.x * ldb + lane * VEC;
#pragma unroll
                    for (int v = 0; v < NV; ++v)
                        if (colok[v]) ldg_vec<VEC>(bv[u][v], brow + v * 32 * VEC);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (u < cnt) {
                    const long long qq = q + u;
                    while (e <= qq) flush();  // rows ending before nonzero qq (rows first on ties)
                    const T aval = from_bits<T>(av[u]);
#pragma unroll
                    for (int v = 0; v < NV; ++v)
#pragma unroll
                        for (int x = 0; x < VEC; ++x) acc[v][x] = R::mac(acc[v][x], aval, from_bits<T>(bv[u][v][x]));
                    dirty = true;
                }
            }
            q += cnt;
        }
        while (r < ib) flush();  // remaining row-end items of this worker

        // ---- carry of this worker: partial of row ib (open at its end) -> shared slot
        if (lane == 0) { Crow[warp] = (int)ib; Cflag[warp] = dirty ? 1 : 0; }
        if (dirty) {
#pragma unroll
            for (int v = 0; v < NV; ++v)
#pragma unroll
                for (int x = 0; x < VEC; ++x) {
                    const int cc = lane * VEC + v * 32 * VEC + x;
                    if (colok[v]) Cw[warp * n + cc] = acc[v][x];
                }
        }
        __syncthreads();

        // ---- in-CTA carry resolution (warp 0, ascending worker order)
        if (warp == 0) {
            int w = 0;
            while (w < WARPS_PER_CTA) {
                const int row = Crow[w];
                bool any = false;
                T s[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) s[t] = R::id();
                int w2 = w;
                while (w2 < WARPS_PER_CTA && Crow[w2] == row) {
                    if (Cflag[w2]) {
                        any = true;
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            const int cc = lane + 32 * t;
                            if (cc < n) s[t] = R::add(s[t], Cw[w2 * n + cc]);
                        }
                    }
                    ++w2;
                }
                if (row == (int)re) {  // the tile's open row: carry it forward
                    if (lane == 0) { Crow[WARPS_PER_CTA] = row; Cflag[WARPS_PER_CTA] = any ? 1 : 0; }
                    if (any) {
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            const int cc = lane + 32 * t;
                            if (cc < n) Cw[WARPS_PER_CTA * n + cc] = s[t];
                        }
                    }
                } else if (any && row < m) {  // owner already wrote C[row] in this tile
                    T* crow = C + (long long)row * ldc;
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int cc = lane + 32 * t;
                        if (cc < n) crow[cc] = R::add(crow[cc], s[t]);
                    }
                }
                w = w2;
            }
        }
        __syncthreads();
        done += Ls;
        rs = re;
        zs = ze;
    }

    // ---- CTA carry-out (Alg. 1 line 22): the open row at the CTA end
    if (warp == 0) {
        const int row = (cta_re < m) ? (int)cta_re : -1;
        const bool any = (row >= 0) && Cflag[WARPS_PER_CTA] && Crow[WARPS_PER_CTA] == row;
        if (lane == 0) { carry_row[cta] = row; carry_flag[cta] = any ? 1 : 0; }
        if (any) {
            for (int cc = lane; cc < n; cc += 32) carry_val[(long long)cta * n + cc] = Cw[WARPS_PER_CTA * n + cc];
        }
    }
}

// FixCarryOut (Alg. 1 line 24): one warp per CTA carry; the first CTA of each run of equal carry
// rows sums the run in ascending CTA order and adds it into C[row].
template <typename T, int SR>
__global__ void __launch_bounds__(THREADS)
k_fixup(int num_ctas, int n, const int* __restrict__ carry_row, const int* __restrict__ carry_flag,
        const T* __restrict__ carry_val, T* __restrict__ C, long long ldc) {
    using R = Ring<T, SR>;
    const int lane = threadIdx.x & 31;
    const long long c = (long long)blockIdx.x * WARPS_PER_CTA + (threadIdx.x >> 5);
    if (c >= num_ctas) return;
    const int row = carry_row[c];
    if (row < 0) return;
    if (c > 0 && carry_row[c - 1] == row) return;  // not the head of its run
    T s[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) s[t] = R::id();
    bool any = false;
    for (long long cc = c; cc < num_ctas && carry_row[cc] == row; ++cc) {
        if (carry_flag[cc]) {
            any = true;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int j = lane + 32 * t;
                if (j < n) s[t] = R::add(s[t], carry_val[cc * n + j]);
            }
        }
    }
    if (!any) return;
    T* crow = C + (long long)row * ldc;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int j = lane + 32 * t;
        if (j < n) crow[j] = R::add(crow[j], s[t]);
    }
}

}  // namespace spmm
