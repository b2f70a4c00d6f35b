// merge.cuh -- Algorithm II, merge-based SpMM (§4.2, Algorithm 1), sm_100a.
//
// Phase 1, PartitionSpmm (Alg. 1 line 2): k_partition writes the merge-path state
//   (row, nonzero) at which every task starts (the paper partitions per CTA; here a task is one merge
//   worker's slice).  2-D merge path (Fig. 2(c)): task c starts on diagonal c*I of the
//   merge of row-end offsets with nonzero indices (rows first on ties), so every task gets I items =
//   rows + nonzeros, which also charges the C write of empty rows.  1-D nonzero split
//   (PAPER.md:80, the paper's own choice, :89): task c starts at nonzero c*I in the largest row r with
//   ro[r] <= c*I.  One warp per boundary, 32-ary search (~6 dependent probes).
// Phase 2 (Alg. 1 lines 3-23) is k_merge_w in merge_w.cuh: each warp streams its tasks' items from
//   global memory through small windows (the GlobalToShared of line 5 becomes a per-warp cp.async
//   window), with a running accumulator flushed on each row end; a task's open row becomes its
//   carry-out (line 22).
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
k_partition(const int* __restrict__ ro, int m, int nnz, int items, int mode, int num_ctas, int* __restrict__ states,
            int* __restrict__ task_ctr) {
    const int lane = threadIdx.x & 31;
    if (task_ctr && blockIdx.x == 0 && threadIdx.x == 0) *task_ctr = 0;  // the compute kernel's task queue
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

// FixCarryOut (Alg. 1 line 24): one warp per task carry; the first task of each run of equal carry
// rows sums the run in ascending task order and adds it into C[row].
template <typename T, int SR>
__global__ void __launch_bounds__(THREADS)
k_fixup(int num_ctas, int n, const int* __restrict__ carry_row, const int* __restrict__ carry_flag,
        const T* __restrict__ carry_val, T* __restrict__ C, long long ldc, const EpiParams E) {
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
    // C[row] (+)= the run (the owner's write, already accumulated into C if requested, came first); the
    // final row also goes to the peer copies of C
    T* crow = C + (long long)row * ldc;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const int j = lane + 32 * t;
        if (j < n) {
            const T v = R::add(crow[j], s[t]);
            crow[j] = v;
            for (int i = 0; i < E.npeers; ++i) static_cast<T*>(E.peer[i])[(row + E.peer_row0) * E.peer_ldc + j] = v;
        }
    }
}

}  // namespace spmm
