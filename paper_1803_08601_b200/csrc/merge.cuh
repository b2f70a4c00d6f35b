// merge.cuh -- Algorithm II, merge-based SpMM (§4.2, Algorithm 1), sm_100a.
//
// Phase 1, PartitionSpmm (Alg. 1 line 2): k_partition writes the merge-path state
//   (row, nonzero) at which every task starts (the paper partitions per CTA; here a task is one merge
//   worker's slice).  2-D merge path (Fig. 2(c)): task c starts on diagonal c*I of the
//   merge of row-end offsets with nonzero indices (rows first on ties), so every task gets I items =
//   rows + nonzeros, which also charges the C write of empty rows.  1-D nonzero split
//   (PAPER.md:80, the paper's own choice, :89): task c starts at nonzero c*I in the largest row r with
//   ro[r] <= c*I.  One coalesced pass over the rows: each row writes the boundaries that fall inside it.
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

constexpr int PART_ROWS = 16;  // k_partition: rows per thread and iteration
constexpr int PART_MINB = 4;   // k_partition: resident CTAs per SM (register budget of PART_ROWS + 1 offsets)

// states[2c] = row, states[2c+1] = nonzero, c in [0, num_ctas]: one pass over the rows instead of a
// search per boundary.  2-D merge path: the row-end item of row r sits at path position
// p_r = r + ro[r+1] (rows first on ties), so the boundary on diagonal d = c*I (< m + nnz) has consumed
// exactly the rows with p_r < d, i.e. row r for p_{r-1} < d <= p_r, and nonzero d - r (the oracle's
// characterisation, tests/test_oracle.py).  1-D nonzero split: the boundary at nonzero t = c*I lies in
// the non-empty row r with ro[r] <= t < ro[r+1] (the largest r with ro[r] <= t).  Boundary 0 is
// (0, 0) and boundary num_ctas is (m, nnz) in both.  Thread r reads ro[r], ro[r+1] (coalesced) and
// writes the boundaries inside its row -- usually none or one; a row longer than I owns several.
// (PART_ROWS consecutive rows per thread and iteration.)
// It also zeroes the compute kernel's task queue.
__global__ void __launch_bounds__(THREADS, PART_MINB)
k_partition(const int* __restrict__ ro, int m, int nnz, int items, int mode, int num_ctas, int* __restrict__ states,
            int* __restrict__ task_ctr) {
    const long long tid0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid0 == 0) {
        if (task_ctr) *task_ctr = 0;
        states[0] = 0;
        states[1] = 0;
        states[2LL * num_ctas] = m;
        states[2LL * num_ctas + 1] = nnz;
    }
    const long long I = items;
    const long long last = (long long)num_ctas - 1;  // interior boundaries 1 .. num_ctas - 1
    // a warp takes 32 x PART_ROWS consecutive rows per iteration; their offsets are loaded coalesced
    // (one 128-byte line per load instruction) into a per-warp shared buffer, skewed by one word per 32
    // so that lane l then reads its own PART_ROWS + 1 consecutive offsets (rows 16 l ..) without bank
    // conflicts; the warp's loads are issued back to back (one memory round trip per iteration)
    constexpr int WR = 32 * PART_ROWS;  // rows per warp and iteration
    __shared__ int sro[WARPS_PER_CTA][WR + 1 + (WR + 1) / 32 + 1];
    const int lane = threadIdx.x & 31;
    int* so = sro[threadIdx.x >> 5];
    const long long gwarp = tid0 >> 5;
    const long long wstride = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long wb = gwarp * WR; wb < m; wb += wstride * WR) {
        int v[PART_ROWS + 1];
#pragma unroll
        for (int k = 0; k <= PART_ROWS; ++k) {
            const long long idx = wb + 32LL * k + lane;
            v[k] = (idx <= m && (k < PART_ROWS || lane == 0)) ? __ldg(ro + idx) : 0;
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k <= PART_ROWS; ++k) {
            const int i = 32 * k + lane;  // position i + i / 32
            if (k < PART_ROWS || lane == 0) so[i + k] = v[k];
        }
        __syncwarp();
        const long long r0 = wb + (long long)PART_ROWS * lane;
        int o[PART_ROWS + 1];
#pragma unroll
        for (int u = 0; u <= PART_ROWS; ++u) {
            const int i = PART_ROWS * lane + u;
            o[u] = so[i + (i >> 5)];
        }
        if (r0 >= m) continue;
        // the first boundary at or after this thread's first row: one division per PART_ROWS rows, then
        // the rows are walked with D = c * I advancing by I (no per-row division)
        long long c = (mode == 0) ? (r0 - 1 + o[0]) / I + 1  // first c with c*I > p_{r0-1} (p_{-1} = -1)
                                  : (o[0] + I - 1) / I;      // first c with c*I >= ro[r0]
        if (c < 1) c = 1;
        long long D = c * I;
#pragma unroll
        for (int u = 0; u < PART_ROWS; ++u) {
            const long long r = r0 + u;
            if (r >= m) break;
            // 2-D: boundaries with p_{r-1} < D <= p_r = r + ro[r+1] hold row r, nonzero D - r;
            // 1-D: boundaries with ro[r] <= D < ro[r+1] hold row r, nonzero D (empty rows hold none)
            const long long lim = (mode == 0) ? r + o[u + 1] + 1 : (long long)o[u + 1];
            for (; c <= last && D < lim; ++c, D += I) {
                states[2 * c] = (int)r;
                states[2 * c + 1] = (int)((mode == 0) ? D - r : D);
            }
        }
    }
}

// grid of k_partition: PART_ROWS rows per thread and iteration, one wave (PART_MINB CTAs per SM)
inline unsigned partition_grid(long long m) {
    const long long g = (m + (long long)PART_ROWS * THREADS - 1) / ((long long)PART_ROWS * THREADS);
    return (unsigned)(g < 1 ? 1 : (g > (long long)PART_MINB * 148 ? (long long)PART_MINB * 148 : g));
}

// FixCarryOut (Alg. 1 line 24): the first task of each run of equal carry rows sums the run in
// ascending task order and adds it into C[row].  One warp per FIX_K consecutive carries, lanes over
// columns: every load of the common case (runs of one carry) is issued before the first use, so the
// kernel costs two memory round trips (carries, then the C rows) instead of one chain per carry.
// (Carry values are read even when their flag is 0 -- workspace memory, never used then.)
constexpr int FIX_K = 4;
inline unsigned fixup_grid(long long num_ctas) {
    return (unsigned)((num_ctas + (long long)FIX_K * WARPS_PER_CTA - 1) / ((long long)FIX_K * WARPS_PER_CTA));
}
template <typename T, int SR>
__global__ void __launch_bounds__(THREADS)
k_fixup(int num_ctas, int n, const int* __restrict__ carry_row, const int* __restrict__ carry_flag,
        const T* __restrict__ carry_val, T* __restrict__ C, long long ldc, const EpiParams E) {
    using R = Ring<T, SR>;
    const int lane = threadIdx.x & 31;
    const long long c0 = ((long long)blockIdx.x * WARPS_PER_CTA + (threadIdx.x >> 5)) * FIX_K;
    if (c0 >= num_ctas) return;
    int rw[FIX_K + 2];  // carry rows of tasks c0 - 1 .. c0 + FIX_K (-1: none)
#pragma unroll
    for (int i = 0; i < FIX_K + 2; ++i) {
        const long long cc = c0 - 1 + i;
        rw[i] = (cc >= 0 && cc < num_ctas) ? carry_row[cc] : -1;
    }
    int fl[FIX_K];
    T s[FIX_K][4];
#pragma unroll
    for (int k = 0; k < FIX_K; ++k) {
        const long long cc = c0 + k;
        fl[k] = cc < num_ctas ? carry_flag[cc] : 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int j = lane + 32 * t;
            s[k][t] = (cc < num_ctas && j < n) ? carry_val[cc * n + j] : R::id();
        }
    }
    bool head[FIX_K];
#pragma unroll
    for (int k = 0; k < FIX_K; ++k) {
        const int row = rw[k + 1];
        bool any = fl[k] != 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) s[k][t] = any ? R::add(R::id(), s[k][t]) : R::id();
        head[k] = row >= 0 && rw[k] != row;  // the first carry of its run
        if (head[k] && rw[k + 2] == row) {  // a run of several carries (a row spanning > 2 tasks; warp-uniform)
            // 32 carries per round: lanes load their row / flag, a ballot finds where the run ends, then
            // the flagged partials are added in ascending task order (their loads are independent)
            for (long long cc = c0 + k + 1;; cc += 32) {
                const long long cl = cc + lane;
                const int rl = cl < num_ctas ? carry_row[cl] : -1;
                const int fg = cl < num_ctas ? carry_flag[cl] : 0;
                const unsigned same = __ballot_sync(FULL, rl == row);
                const int len = (same == FULL) ? 32 : __ffs(~same) - 1;  // run members in this round
                unsigned fm = __ballot_sync(FULL, fg != 0) & (len == 32 ? FULL : ((1u << len) - 1u));
                any = any || fm != 0u;
#pragma unroll 4
                for (; fm; fm &= fm - 1u) {
                    const long long cf = cc + (__ffs(fm) - 1);
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int j = lane + 32 * t;
                        if (j < n) s[k][t] = R::add(s[k][t], carry_val[cf * n + j]);
                    }
                }
                if (len < 32) break;
            }
        }
        head[k] = head[k] && any;
    }
    // C[row] (+)= the run (the owner's write, already accumulated into C if requested, came first); the
    // final row also goes to the peer copies of C.  All C rows are read before the first store.
    T cv[FIX_K][4];
#pragma unroll
    for (int k = 0; k < FIX_K; ++k)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int j = lane + 32 * t;
            cv[k][t] = (head[k] && j < n) ? C[(long long)rw[k + 1] * ldc + j] : R::id();
        }
#pragma unroll
    for (int k = 0; k < FIX_K; ++k) {
        if (!head[k]) continue;
        const long long row = rw[k + 1];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int j = lane + 32 * t;
            if (j < n) {
                const T v = R::add(cv[k][t], s[k][t]);
                C[row * ldc + j] = v;
                for (int i = 0; i < E.npeers; ++i) static_cast<T*>(E.peer[i])[(row + E.peer_row0) * E.peer_ldc + j] = v;
            }
        }
    }
}

}  // namespace spmm
