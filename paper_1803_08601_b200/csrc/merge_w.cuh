// merge_w.cuh -- Algorithm II, merge-based SpMM, phase 2 (Alg. 1 lines 3-23) as a
// register-light, warp-autonomous kernel for sm_100a.
//
// Why this shape (profiles/r02_gather_probe.txt): on R-MAT matrices the merge kernel is bound by the
// latency of scattered 256-byte B-row gathers (ILP and TLP share the register budget).
// The only lever that moved the gather ceiling on B200 was rows in flight per SM (warps x gathers per
// warp); TMA bulk row copies and L2 evict-last hints for hot rows did not.  So a worker here holds no
// staged tile: it streams its own slice of the merge path straight from global memory through small
// register windows, and every register it saves becomes resident warps (more gathers in flight).
//
//   task     = I consecutive merge-path items (rows + nonzeros), PartitionSpmm (Alg. 1 line 2,
//              k_partition) gives its start state (row, nonzero); tasks are taken round-robin by the
//              persistent warps (equal items per task, so equal work -- the point of merge path).
//   windows  = 32 column indices + 32 values (one coalesced 4-byte load per lane each, prefetched one
//              window ahead) copied into a 256-byte per-warp shared-memory slot and read back as LDS.128
//              broadcasts (the paper's 32 Broadcast rounds, Alg. 1 lines 14-17); 32 row ends
//              (row_offsets[r+1]) in one register per lane, handed out with __shfl_sync.
//   gathers  = U B rows per batch, lanes over columns, issued back to back before
//              the first FMA; a running accumulator is flushed to C on each row end (rows first on
//              ties), empty rows get the semiring identity -- Alg. 1's valB[32] + PrepareSpmm +
//              segmented reduction (lines 18-22) collapse into this flush because every lane of the
//              worker sees the same row id.
//   carries  = the row open at the task's end (Alg. 1 line 22): its partial goes to carry[task]; the
//              worker that consumes a row's end item writes the row (SURVEY.md §8(c) ambiguity 20) and
//              k_fixup adds the carries in ascending task order after this kernel (Alg. 1 line 24).
#pragma once
#include "common.cuh"
#include "ptx.cuh"

namespace spmm {

constexpr int MW_THREADS = 256;

struct MergeParams {
    int m, n, nnz;
    const int* ro;
    const int* col;
    const void* val;
    const void* B;
    unsigned ldb_bytes;
    void* C;
    long long ldc;
    const int* states;  // (row, nonzero) at every task boundary, num_tasks + 1 pairs
    int num_tasks;
    int* carry_row;
    int* carry_flag;
    void* carry_val;
    int* task_ctr;  // non-null: warps take tasks from this queue (zeroed by k_partition), else a static
                    // block of consecutive tasks per warp
    EpiParams epi;  // accumulate / peer copies of finished rows
};

// next task of this warp: from the queue (one atomic per task, lane 0) or the next of its static block
__device__ __forceinline__ int mw_grab(const MergeParams& P) {
    int t = 0;
    if ((threadIdx.x & 31) == 0) t = atomicAdd(P.task_ctr, 1);
    return __shfl_sync(0xffffffffu, t, 0);
}

// accumulator of VEC*NV columns for one lane
template <typename T, int SR, int VEC, int NV> struct MAcc {
    T v[NV][VEC];
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int a = 0; a < NV; ++a)
#pragma unroll
            for (int x = 0; x < VEC; ++x) v[a][x] = Ring<T, SR>::id();
    }
    __device__ __forceinline__ void mac(T a, const unsigned (&b)[NV][VEC]) {
        if constexpr (std::is_same<T, float>::value && SR == SR_PLUS_TIMES && VEC % 2 == 0) {
            const float2 aa = make_float2(a, a);
#pragma unroll
            for (int q = 0; q < NV; ++q)
#pragma unroll
                for (int x = 0; x < VEC; x += 2) {
                    float2 c = make_float2(v[q][x], v[q][x + 1]);
                    c = ffma2(aa, make_float2(__uint_as_float(b[q][x]), __uint_as_float(b[q][x + 1])), c);
                    v[q][x] = c.x;
                    v[q][x + 1] = c.y;
                }
        } else {
#pragma unroll
            for (int q = 0; q < NV; ++q)
#pragma unroll
                for (int x = 0; x < VEC; ++x) v[q][x] = Ring<T, SR>::mac(v[q][x], a, from_bits<T>(b[q][x]));
        }
    }
};

#ifndef MW_LDG_HINT
#define MW_LDG_HINT ".nc"  // B-row gathers: read-only path
#endif
template <int VEC> __device__ __forceinline__ void mw_ldg(unsigned (&o)[VEC], const void* p);
template <> __device__ __forceinline__ void mw_ldg<1>(unsigned (&o)[1], const void* p) {
    asm volatile("ld.global" MW_LDG_HINT ".b32 %0, [%1];" : "=r"(o[0]) : "l"(p));
}
template <> __device__ __forceinline__ void mw_ldg<2>(unsigned (&o)[2], const void* p) {
    asm volatile("ld.global" MW_LDG_HINT ".v2.b32 {%0, %1}, [%2];" : "=r"(o[0]), "=r"(o[1]) : "l"(p));
}
template <> __device__ __forceinline__ void mw_ldg<4>(unsigned (&o)[4], const void* p) {
    asm volatile("ld.global" MW_LDG_HINT ".v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]) : "l"(p));
}

__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <typename T, int SR, int VEC, int NV, int U, int MINB, bool EPI>
__global__ void __launch_bounds__(MW_THREADS, MINB) k_merge_w(const MergeParams P) {
    static_assert(32 % U == 0, "a window of 32 nonzeros holds whole batches");
    // per warp: two nonzero windows (column indices | values, filled by cp.async one window ahead) and
    // one window of 32 row ends
    __shared__ __align__(16) unsigned zwin[MW_THREADS / 32][2][2][32];
    __shared__ __align__(16) int ewin[MW_THREADS / 32][32];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int m = P.m, n = P.n;
    const uint32_t zbase = smem_u32(&zwin[wib][0][0][0]);  // slot s: + 256 s; values: + 128
    const uint32_t ebase = smem_u32(&ewin[wib][0]);

    // this lane's column blocks; lanes past n gather column 0 of the same row (valid memory, never
    // stored), so the gathers need no column predicate
    int cofs[NV];
    bool colok[NV];
    const char* Blv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        cofs[v] = (v * 32 + lane) * VEC;
        colok[v] = cofs[v] < n;
        Blv[v] = opaque_ptr(static_cast<const char*>(P.B) + (colok[v] ? (size_t)cofs[v] * sizeof(T) : (size_t)0));
    }
    const unsigned ldb_bytes = P.ldb_bytes;
    const int* __restrict__ ro = P.ro;
    const int* __restrict__ colg = P.col;
    const unsigned* __restrict__ valg = static_cast<const unsigned*>(P.val);

    // tasks [t0, t1) of this warp, processed in path order: the next task starts where this one ends,
    // so only the end state is loaded per task
    const bool dyn = P.task_ctr != nullptr;
    const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int tpw = (P.num_tasks + nwarps - 1) / nwarps;
    int task = dyn ? mw_grab(P) : gw * tpw;
    const int t1 = dyn ? P.num_tasks : min(P.num_tasks, gw * tpw + tpw);
    int r = 0, q = 0;
    if (task < t1) { r = __ldg(P.states + 2 * task); q = __ldg(P.states + 2 * task + 1); }
    while (task < t1) {
        const int next = dyn ? mw_grab(P) : task + 1;  // taken early: the atomic's latency overlaps the task
        if (dyn) { r = __ldg(P.states + 2 * task); q = __ldg(P.states + 2 * task + 1); }
        const int r1 = __ldg(P.states + 2 * task + 2), q1 = __ldg(P.states + 2 * task + 3);
        // nonzero windows: window w = nonzeros [q_task + 32 w, +32) in slot w & 1
        auto load_window = [&](int zstart, uint32_t slot) {
            if (zstart + lane < q1) {
                cp_async4(slot + 4u * lane, colg + zstart + lane);
                cp_async4(slot + 128u + 4u * lane, valg + zstart + lane);
            }
            cp_async_commit();
        };
        // row-end window: slot j holds row_offsets[rb + j + 1] (end of row rb + j), INT_MAX past r1 / m
        auto load_ends = [&](int rbase) {
            const int ev = (rbase + lane < m && rbase + lane <= r1) ? __ldg(ro + rbase + lane + 1) : 0x7fffffff;
            __syncwarp();
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(ebase + 4u * lane), "r"(ev) : "memory");
            __syncwarp();
        };
        int rb = r;
        int zb = q;
        uint32_t slot = zbase;
        load_window(zb, slot);
        load_ends(rb);
        int e = (int)lds_u32(ebase);
        MAcc<T, SR, VEC, NV> acc;
        acc.reset();
        bool dirty = false;

        auto store_row = [&](int row) {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (colok[v]) {
                    unsigned o[VEC];
#pragma unroll
                    for (int x = 0; x < VEC; ++x) o[x] = to_bits<T>(acc.v[v][x]);
                    T* p = static_cast<T*>(P.C) + (long long)row * P.ldc + cofs[v];
                    if constexpr (EPI) epi_store_ext<T, SR, VEC>(P.epi, p, row, cofs[v], o);  // accumulate / peers
                    else st_vec<VEC>(p, o);
                }
            }
        };
        auto flush = [&]() {  // the row-end item of row r: write it (owner), identity if nothing was added
            store_row(r);
            acc.reset();
            dirty = false;
            ++r;
            if (r - rb == 32) {  // next 32 row ends (a dependent load, once per 32 rows)
                rb = r;
                load_ends(rb);
            }
            e = (int)lds_u32(ebase + 4u * (uint32_t)(r - rb));
        };

        while (q < q1) {
            // window at zb has landed (the only cp.async group in flight); start the next one
            cp_async_wait_all();
            __syncwarp();
            const uint32_t wcol = slot, wval = slot + 128u;
            const int zn = zb + 32;
            slot ^= 256u;
            if (zn < q1) load_window(zn, slot);
            while (q < min(zn, q1)) {
                const uint32_t wp4 = 4u * (uint32_t)(q - zb);
                unsigned bv[U][NV][VEC];
                unsigned cu[U];
                if (q + U <= min(zn, q1)) {
                    // full batch: U gathers back to back (ILP), then accumulate with row-end checks
#pragma unroll
                    for (int u = 0; u < U; u += 4) {
                        const uint4 c4 = lds_u128(wcol + wp4 + 4u * u);
                        cu[u] = c4.x; cu[u + 1] = c4.y; cu[u + 2] = c4.z; cu[u + 3] = c4.w;
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u)
#pragma unroll
                        for (int v = 0; v < NV; ++v) mw_ldg<VEC>(bv[u][v], Blv[v] + (size_t)cu[u] * ldb_bytes);
                    if (q + U <= e) {  // the whole batch lies inside row r
#pragma unroll
                        for (int u = 0; u < U; u += 2) {
                            const uint2 a2 = lds_u64(wval + wp4 + 4u * u);
                            acc.mac(from_bits<T>(a2.x), bv[u]);
                            acc.mac(from_bits<T>(a2.y), bv[u + 1]);
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            while (e <= q + u) flush();  // rows ending before nonzero q+u (rows first on ties)
                            acc.mac(from_bits<T>(lds_u32(wval + wp4 + 4u * u)), bv[u]);
                        }
                    }
                    q += U;
                } else {
                    // task tail: fewer than U nonzeros left
                    const int cnt = min(zn, q1) - q;
#pragma unroll
                    for (int u = 0; u < U; ++u) cu[u] = lds_pred(wcol + wp4 + 4u * u, u < cnt);
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (u < cnt) {
#pragma unroll
                            for (int v = 0; v < NV; ++v) mw_ldg<VEC>(bv[u][v], Blv[v] + (size_t)cu[u] * ldb_bytes);
                        }
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (u < cnt) {
                            while (e <= q + u) flush();
                            acc.mac(from_bits<T>(lds_u32(wval + wp4 + 4u * u)), bv[u]);
                        }
                    q += cnt;
                }
                dirty = true;
            }
            zb = zn;
        }
        while (r < r1) flush();  // row ends after the task's last nonzero (incl. empty rows)
        // carry-out (Alg. 1 line 22): the partial of row r1, whose end item belongs to a later task
        if (lane == 0) {
            P.carry_row[task] = (r1 < m) ? r1 : -1;
            P.carry_flag[task] = (dirty && r1 < m) ? 1 : 0;
        }
        if (dirty && r1 < m) {
            T* cv = static_cast<T*>(P.carry_val) + (long long)task * n;
#pragma unroll
            for (int v = 0; v < NV; ++v)
                if (colok[v]) {
#pragma unroll
                    for (int x = 0; x < VEC; ++x)
                        if (cofs[v] + x < n) cv[cofs[v] + x] = acc.v[v][x];
                }
        }
        __syncwarp();  // the next task reuses the window slots
        task = next;
    }
}

}  // namespace spmm
