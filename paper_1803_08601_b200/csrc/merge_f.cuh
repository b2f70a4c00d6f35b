// merge_f.cuh -- Algorithm II, merge-based SpMM, phase 2 (Alg. 1 lines 3-23) for
// narrow B (n <= 16): lane-folded workers.
//
// k_merge_w gives every merge worker a whole warp with lanes over B's columns; at n = 1 that leaves
// 31 of 32 lanes idle -- the paper's Type-2 waste (§3.2).  Here a warp is split into
// P = 32 / G slots of G lanes (G * VEC >= n columns), and the P slots walk P consecutive pieces of
// the warp's merge path at once, the paper's thread-level remedy for short work (§4.1)
// applied to the merge path:
//
//   chunk    = P * L consecutive items (rows + nonzeros) of the warp's task; its row ends
//              (row_offsets[r + 1]) and nonzeros (col, val) are staged in a per-warp shared-memory
//              window with cp.async, double-buffered (the next chunk streams in during this one).
//   slot s   = items [s L, (s + 1) L) of the chunk: its start state (row, nonzero) is the merge-path
//              split of diagonal s L (the paper's 2-D partition, applied per slot), found
//              in one warp-parallel pass over the staged row ends' path positions; it gathers its <= L B rows back to back (ILP), then walks its items in path
//              order (rows first on ties): a row that starts and ends inside the slot is written
//              directly; the first row end of the slot closes a row that may have started in an
//              earlier slot ("head"); the row open at the slot's end is its "tail".
//   combine  = a segmented scan over the slots' tails (segments restart at every slot that
//              consumed a row end) gives each head the partials of the slots before it -- the
//              paper's segmented reduction (Alg. 1 lines 19-22) across slots instead of lanes;
//              the chunk's last tail is carried into the next chunk, and the task's last tail is
//              its carry-out (Alg. 1 line 22), fixed up by k_fixup (line 24).
// Ownership is the same as k_merge_w (SURVEY.md §8(c) ambiguity 20): whoever consumes a row's end
// item writes the row, earlier partials of the same task are folded in before the write, and
// partials of earlier tasks are added by k_fixup in ascending task order.
#pragma once
#include "common.cuh"
#include "merge_w.cuh"
#include "ptx.cuh"

namespace spmm {

#ifndef MF_THREADS_DEF
#define MF_THREADS_DEF 128
#endif
constexpr int MF_THREADS = MF_THREADS_DEF;  // 4 warps per CTA (the per-warp windows are a few KB each)

template <int VEC> __device__ __forceinline__ void mf_ldg(unsigned (&o)[VEC], const void* p, bool pred);
template <> __device__ __forceinline__ void mf_ldg<1>(unsigned (&o)[1], const void* p, bool pred) {
    asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; mov.b32 %0, 0; @q ld.global.nc.b32 %0, [%1];}"
                 : "=r"(o[0]) : "l"(p), "r"((int)pred));
}
template <> __device__ __forceinline__ void mf_ldg<2>(unsigned (&o)[2], const void* p, bool pred) {
    asm volatile("{.reg .pred q; setp.ne.b32 q, %3, 0; mov.b32 %0, 0; mov.b32 %1, 0; @q ld.global.nc.v2.b32 {%0, %1}, [%2];}"
                 : "=r"(o[0]), "=r"(o[1]) : "l"(p), "r"((int)pred));
}
template <> __device__ __forceinline__ void mf_ldg<4>(unsigned (&o)[4], const void* p, bool pred) {
    asm volatile("{.reg .pred q; setp.ne.b32 q, %5, 0; mov.b32 %0, 0; mov.b32 %1, 0; mov.b32 %2, 0; mov.b32 %3, 0;"
                 " @q ld.global.nc.v4.b32 {%0, %1, %2, %3}, [%4];}"
                 : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]) : "l"(p), "r"((int)pred));
}

template <typename T, int SR, int VEC, int G, int L, int MINB, bool EPI>
__global__ void __launch_bounds__(MF_THREADS, MINB) k_merge_f(const MergeParams P) {
    using R = Ring<T, SR>;
    constexpr int NS = 32 / G;      // slots per warp
    constexpr int CH = NS * L;      // items per chunk
    constexpr int EW = CH + 4;      // staged row ends per buffer (CH + 1, padded)
    constexpr int BUFW = EW + 2 * CH;
    __shared__ __align__(16) unsigned win[MF_THREADS / 32][2][BUFW];
    __shared__ int sst[MF_THREADS / 32][33];  // start row (relative to the chunk) of each slot, + chunk end
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const int slot = lane / G;
    const int j = lane % G;  // lane within the slot: columns [j VEC, j VEC + VEC)
    const int m = P.m, n = P.n;
    const int cofs = j * VEC;
    const bool colok = cofs < n;
    const char* Bl = static_cast<const char*>(P.B) + (colok ? (size_t)cofs * sizeof(T) : (size_t)0);
    const unsigned ldb_bytes = P.ldb_bytes;
    const int* __restrict__ ro = P.ro;
    const unsigned* __restrict__ colg = reinterpret_cast<const unsigned*>(P.col);
    const unsigned* __restrict__ valg = static_cast<const unsigned*>(P.val);
    const uint32_t wbase = smem_u32(&win[wib][0][0]);

    const bool dyn = P.task_ctr != nullptr;
    const int nwarps = (int)((gridDim.x * blockDim.x) >> 5);
    const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int tpw = (P.num_tasks + nwarps - 1) / nwarps;
    int task = dyn ? mw_grab(P) : gw * tpw;
    const int t1 = dyn ? P.num_tasks : min(P.num_tasks, gw * tpw + tpw);

    auto store = [&](int row, const T (&v)[VEC]) {
        if (colok) {
            unsigned o[VEC];
#pragma unroll
            for (int x = 0; x < VEC; ++x) o[x] = to_bits<T>(v[x]);
            T* p = static_cast<T*>(P.C) + (long long)row * P.ldc + cofs;
            if constexpr (EPI) epi_store_ext<T, SR, VEC>(P.epi, p, row, cofs, o);  // accumulate / peers
            else st_vec<VEC>(p, o);
        }
    };

    while (task < t1) {
        const int next = dyn ? mw_grab(P) : task + 1;
        int rc = __ldg(P.states + 2 * task), qc = __ldg(P.states + 2 * task + 1);
        const int r1 = __ldg(P.states + 2 * task + 2), q1 = __ldg(P.states + 2 * task + 3);
        // stage the window of the chunk starting at (rs, zs) into buffer b: row ends of rows rs.. (only
        // rows < r1: the task's last row ends in a later task) and nonzeros zs.. (only < q1)
        auto stage = [&](int b, int rs, int zs) {
            const uint32_t eb = wbase + 4u * (uint32_t)(b * BUFW);
            for (int x = lane; x <= CH; x += 32)
                if (rs + x < r1) cp_async4(eb + 4u * x, ro + rs + x + 1);
            for (int x = lane; x < CH; x += 32)
                if (zs + x < q1) {
                    cp_async4(eb + 4u * (EW + x), colg + zs + x);
                    cp_async4(eb + 4u * (EW + CH + x), valg + zs + x);
                }
            cp_async_commit();
        };
        int left = (r1 - rc) + (q1 - qc);  // items of this task not yet consumed
        T carry[VEC];
#pragma unroll
        for (int x = 0; x < VEC; ++x) carry[x] = R::id();
        bool carry_dirty = false;
        int b = 0;
        if (left > 0) stage(0, rc, qc);
        while (left > 0) {
            cp_async_wait_all();
            __syncwarp();
            const uint32_t eb = wbase + 4u * (uint32_t)(b * BUFW);
            const uint32_t cb = eb + 4u * EW, vb = cb + 4u * CH;
            const int ic = min(CH, left);
            const int rows_lim = r1 - rc;
            // slot boundaries (the merge-path split of diagonals s L): row end x of the chunk
            // sits at path position x + (E[x] - qc) (rows first on ties), so slot s starts after the
            // row ends with position < min(s L, ic).  One pass over the chunk's row ends, 32 at a time
            // in path order: row end x writes itself as the start row of the slots (slot(x-1), slot(x)].
            const uint32_t sb = smem_u32(&sst[wib][0]);
            const int rmax = min(rows_lim, ic);
            int rc_chunk = 0, last = -1;
            for (int x0 = 0; x0 < rmax; x0 += 32) {
                const int x = x0 + lane;
                const int pos = (x < rmax) ? x + (int)lds_u32(eb + 4u * x) - qc : 0x7fffffff;
                const bool inside = pos < ic;
                const int sl = inside ? pos / L : NS;
                int slp = __shfl_up_sync(FULL, sl, 1);
                if (lane == 0) slp = last;
                if (inside)
                    for (int q = slp + 1; q <= sl; ++q) asm volatile("st.shared.b32 [%0], %1;" ::"r"(sb + 4u * q), "r"(x) : "memory");
                const unsigned bal = __ballot_sync(FULL, inside);
                rc_chunk += __popc(bal);
                if (bal) last = __shfl_sync(FULL, sl, 31 - __clz(bal));
                if (bal != FULL) break;
            }
            if (lane > last) asm volatile("st.shared.b32 [%0], %1;" ::"r"(sb + 4u * lane), "r"(rc_chunk) : "memory");
            if (lane == 0) asm volatile("st.shared.b32 [%0], %1;" ::"r"(sb + 4u * NS), "r"(rc_chunk) : "memory");
            __syncwarp();
            const int is = (int)lds_u32(sb + 4u * slot);
            const int in = (int)lds_u32(sb + 4u * (slot + 1));
            const int zs = min(slot * L, ic) - is;
            const int zn = min((slot + 1) * L, ic) - in;
            const int ie_chunk = rc_chunk;
            const int ze_chunk = ic - ie_chunk;
            // the next chunk's window streams in while this one is processed
            const int left_next = left - ic;
            if (left_next > 0) stage(b ^ 1, rc + ie_chunk, qc + ze_chunk);
            const int cnt = zn - zs;
            // gathers of the slot's nonzeros, back to back
            unsigned bv[L][VEC];
#pragma unroll
            for (int u = 0; u < L; ++u) {
                const unsigned c = lds_pred(cb + 4u * (uint32_t)(zs + u), u < cnt);
                mf_ldg<VEC>(bv[u], Bl + (size_t)c * ldb_bytes, u < cnt);
            }
            // walk the slot's items in path order
            T acc[VEC], head[VEC];
#pragma unroll
            for (int x = 0; x < VEC; ++x) { acc[x] = R::id(); head[x] = R::id(); }
            bool has_end = false, tail_nz = false;
            int x = is;
            int e = (x < in) ? (int)lds_u32(eb + 4u * x) : 0x7fffffff;
            auto flush = [&]() {
                if (!has_end) {
#pragma unroll
                    for (int q = 0; q < VEC; ++q) head[q] = acc[q];
                    has_end = true;
                } else {
                    store(rc + x, acc);
                }
#pragma unroll
                for (int q = 0; q < VEC; ++q) acc[q] = R::id();
                tail_nz = false;
                ++x;
                e = (x < in) ? (int)lds_u32(eb + 4u * x) : 0x7fffffff;
            };
#pragma unroll
            for (int u = 0; u < L; ++u) {
                if (u < cnt) {
                    const int zabs = qc + zs + u;
                    while (e <= zabs) flush();
                    const T a = from_bits<T>(lds_u32(vb + 4u * (uint32_t)(zs + u)));
#pragma unroll
                    for (int q = 0; q < VEC; ++q) acc[q] = R::mac(acc[q], a, from_bits<T>(bv[u][q]));
                    tail_nz = true;
                }
            }
            while (x < in) flush();
            // segmented inclusive scan of the tails over the slots (segment starts at a slot with a row
            // end); slot 0 starts from the chunk's carry-in unless its segment restarts
            T tv[VEC];
#pragma unroll
            for (int q = 0; q < VEC; ++q) tv[q] = (slot == 0 && !has_end) ? R::add(carry[q], acc[q]) : acc[q];
            bool tf = has_end;
            bool td = (slot == 0 && !has_end) ? (carry_dirty || tail_nz) : tail_nz;
#pragma unroll
            for (int off = 1; off < NS; off <<= 1) {
                T up[VEC];
#pragma unroll
                for (int q = 0; q < VEC; ++q) up[q] = from_bits<T>(__shfl_up_sync(FULL, to_bits<T>(tv[q]), off * G));
                const bool uf = __shfl_up_sync(FULL, (int)tf, off * G) != 0;
                const bool ud = __shfl_up_sync(FULL, (int)td, off * G) != 0;
                if (slot >= off) {
                    if (!tf) {
#pragma unroll
                        for (int q = 0; q < VEC; ++q) tv[q] = R::add(up[q], tv[q]);
                        td = td || ud;
                    }
                    tf = tf || uf;
                }
            }
            // heads: partial carried in from the slots before (slot 0: the chunk's carry)
            T cin[VEC];
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
                const T up = from_bits<T>(__shfl_up_sync(FULL, to_bits<T>(tv[q]), G));
                cin[q] = slot == 0 ? carry[q] : up;
            }
            if (has_end) {
#pragma unroll
                for (int q = 0; q < VEC; ++q) head[q] = R::add(cin[q], head[q]);
                store(rc + is, head);
            }
            // the chunk's carry-out = the last slot's scanned tail
#pragma unroll
            for (int q = 0; q < VEC; ++q)
                carry[q] = from_bits<T>(__shfl_sync(FULL, to_bits<T>(tv[q]), (NS - 1) * G + j));
            carry_dirty = __shfl_sync(FULL, (int)td, (NS - 1) * G + j) != 0;
            rc += ie_chunk;
            qc += ze_chunk;
            left = left_next;
            b ^= 1;
        }
        // carry-out of the task (Alg. 1 line 22): the partial of row r1, whose end item is in a later task
        if (lane == 0) {
            P.carry_row[task] = (r1 < m) ? r1 : -1;
            P.carry_flag[task] = (carry_dirty && r1 < m) ? 1 : 0;
        }
        if (slot == 0 && carry_dirty && r1 < m) {
            T* cv = static_cast<T*>(P.carry_val) + (long long)task * n;
#pragma unroll
            for (int q = 0; q < VEC; ++q)
                if (cofs + q < n) cv[cofs + q] = carry[q];
        }
        __syncwarp();  // the next task reuses the window buffers
        task = next;
    }
}

}  // namespace spmm
