// tile.cuh -- Algorithm I, row-splitting SpMM (§4.1), as a persistent,
// warp-specialised "tile engine" for sm_100a.  (Algorithm II, merge-based, is merge_w.cuh / merge_f.cuh.)
//
//   warp 8 (producer, one elected lane issues): walks this CTA's tiles, computes each tile's bounds
//     and stages the tile's slice of A -- row offsets, column indices, values -- into shared memory
//     with 1-D TMA bulk copies (cp.async.bulk, L2 evict-first), double-buffered, completion on a
//     transaction-count mbarrier.  This is the paper's GlobalToShared step (Alg. 1 line 5,
//     PAPER.md:146), made asynchronous so the next tile streams in while this one is computed.
//   warps 0..7 (consumers): read (col, val) pairs from shared memory as broadcasts (every lane of a
//     row group needs the same pair: the role of the paper's 32 `__shfl` broadcast rounds,
//     PAPER.md:122, Alg. 1 lines 14-17), gather B rows with lanes over columns (coalesced float4 /
//     float2 loads of row-major B), U gathers in flight before the first FMA (ILP,
//     PAPER.md:55-57), accumulate with packed FFMA2, and write finished rows of C with streaming stores.
//
// A tile is a fixed block of rows; each row is owned by one group of G lanes (G = ceil(n/VEC) rounded
// to a power of two, so a warp runs 32/G rows); no carries.
#pragma once
#include <type_traits>

#include "common.cuh"
#include "ptx.cuh"

namespace spmm {

#ifndef TE_CWARPS_DEF
#define TE_CWARPS_DEF 8
#endif
constexpr int TE_CWARPS = TE_CWARPS_DEF;        // consumer warps
constexpr int TE_THREADS = 32 * (TE_CWARPS + 1);  // + 1 producer warp
#ifndef TE_MINB
#define TE_MINB 2  // row split: CTAs per SM the register allocation targets (__launch_bounds__)
#endif
constexpr int TE_MAX_STAGES = 8;                // shared-memory pipeline depth limit (tiles in flight)
enum : int { MODE_ROWSPLIT = 0 };

struct TileParams {
    int m, n, nnz;
    const int* ro;
    const int* col;
    const void* val;
    const void* B;
    unsigned ldb_bytes;  // ldb * sizeof(T) (< 2^32)
    void* C;
    long long ldc;
    int num_ranges;     // row tiles
    int rows_per_tile;
    int capr, capz;     // elements per buffer: row offsets / (col, val)
    unsigned pf_bytes;  // bytes of each B row to prefetch into L2 ahead of the consumers (0 = off)
    int stages;         // shared-memory pipeline depth (2..TE_MAX_STAGES)
    int capb;           // rowsplit: bytes per stage for the tile's B row span (0 = B is gathered from global)
    int* tile_ctr;      // tile queue (irregular rows; zeroed before the launch); null = static round robin
    EpiParams epi;      // accumulate / peer copies of finished rows
};

// tile descriptor written by the producer next to the staged data
struct TileInfo {
    int rs, zs, re, ze;  // rows [rs, re) of the tile, nonzeros [zs = ro[rs], ze = ro[re])
    int ebase, zbase;    // global index of E[0] and of COL[0]
    int range;           // row tile
    int flags;           // 1 first sub-tile, 2 last sub-tile, 4 staged, 8 done, 16 B span staged
    int blo;             // flags & 16: B row held at the start of the staged B span
    int vbase;           // global index of VAL[0] (its own 16-byte phase: TMA copies align by address)
};

// one pipeline stage: row offsets | column indices | values | TileInfo (64 B) | B row span (capb bytes)
__host__ __device__ inline size_t te_buf_bytes(int capr, int capz, int elem, int capb = 0) {
    return (size_t)capr * 4 + (size_t)capz * 4 + (size_t)capz * elem + 64 + (size_t)capb;
}
constexpr int TE_BAR_BYTES = 24 * TE_MAX_STAGES;  // full / empty / csr-landed mbarriers
// every byte of shared memory the tile engine does not claim stays L1 (unified carveout) for B-row reuse
__host__ __device__ inline size_t te_smem_bytes(int capr, int capz, int elem, int stages, int capb = 0) {
    return stages * te_buf_bytes(capr, capz, elem, capb) + TE_BAR_BYTES;
}

// stage global src[begin, end) (4-byte elements, arr_len elements in the array) at dst; returns the
// global index of the element stored at dst[0] and adds TMA bytes to *tx.  The TMA copy covers the
// 16-byte aligned ADDRESS range around [begin, end) -- src itself may be any 4-byte aligned pointer
// (e.g. a row block sliced out of a larger CSR), so the returned index can be below begin (down to
// begin - 3, or -3 at the array start: same 16-byte granule, never another page).  The part past the
// array's last full granule is loaded with plain loads (never read past arr_len).
__device__ __forceinline__ int te_stage(void* dst, const void* src, long long begin, long long end, long long arr_len,
                                        uint64_t* bar, uint64_t pol, uint32_t* tx) {
    const long long mis = (long long)((reinterpret_cast<uintptr_t>(src) >> 2) & 3);  // elements past a granule
    const unsigned* srca = static_cast<const unsigned*>(src) - mis;                     // 16-byte aligned
    const long long a_al = (begin + mis) & ~3LL;  // indices into srca
    if (end <= begin) return (int)(a_al - mis);
    long long b_al = (end + mis + 3) & ~3LL;
    const long long lim = (arr_len + mis) & ~3LL;
    if (b_al > lim) b_al = lim;
    if (b_al > a_al) {
        const uint32_t bytes = (uint32_t)((b_al - a_al) * 4);
        tma_load_1d(dst, srca + a_al, bytes, bar, pol);
        *tx += bytes;
    }
    for (long long p = (b_al - mis > begin ? b_al - mis : begin); p < end; ++p)
        static_cast<unsigned*>(dst)[p + mis - a_al] = static_cast<const unsigned*>(src)[p];
    return (int)(a_al - mis);
}


// predicated vector gather of B (no branch): o valid only if pred
template <int VEC> __device__ __forceinline__ void ldg_pred(unsigned (&o)[VEC], const void* p, bool pred);
template <> __device__ __forceinline__ void ldg_pred<1>(unsigned (&o)[1], const void* p, bool pred) {
    asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; mov.b32 %0, 0; @q ld.global.nc.b32 %0, [%1];}"
                 : "=r"(o[0]) : "l"(p), "r"((int)pred));
}
template <> __device__ __forceinline__ void ldg_pred<2>(unsigned (&o)[2], const void* p, bool pred) {
    asm volatile("{.reg .pred q; setp.ne.b32 q, %3, 0; mov.b32 %0, 0; mov.b32 %1, 0; @q ld.global.nc.v2.b32 {%0, %1}, [%2];}"
                 : "=r"(o[0]), "=r"(o[1]) : "l"(p), "r"((int)pred));
}
template <> __device__ __forceinline__ void ldg_pred<4>(unsigned (&o)[4], const void* p, bool pred) {
    asm volatile("{.reg .pred q; setp.ne.b32 q, %5, 0; mov.b32 %0, 0; mov.b32 %1, 0; mov.b32 %2, 0; mov.b32 %3, 0;"
                 " @q ld.global.nc.v4.b32 {%0, %1, %2, %3}, [%4];}"
                 : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]) : "l"(p), "r"((int)pred));
}

// predicated vector load from shared memory (o = 0 if !pred; no access)
template <int VEC> __device__ __forceinline__ void lds_vpred(unsigned (&o)[VEC], uint32_t a, bool pred);
template <> __device__ __forceinline__ void lds_vpred<1>(unsigned (&o)[1], uint32_t a, bool pred) {
    asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; mov.b32 %0, 0; @q ld.shared.b32 %0, [%1];}"
                 : "=r"(o[0]) : "r"(a), "r"((int)pred));
}
template <> __device__ __forceinline__ void lds_vpred<2>(unsigned (&o)[2], uint32_t a, bool pred) {
    asm volatile("{.reg .pred q; setp.ne.b32 q, %3, 0; mov.b32 %0, 0; mov.b32 %1, 0; @q ld.shared.v2.b32 {%0, %1}, [%2];}"
                 : "=r"(o[0]), "=r"(o[1]) : "r"(a), "r"((int)pred));
}
template <> __device__ __forceinline__ void lds_vpred<4>(unsigned (&o)[4], uint32_t a, bool pred) {
    asm volatile("{.reg .pred q; setp.ne.b32 q, %5, 0; mov.b32 %0, 0; mov.b32 %1, 0; mov.b32 %2, 0; mov.b32 %3, 0;"
                 " @q ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];}"
                 : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]) : "r"(a), "r"((int)pred));
}


// accumulator of VEC*NV columns for one lane
template <typename T, int SR, int VEC, int NV> struct Acc {
    T v[NV][VEC];
    __device__ __forceinline__ void reset() {
#pragma unroll
        for (int a = 0; a < NV; ++a)
#pragma unroll
            for (int x = 0; x < VEC; ++x) v[a][x] = Ring<T, SR>::id();
    }
    __device__ __forceinline__ void fold(const Acc& o) {  // this (+)= o
#pragma unroll
        for (int a = 0; a < NV; ++a)
#pragma unroll
            for (int x = 0; x < VEC; ++x) v[a][x] = Ring<T, SR>::add(v[a][x], o.v[a][x]);
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

template <typename T, int SR, int MODE, int VEC, int G, int NV, int U>
__device__ __forceinline__ void tile_body(const TileParams& P) {
    using R = Ring<T, SR>;
    extern __shared__ __align__(128) unsigned char smem[];
    const int capr = P.capr, capz = P.capz, n = P.n, m = P.m;
    const size_t bufb = te_buf_bytes(capr, capz, (int)sizeof(T), P.capb);
    auto E_of = [&](int b) { return reinterpret_cast<int*>(smem + b * bufb); };
    auto COL_of = [&](int b) { return reinterpret_cast<int*>(smem + b * bufb + (size_t)capr * 4); };
    auto VAL_of = [&](int b) { return reinterpret_cast<T*>(smem + b * bufb + (size_t)capr * 4 + (size_t)capz * 4); };
    auto INFO_of = [&](int b) {
        return reinterpret_cast<TileInfo*>(smem + b * bufb + (size_t)capr * 4 + (size_t)capz * (4 + sizeof(T)));
    };
    auto BS_of = [&](int b) { return smem + b * bufb + (size_t)capr * 4 + (size_t)capz * (4 + sizeof(T)) + 64; };
    const int NS = P.stages;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * bufb);
    uint64_t* empty = full + TE_MAX_STAGES;
    uint64_t* landed = empty + TE_MAX_STAGES;  // rowsplit + B staging: the tile's CSR slice has landed

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], TE_CWARPS);
            mbar_init(&landed[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();

    // =============================== producer warp ===============================
    if (warp == TE_CWARPS) {
        const uint64_t pol = policy_evict_first();
        int i = 0;
        auto acquire = [&](int& b) {
            b = i % NS;
            if (i >= NS) {
                while (!mbar_try_wait(&empty[b], ((i / NS) - 1) & 1)) __nanosleep(64);
            }
        };
        auto prefetch_span = [&](int lo, long long span) {
            const char* base = static_cast<const char*>(P.B) + (size_t)(unsigned)lo * P.ldb_bytes;
            const long long bytes = (span - 1) * (long long)P.ldb_bytes + P.pf_bytes;
            constexpr long long CHUNK = 16384;
            for (long long off = (long long)lane * CHUNK; off < bytes; off += 32 * CHUNK) {
                const long long len = min(CHUNK, bytes - off);
                prefetch_l2_bulk(base + off, (uint32_t)(len & ~15LL));
            }
        };
        // L2 prefetch of the B rows a staged tile will gather, when the tile's columns are clustered
        // (banded / mesh-like matrices): one TMA bulk prefetch (cp.async.bulk.prefetch.L2) of the
        // tile's B row span, issued once the tile's column indices have landed in shared memory, so
        // the consumers' first-touch gathers hit L2 instead of paying a DRAM round trip.
        auto prefetch_tile_b = [&](int pb, int ti) {
            mbar_wait(&full[pb], (ti / NS) & 1);
            const TileInfo pi = *INFO_of(pb);
            if (!(pi.flags & 4)) return;
            const int cnt = pi.ze - pi.zs;
            if (cnt <= 0) return;
            const int* pc = COL_of(pb) + (pi.zs - pi.zbase);
            int lo = 0x7fffffff, hi = -1;
            for (int t = lane; t < cnt; t += 32) {
                const int c = pc[t];
                lo = min(lo, c);
                hi = max(hi, c);
            }
            lo = __reduce_min_sync(FULL, lo);
            hi = __reduce_max_sync(FULL, hi);
            const long long span = (long long)hi - lo + 1;
            if (span > 2LL * cnt) return;  // scattered columns: nothing compact to prefetch
            prefetch_span(lo, span);
        };
        // B staging (row split, P.capb > 0): once tile ti's CSR slice has landed (`landed` barrier), the
        // producer finds the tile's B row span [lo, hi] and, when it is compact (at most 2 rows per
        // nonzero) and fits the stage, copies those B rows into shared memory with one TMA bulk copy
        // that completes on the consumers' `full` barrier.  The consumers then gather B rows from
        // shared memory (no DRAM / L2 latency left in their dependency chain); other tiles keep the
        // global gathers (+ L2 prefetch when the span is compact but too large).
        const uint64_t polb = policy_evict_last();
        auto finish_tile = [&](int pb, int ti) {
            mbar_wait(&landed[pb], (ti / NS) & 1);
            TileInfo* ip = INFO_of(pb);
            const TileInfo pi = *ip;
            __syncwarp();  // every lane has read the descriptor before lane 0 updates it below
            uint32_t btx = 0;
            const int cnt = pi.ze - pi.zs;
            if ((pi.flags & 4) && cnt > 0) {
                const int* pc = COL_of(pb) + (pi.zs - pi.zbase);
                int lo = 0x7fffffff, hi = -1;
                for (int t = lane; t < cnt; t += 32) {
                    const int c = pc[t];
                    lo = min(lo, c);
                    hi = max(hi, c);
                }
                lo = __reduce_min_sync(FULL, lo);
                hi = __reduce_max_sync(FULL, hi);
                const long long span = (long long)hi - lo + 1;
                // rows lo..hi at pitch ldb, the last one only up to column n (never past B's last
                // element; B staging is planned only when n * sizeof(T) is a multiple of 16)
                const long long bytes = (span - 1) * (long long)P.ldb_bytes + (long long)n * (long long)sizeof(T);
                if (span <= 2LL * cnt && bytes <= P.capb) {
                    if (lane == 0) {
                        fence_proxy_async_smem();
                        tma_load_1d(BS_of(pb), static_cast<const char*>(P.B) + (size_t)(unsigned)lo * P.ldb_bytes,
                                    (uint32_t)bytes, &full[pb], polb);
                        ip->flags = pi.flags | 16;
                        ip->blo = lo;
                    }
                    btx = (uint32_t)bytes;
                } else if (span <= 2LL * cnt && P.pf_bytes) {
                    prefetch_span(lo, span);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive_expect_tx(&full[pb], btx);
        };
        const bool bstage = P.capb > 0;
        int pend = -1;  // B staging: tile index whose CSR slice is in flight
        // tiles: static round robin, or (irregular rows) taken from a global queue
        // so CTAs that finish early take more of the variable-cost tiles
        auto next_tile = [&](int cur) -> int {
            if (P.tile_ctr) {
                int nx = 0;
                if (lane == 0) nx = atomicAdd(P.tile_ctr, 1);
                return __shfl_sync(FULL, nx, 0);
            }
            return cur < 0 ? (int)blockIdx.x : cur + (int)gridDim.x;
        };
        for (int c = next_tile(-1); c < P.num_ranges; c = next_tile(c)) {
            const long long rs = (long long)c * P.rows_per_tile;
            const long long re = min((long long)m, rs + P.rows_per_tile);
            const long long zs = ld_stream(P.ro + rs);
            const long long ze = ld_stream(P.ro + re);
            long long cr = rs, cz = zs;  // current sub-tile start
            bool first = true;
            while (true) {
                const long long nr = re, nz = ze;
                const bool last = (nr == re && nz == ze);
                int b;
                acquire(b);
                uint64_t* csr_bar = bstage ? &landed[b] : &full[b];
                if (lane == 0) {
                    uint32_t tx = 0;
                    TileInfo inf;
                    inf.blo = 0;
                    inf.rs = (int)cr; inf.zs = (int)cz; inf.re = (int)nr; inf.ze = (int)nz;
                    inf.range = c;
                    fence_proxy_async_smem();
                    const bool staged = (nz - cz) + 8 <= capz;
                    inf.ebase = te_stage(E_of(b), P.ro, cr, nr + 1, (long long)m + 1, csr_bar, pol, &tx);
                    if (staged) {
                        inf.zbase = te_stage(COL_of(b), P.col, cz, nz, P.nnz, csr_bar, pol, &tx);
                        // the values get their own index base: the two arrays may sit at different
                        // 16-byte phases (views at arbitrary offsets), and TMA copies align by address
                        inf.vbase = te_stage(VAL_of(b), P.val, cz, nz, P.nnz, csr_bar, pol, &tx);
                    } else {
                        inf.zbase = 0;
                        inf.vbase = 0;
                    }
                    inf.flags = (first ? 1 : 0) | (last ? 2 : 0) | (staged ? 4 : 0);
                    *INFO_of(b) = inf;
                    mbar_arrive_expect_tx(csr_bar, tx);
                }
                __syncwarp();
                if (bstage) {
                    if (pend >= 0) finish_tile(pend % NS, pend);  // overlaps this tile's CSR load
                    pend = i;
                } else if (P.pf_bytes && i >= 1) {
                    prefetch_tile_b((i - 1) % NS, i - 1);
                }
                ++i;
                first = false;
                if (last) break;
                cr = nr;
                cz = nz;
            }
        }
        if (pend >= 0) finish_tile(pend % NS, pend);
        int b;
        acquire(b);
        if (lane == 0) {
            TileInfo inf{};
            inf.flags = 8;  // done
            *INFO_of(b) = inf;
            mbar_arrive(&full[b]);
        }
        return;
    }

    // =============================== consumer warps ===============================
    constexpr int S = 32 / G;
#ifndef RS_NA
#define RS_NA 1  // row split: one accumulator set per row (measured 1-7% faster than 2 interleaved)
#endif
    constexpr int NA = RS_NA;
    const int slot = lane / G;
    const int gl = lane - slot * G;
    bool colok[NV];
    // column offset of this lane's v-th vector block; the blocks are rotated by the group's slot so
    // that groups reading different B rows at the same time cover different shared-memory banks
    // when a group's block is narrower than 128 B (G * VEC < 32)
    int cofs[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) cofs[v] = gl * VEC + ((v + slot) % NV) * G * VEC;
#pragma unroll
    for (int v = 0; v < NV; ++v) colok[v] = cofs[v] < n;
    // per-lane B base of each column block; lanes past n read column 0 of the same row instead
    // (valid memory, never stored), so the gathers need no column predicate or branch
    const char* Blv[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v)
        Blv[v] = opaque_ptr(static_cast<const char*>(P.B) +
                            (colok[v] ? (size_t)cofs[v] * sizeof(T) : (size_t)0));
    const char* Bl = Blv[0];
    uint32_t boff[NV];  // byte offset of this lane's column block inside a B row (staged B span)
#pragma unroll
    for (int v = 0; v < NV; ++v) boff[v] = colok[v] ? (uint32_t)(cofs[v] * sizeof(T)) : 0u;
    const unsigned ldb_bytes = P.ldb_bytes;

    auto gather = [&](unsigned (&o)[NV][VEC], int c, bool ok) {
#pragma unroll
        for (int v = 0; v < NV; ++v) ldg_pred<VEC>(o[v], Blv[v] + (size_t)(unsigned)c * ldb_bytes, ok);
    };
    auto gather_full = [&](unsigned (&o)[NV][VEC], int c) {
#pragma unroll
        for (int v = 0; v < NV; ++v) ldg_vec<VEC>(o[v], Blv[v] + (size_t)(unsigned)c * ldb_bytes);
    };
    auto store_row = [&](long long row, const Acc<T, SR, VEC, NV>& acc, bool ok) {
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            if (ok && colok[v]) {
                unsigned o[VEC];
#pragma unroll
                for (int x = 0; x < VEC; ++x) o[x] = to_bits<T>(acc.v[v][x]);
                epi_store<T, SR, VEC>(P.epi, static_cast<T*>(P.C), P.ldc, row, cofs[v], o);
            }
        }
    };


    for (int i = 0;; ++i) {
        const int b = i % NS;
        mbar_wait(&full[b], (i / NS) & 1);
        const TileInfo inf = *INFO_of(b);
        if (inf.flags & 8) break;
        const int* E = E_of(b);
        const int* COL = COL_of(b);
        const T* VAL = VAL_of(b);
        const bool staged = inf.flags & 4;

        if (MODE == MODE_ROWSPLIT) {
            // ---------------- Algorithm I: rows of the tile, one row per G-lane group ----------------
            const int rows = inf.re - inf.rs;
            const int NG = TE_CWARPS * S;
            const int gid = warp * S + slot;
            // one row's entries [s, s + len) into accs; every group of the warp runs the same trip count
            // (B rows gathered from shared memory when the tile's B span is staged, else from global)
            const bool bsm = inf.flags & 16;
            const uint32_t bsb = smem_u32(BS_of(b)) - (uint32_t)inf.blo * ldb_bytes;
            auto sgather = [&](unsigned (&o)[NV][VEC], int c, bool ok) {
#pragma unroll
                for (int v = 0; v < NV; ++v) lds_vpred<VEC>(o[v], bsb + (uint32_t)c * ldb_bytes + boff[v], ok);
            };
            auto sgather_full = [&](unsigned (&o)[NV][VEC], int c) {
#pragma unroll
                for (int v = 0; v < NV; ++v) lds_vec<VEC>(o[v], bsb + (uint32_t)c * ldb_bytes + boff[v]);
            };
            auto GF = [&](const bool kS, unsigned (&o)[NV][VEC], int c) {
                if (kS) sgather_full(o, c); else gather_full(o, c);
            };
            auto GP = [&](const bool kS, unsigned (&o)[NV][VEC], int c, bool ok) {
                if (kS) sgather(o, c, ok); else gather(o, c, ok);
            };
            auto row_pass = [&](const bool kS, const int s, const int len, Acc<T, SR, VEC, NV>(&accs)[NA]) {
                const int maxlen = __reduce_max_sync(FULL, len);
                if (staged) {
                    const uint32_t cs = smem_u32(COL) + 4u * (uint32_t)(s - inf.zbase);
                    const uint32_t vs = smem_u32(VAL) + 4u * (uint32_t)(s - inf.vbase);
                    for (int p0 = 0; p0 < maxlen; p0 += U) {
                        const int rem = len - p0;
                        unsigned bv[U][NV][VEC];
                        unsigned cu[U], av[U];
                        const bool full_b = rem >= U;
                        if (__all_sync(FULL, full_b && (((cs | vs) & 15u) == 0))) {  // full, 16B-aligned: LDS.128
#pragma unroll
                            for (int u = 0; u < U; u += 4) {
                                const uint4 c4 = lds_u128(cs + 4u * (p0 + u));
                                const uint4 a4 = lds_u128(vs + 4u * (p0 + u));
                                cu[u] = c4.x; cu[u + 1] = c4.y; cu[u + 2] = c4.z; cu[u + 3] = c4.w;
                                av[u] = a4.x; av[u + 1] = a4.y; av[u + 2] = a4.z; av[u + 3] = a4.w;
                            }
#pragma unroll
                            for (int u = 0; u < U; ++u) GF(kS, bv[u], (int)cu[u]);
#pragma unroll
                            for (int u = 0; u < U; ++u) accs[u % NA].mac(from_bits<T>(av[u]), bv[u]);
                            continue;
                        }
                        if (__all_sync(FULL, full_b)) {  // full batch for every group of the warp
#pragma unroll
                            for (int u = 0; u < U; ++u) {
                                cu[u] = lds_u32(cs + 4u * (p0 + u));
                                av[u] = lds_u32(vs + 4u * (p0 + u));
                            }
#pragma unroll
                            for (int u = 0; u < U; ++u) GF(kS, bv[u], (int)cu[u]);
#pragma unroll
                            for (int u = 0; u < U; ++u) accs[u % NA].mac(from_bits<T>(av[u]), bv[u]);
                            continue;
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            cu[u] = lds_pred(cs + 4u * (p0 + u), u < rem);
                            av[u] = lds_pred(vs + 4u * (p0 + u), u < rem);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) GP(kS, bv[u], (int)cu[u], u < rem);
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            if (u < rem) accs[u % NA].mac(from_bits<T>(av[u]), bv[u]);
                    }
                } else {  // tile too large for the staged slice (long rows): stream A from global
                    const int* cg = P.col + s;
                    const unsigned* vg = static_cast<const unsigned*>(P.val) + s;
                    for (int p0 = 0; p0 < maxlen; p0 += U) {
                        const int rem = len - p0;
                        unsigned bv[U][NV][VEC];
                        unsigned cu[U], av[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            cu[u] = ldg_stream_pred(cg + p0 + u, u < rem);
                            av[u] = ldg_stream_pred(vg + p0 + u, u < rem);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) GP(kS, bv[u], (int)cu[u], u < rem);
#pragma unroll
                        for (int u = 0; u < U; ++u)
                            if (u < rem) accs[u % NA].mac(from_bits<T>(av[u]), bv[u]);
                    }
                }
            };
            {
                const int rounds = (rows + NG - 1) / NG;
                for (int t = 0; t < rounds; ++t) {
                    const int lr = t * NG + gid;
                    const bool active = lr < rows;
                    const int s = active ? E[inf.rs + lr - inf.ebase] : 0;
                    const int e = active ? E[inf.rs + lr + 1 - inf.ebase] : 0;
                    Acc<T, SR, VEC, NV> accs[NA];  // NA interleaved partial sums: short FMA dependency chains
#pragma unroll
                    for (int k = 0; k < NA; ++k) accs[k].reset();
                    if (bsm) row_pass(true, s, e - s, accs);
                    else row_pass(false, s, e - s, accs);
#pragma unroll
                    for (int k = 1; k < NA; ++k) accs[0].fold(accs[k]);
                    store_row(inf.rs + lr, accs[0], active);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[b]);
        }
    }
}

template <typename T, int SR, int MODE, int VEC, int G, int NV, int U>
__global__ void __launch_bounds__(TE_THREADS, TE_MINB) k_tile(const TileParams P) {
    tile_body<T, SR, MODE, VEC, G, NV, U>(P);
}

}  // namespace spmm
