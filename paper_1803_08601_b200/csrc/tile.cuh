// tile.cuh -- the sm_100a compute kernel shared by both of the paper's algorithms: a persistent,
// warp-specialised "tile engine".
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
// MODE_ROWSPLIT (Algorithm I, §4.1): a tile is a fixed block of rows; each row is owned by one group
//   of G lanes (G = ceil(n/VEC) rounded to a power of two, so a warp runs 32/G rows); no carries.
// MODE_MERGE (Algorithm II, §4.2): a tile is one CTA range of the merge-path partition (k_partition,
//   Alg. 1 line 2); each warp takes an equal share of the tile's items (rows + nonzeros) by a second
//   merge-path search in shared memory and streams them; carry-outs are resolved in the CTA and the
//   CTA's open row goes to the global carry array for k_fixup (Alg. 1 lines 22-24).
#pragma once
#include <type_traits>

#include "common.cuh"
#include "merge.cuh"
#include "ptx.cuh"

namespace spmm {

#ifndef TE_CWARPS_DEF
#define TE_CWARPS_DEF 8
#endif
constexpr int TE_CWARPS = TE_CWARPS_DEF;        // consumer warps
constexpr int TE_THREADS = 32 * (TE_CWARPS + 1);  // + 1 producer warp
constexpr int TE_CONSUMERS = 32 * TE_CWARPS;
#ifndef TE_MINB
#define TE_MINB 2  // row split: CTAs per SM the register allocation targets (__launch_bounds__)
#endif
#ifndef TE_MINB_MG
#define TE_MINB_MG 4  // merge: CTAs per SM (random gathers want many warps: TLP over ILP)
#endif
constexpr int TE_MAX_STAGES = 8;                // shared-memory pipeline depth limit (tiles in flight)
enum : int { MODE_ROWSPLIT = 0, MODE_MERGE = 1 };

struct TileParams {
    int m, n, nnz;
    const int* ro;
    const int* col;
    const void* val;
    const void* B;
    unsigned ldb_bytes;  // ldb * sizeof(T) (< 2^32)
    void* C;
    long long ldc;
    int num_ranges;     // rowsplit: row tiles; merge: partition CTAs
    int rows_per_tile;  // rowsplit
    const int* states;  // merge: (row, nz) per range boundary
    int items;          // merge: items per sub-tile (shared-memory capacity)
    int* carry_row;
    int* carry_flag;
    void* carry_val;
    int capr, capz;     // elements per buffer: row offsets / (col, val)
    unsigned pf_bytes;  // bytes of each B row to prefetch into L2 ahead of the consumers (0 = off)
    int stages;         // shared-memory pipeline depth (2..TE_MAX_STAGES)
    int capb;           // rowsplit: bytes per stage for the tile's B row span (0 = B is gathered from global)
    int* tile_ctr;      // merge, MG_DYN: global tile queue (zeroed by k_partition); null = static round robin
};

// tile descriptor written by the producer next to the staged data
struct TileInfo {
    int rs, zs, re, ze;  // merge-path state at tile start / end (rowsplit: zs = ro[rs], ze = ro[re])
    int ebase, zbase;    // global index of E[0] and of COL[0]/VAL[0]
    int range;           // partition range (merge) / row tile (rowsplit)
    int flags;           // 1 first sub-tile of range, 2 last sub-tile, 4 staged, 8 done, 16 B span staged
    int blo;             // flags & 16: B row held at the start of the staged B span
};

// one pipeline stage: row offsets | column indices | values | TileInfo (64 B) | B row span (capb bytes)
__host__ __device__ inline size_t te_buf_bytes(int capr, int capz, int elem, int capb = 0) {
    return (size_t)capr * 4 + (size_t)capz * 4 + (size_t)capz * elem + 64 + (size_t)capb;
}
constexpr int TE_BAR_BYTES = 24 * TE_MAX_STAGES;  // full / empty / csr-landed mbarriers
// nw = merge workers per CTA (consumer warps x row groups per warp); row split needs no carry slots,
// and every byte of shared memory it does not claim stays L1 (unified carveout) for B-row reuse
__host__ __device__ inline size_t te_smem_bytes(int capr, int capz, int elem, int n, int stages, int nw, bool merge,
                                                int capb = 0) {
    const size_t base = stages * te_buf_bytes(capr, capz, elem, capb) + TE_BAR_BYTES;
    if (!merge) return base;
    return base + (size_t)(nw + 1) * n * elem + (size_t)(nw + 1) * 8 + 64 +
           (size_t)stages * nw * n * elem + (size_t)stages * nw * 8 + stages * 4 + 64;
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

// 16-byte granule phase of a 4-byte element array (TMA copies of two arrays share an index base only
// when their phases agree)
__device__ __forceinline__ int te_phase(const void* p) { return (int)((reinterpret_cast<uintptr_t>(p) >> 2) & 3); }

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

template <typename T, int SR, int MODE, int VEC, int G, int NV, int U, bool PAIR>
__device__ __forceinline__ void tile_body(const TileParams& P) {
    using R = Ring<T, SR>;
    extern __shared__ __align__(128) unsigned char smem[];
    const int capr = P.capr, capz = P.capz, n = P.n, m = P.m;
    const size_t bufb = te_buf_bytes(capr, capz, (int)sizeof(T), MODE == MODE_ROWSPLIT ? P.capb : 0);
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
    T* Cw = reinterpret_cast<T*>(smem + NS * bufb + TE_BAR_BYTES);                 // [W+1][n] worker carries
    constexpr int NWK = TE_CWARPS * (32 / G);  // merge workers per CTA
    int* Crow = reinterpret_cast<int*>(Cw + (size_t)(NWK + 1) * n);  // [NWK+1]
    int* Cflag = Crow + (NWK + 1);                                   // [NWK+1]
    // per-stage worker carry slots for the barrier-free resolution of single-tile ranges
    T* CwS = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(Cflag + (NWK + 1)) + 64);  // [S][NWK][n]
    int* CrowS = reinterpret_cast<int*>(CwS + (size_t)NS * NWK * n);                   // [S][NWK]
    int* CflagS = CrowS + NS * NWK;                                                     // [S][NWK]
    int* Ccnt = CflagS + NS * NWK;                                                      // [S]

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
                const long long bytes = span * (long long)P.ldb_bytes;
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
        const bool bstage = MODE == MODE_ROWSPLIT && P.capb > 0;
        const bool val_tma = te_phase(P.col) == te_phase(P.val);
        int pend = -1;  // B staging: tile index whose CSR slice is in flight
        // tiles: static round robin, or (merge; row split with irregular rows) taken from a global queue
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
            long long rs, zs, re, ze;
            if (MODE == MODE_ROWSPLIT) {
                rs = (long long)c * P.rows_per_tile;
                re = min((long long)m, rs + P.rows_per_tile);
                zs = ld_stream(P.ro + rs);
                ze = ld_stream(P.ro + re);
            } else {
                rs = P.states[2 * c];
                zs = P.states[2 * c + 1];
                re = P.states[2 * c + 2];
                ze = P.states[2 * c + 3];
            }
            long long cr = rs, cz = zs;  // current sub-tile start
            bool first = true;
            while (true) {
                long long nr = re, nz = ze;
                if (MODE == MODE_MERGE && (re - cr) + (ze - cz) > P.items) {
                    // oversize range (1-D nonzero split with many rows): cut at diagonal +items
                    const long long D = cr + cz + P.items;
                    const long long lo = max(cr, D - ze), hi = min(D - cz, re);
                    nr = warp_search_first(lo, hi, MergePred{P.ro, D});
                    nz = D - nr;
                }
                const bool last = (nr == re && nz == ze);
                int b;
                acquire(b);
                uint64_t* csr_bar = bstage ? &landed[b] : &full[b];
                uint32_t ptx_tx = 0;  // lane 0: TMA bytes of a tile whose values the warp copies
                if (lane == 0) {
                    uint32_t tx = 0;
                    TileInfo inf;
                    inf.blo = 0;
                    inf.rs = (int)cr; inf.zs = (int)cz; inf.re = (int)nr; inf.ze = (int)nz;
                    inf.range = c;
                    bool staged;
                    fence_proxy_async_smem();
                    if (MODE == MODE_ROWSPLIT) {
                        staged = (nz - cz) + 8 <= capz;
                        inf.ebase = te_stage(E_of(b), P.ro, cr, nr + 1, (long long)m + 1, csr_bar, pol, &tx);
                    } else {
                        staged = true;
                        const long long e1 = min(nr + 1, (long long)m);  // row ends of rows cr..min(nr, m-1)
                        inf.ebase = te_stage(E_of(b), P.ro, cr + 1, e1 + 1, (long long)m + 1, &full[b], pol, &tx);
                    }
                    if (staged) {
                        inf.zbase = te_stage(COL_of(b), P.col, cz, nz, P.nnz, csr_bar, pol, &tx);
                        // values share the column indices' index base when both arrays have the same
                        // 16-byte phase (always for arrays sliced at the same offset); otherwise the
                        // warp copies them below with plain loads
                        if (val_tma) te_stage(VAL_of(b), P.val, cz, nz, P.nnz, csr_bar, pol, &tx);
                    } else {
                        inf.zbase = 0;
                    }
                    inf.flags = (first ? 1 : 0) | (last ? 2 : 0) | (staged ? 4 : 0);
                    *INFO_of(b) = inf;
                    if (val_tma || !staged) mbar_arrive_expect_tx(csr_bar, tx);
                    else ptx_tx = tx;
                }
                if (!val_tma) {
                    const TileInfo* ip = INFO_of(b);
                    __syncwarp();
                    if (ip->flags & 4) {
                        const int zb = ip->zbase;
                        for (long long p = cz + lane; p < nz; p += 32)
                            static_cast<unsigned*>(static_cast<void*>(VAL_of(b)))[p - zb] =
                                static_cast<const unsigned*>(P.val)[p];
                        __syncwarp();
                        if (lane == 0) mbar_arrive_expect_tx(csr_bar, ptx_tx);
                    }
                }
                __syncwarp();
                if (bstage) {
                    if (pend >= 0) finish_tile(pend % NS, pend);  // overlaps this tile's CSR load
                    pend = i;
                } else if (MODE == MODE_ROWSPLIT && P.pf_bytes && i >= 1) {
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
#ifndef MG_NA
#define MG_NA 1  // merge: accumulator sets per worker (1 measured 1-10% faster than 2 or 4)
#endif
#ifndef RS_NA
#define RS_NA 1  // row split: one accumulator set per row (measured 1-7% faster than 2 interleaved)
#endif
    constexpr int NA = (MODE == MODE_MERGE) ? ((VEC * NV <= 2) ? MG_NA : 2) : RS_NA;
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
    T* Cl = static_cast<T*>(P.C) + gl * VEC;
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
        T* crow = Cl + row * P.ldc;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            if (ok && colok[v]) {
                unsigned o[VEC];
#pragma unroll
                for (int x = 0; x < VEC; ++x) o[x] = to_bits<T>(acc.v[v][x]);
                st_vec<VEC>(crow + (cofs[v] - gl * VEC), o);
            }
        }
    };

    if (MODE == MODE_MERGE && threadIdx.x == 0) {
        Crow[NWK] = -1;
        Cflag[NWK] = 0;
        for (int s = 0; s < NS; ++s) Ccnt[s] = 0;
    }
    if (MODE == MODE_MERGE) named_bar_sync(1, TE_CONSUMERS);

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
                    const uint32_t vs = smem_u32(VAL) + 4u * (uint32_t)(s - inf.zbase);
                    for (int p0 = 0; p0 < maxlen; p0 += U) {
                        const int rem = len - p0;
                        unsigned bv[U][NV][VEC];
                        unsigned cu[U], av[U];
                        const bool full_b = rem >= U;
                        if (__all_sync(FULL, full_b && ((cs & 15u) == 0))) {  // full, 16B-aligned: LDS.128
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
            bool tile_done = false;
            if constexpr (PAIR) {
                auto pair_body = [&]() {
                    // Row pairs (B200 extension of §4.1), only for tiles whose B span is
                    // staged in shared memory: a group owns rows (2i, 2i+1) = (L, Q).  Q's entry j is
                    // matched with L's entry j + delta (delta = #{L cols < Q's first col}) when the two
                    // columns are equal; the B row read for L's entry then also feeds Q, so a banded pair
                    // reads 17 B rows into registers instead of 32.  Q's unmatched entries are read
                    // afterwards.  Every stored entry is used exactly once whatever the column order, so
                    // the result is C = AB for any CSR (sorted columns only make the matching effective).
                    constexpr bool kS = true;
                    const int pairs = (rows + 1) >> 1;
                    const int prounds = (pairs + NG - 1) / NG;
                    const uint32_t colz = smem_u32(COL) - 4u * (uint32_t)inf.zbase;  // + 4p: column of nonzero p
                    const uint32_t valz = smem_u32(VAL) - 4u * (uint32_t)inf.zbase;
                    const unsigned gbits = (G == 32) ? 0xffffffffu : ((1u << G) - 1u);
                    for (int t = 0; t < prounds; ++t) {
                        const int lr = 2 * (t * NG + gid);
                        const bool actL = lr < rows;
                        const bool actQ = lr + 1 < rows;
                        const int sL = actL ? E[inf.rs + lr - inf.ebase] : 0;
                        const int eL = actL ? E[inf.rs + lr + 1 - inf.ebase] : 0;
                        const int eQ = actQ ? E[inf.rs + lr + 2 - inf.ebase] : eL;
                        const int lenL = eL - sL, lenQ = eQ - eL;
                        if (!__all_sync(FULL, lenL <= 32 && lenQ <= 32)) {
                            // a long row in the warp: the two rows one after the other (plain row split)
#pragma unroll 1
                            for (int h = 0; h < 2; ++h) {
                                Acc<T, SR, VEC, NV> accs[NA];
#pragma unroll
                                for (int k = 0; k < NA; ++k) accs[k].reset();
                                row_pass(kS, h ? eL : sL, h ? lenQ : lenL, accs);
#pragma unroll
                                for (int k = 1; k < NA; ++k) accs[0].fold(accs[k]);
                                store_row(inf.rs + lr + h, accs[0], h ? actQ : actL);
                            }
                            continue;
                        }
                        const int maxL = __reduce_max_sync(FULL, lenL);
                        const int maxQ = __reduce_max_sync(FULL, lenQ);
                        // delta and the match mask, the group's lanes in parallel
                        const int q0 = (lenQ > 0) ? (int)lds_u32(colz + 4u * (uint32_t)eL) : 0x7fffffff;
                        int delta = 0;
                        for (int k0 = 0; k0 < maxL; k0 += G) {
                            const int i = k0 + gl;
                            const bool in = i < lenL;
                            const bool lt = in && (int)lds_pred(colz + 4u * (uint32_t)(sL + i), in) < q0;
                            delta += __popc((__ballot_sync(FULL, lt) >> (slot * G)) & gbits);
                        }
                        uint32_t mask = 0;  // bit j: Q's entry j is paired with L's entry j + delta
                        for (int k0 = 0; k0 < maxQ; k0 += G) {
                            const int j = k0 + gl;
                            const bool in = j < lenQ && j + delta < lenL;
                            const unsigned a = lds_pred(colz + 4u * (uint32_t)(eL + j), in);
                            const unsigned c = lds_pred(colz + 4u * (uint32_t)(sL + j + delta), in);
                            const unsigned bits = (__ballot_sync(FULL, in && a == c) >> (slot * G)) & gbits;
                            mask |= bits << k0;
                        }
                        Acc<T, SR, VEC, NV> accL, accQ;
                        accL.reset();
                        accQ.reset();
                        // L's batches in an order rotated by the group's slot (bank spread)
                        const int nb = (maxL + U - 1) / U;
                        int bb = slot % nb;
                        for (int bi = 0; bi < nb; ++bi) {
                            const int p0 = bb * U;
                            bb = (bb + 1 == nb) ? 0 : bb + 1;
                            const int rem = lenL - p0;
                            unsigned bv[U][NV][VEC];
                            unsigned cu[U], av[U], aq[U];
                            const uint32_t ca = colz + 4u * (uint32_t)(sL + p0);
                            const uint32_t va = valz + 4u * (uint32_t)(sL + p0);
                            // mask bits of Q entries p0 - delta .. p0 - delta + U - 1 (p0 - delta < 32)
                            const int j0 = p0 - delta;
                            const uint32_t mw = (j0 >= 0) ? (mask >> j0) : (j0 > -32 ? (mask << -j0) : 0u);
                            if (U % 4 == 0 && __all_sync(FULL, rem >= U && (ca & 15u) == 0)) {
                                // full batch for every group: unpredicated loads; Q's values are read
                                // unconditionally (eL + j0 + u >= sL stays inside the stage buffer) and
                                // used only where the mask says the entry is paired
#pragma unroll
                                for (int u = 0; u < U; u += 4) {
                                    const uint4 c4 = lds_u128(ca + 4u * u);
                                    const uint4 a4 = lds_u128(va + 4u * u);
                                    cu[u] = c4.x; cu[u + 1] = c4.y; cu[u + 2] = c4.z; cu[u + 3] = c4.w;
                                    av[u] = a4.x; av[u + 1] = a4.y; av[u + 2] = a4.z; av[u + 3] = a4.w;
                                }
#pragma unroll
                                for (int u = 0; u < U; ++u) aq[u] = lds_u32(valz + 4u * (uint32_t)(eL + j0 + u));
#pragma unroll
                                for (int u = 0; u < U; ++u) GF(kS, bv[u], (int)cu[u]);
#pragma unroll
                                for (int u = 0; u < U; ++u) {
                                    accL.mac(from_bits<T>(av[u]), bv[u]);
                                    if ((mw >> u) & 1u) accQ.mac(from_bits<T>(aq[u]), bv[u]);
                                }
                                continue;
                            }
#pragma unroll
                            for (int u = 0; u < U; ++u) {
                                cu[u] = lds_pred(ca + 4u * u, u < rem);
                                av[u] = lds_pred(va + 4u * u, u < rem);
                            }
#pragma unroll
                            for (int u = 0; u < U; ++u)
                                aq[u] = lds_pred(valz + 4u * (uint32_t)(eL + j0 + u), (mw >> u) & 1u);
#pragma unroll
                            for (int u = 0; u < U; ++u) GP(kS, bv[u], (int)cu[u], u < rem);
#pragma unroll
                            for (int u = 0; u < U; ++u) {
                                if (u < rem) accL.mac(from_bits<T>(av[u]), bv[u]);
                                if ((mw >> u) & 1u) accQ.mac(from_bits<T>(aq[u]), bv[u]);
                            }
                        }
                        // Q's entries without a partner
                        uint32_t todo = (lenQ >= 32 ? 0xffffffffu : ((1u << lenQ) - 1u)) & ~mask;
                        const int maxc = __reduce_max_sync(FULL, __popc(todo));
                        for (int c0 = 0; c0 < maxc; c0 += U) {
                            unsigned bv[U][NV][VEC];
                            unsigned aq[U];
                            bool ok[U];
#pragma unroll
                            for (int u = 0; u < U; ++u) {
                                ok[u] = todo != 0u;
                                const int j = ok[u] ? __ffs((int)todo) - 1 : 0;
                                todo &= todo - 1u;
                                const unsigned cq = lds_pred(colz + 4u * (uint32_t)(eL + j), ok[u]);
                                aq[u] = lds_pred(valz + 4u * (uint32_t)(eL + j), ok[u]);
                                if (c0 + u < maxc) GP(kS, bv[u], (int)cq, ok[u]);
                            }
#pragma unroll
                            for (int u = 0; u < U; ++u)
                                if (ok[u]) accQ.mac(from_bits<T>(aq[u]), bv[u]);
                        }
                        store_row(inf.rs + lr, accL, actL);
                        store_row(inf.rs + lr + 1, accQ, actQ);
                    }
                };
                if (staged && bsm) {  // pairs only from a staged B span (short latencies); else plain rows
                    pair_body();
                    tile_done = true;
                }
            }
            if (!tile_done) {
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
        } else {
            // ---------------- Algorithm II: merge-path items; a worker = a warp (G = 32) or, for
            // small n, a group of G lanes (32/G independent workers per warp, lane folding) ----------
            const int rs = inf.rs, zs = inf.zs, re = inf.re, ze = inf.ze;
            const int L = (re - rs) + (ze - zs);
            const int wid = warp * S + slot;  // worker id, ascending along the merge path
            const int per = (L + NWK - 1) / NWK;
            const int* Eb = E + 1 - inf.ebase;  // Eb[x] = ro[x+1] (row end of row x)
            auto search = [&](int d) -> int {
                const int D = rs + zs + d;
                int lo = max(rs, D - ze), hi = min(D - zs, re);
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (Eb[mid] <= D - mid - 1) lo = mid + 1; else hi = mid;
                }
                return lo;
            };
            const int d0 = min(wid * per, L), d1 = min((wid + 1) * per, L);
            const int ia = search(d0), ja = rs + zs + d0 - ia;
            const int ib = search(d1), jb = rs + zs + d1 - ib;

            Acc<T, SR, VEC, NV> accs[NA];  // NA interleaved partial sums: short FMA dependency chains
#pragma unroll
            for (int k = 1; k < NA; ++k) accs[k].reset();
            Acc<T, SR, VEC, NV>& acc = accs[0];
            bool dirty = false;
            if (wid == 0 && !(inf.flags & 1) && Cflag[NWK]) {  // carry-in from the previous sub-tile
#pragma unroll
                for (int v = 0; v < NV; ++v)
#pragma unroll
                    for (int x = 0; x < VEC; ++x) {
                        const int cc = cofs[v] + x;
                        acc.v[v][x] = (cc < n) ? Cw[NWK * n + cc] : R::id();
                    }
                dirty = true;
            } else {
                acc.reset();
            }
            int r = ia, q = ja;
            int e = (r < m) ? Eb[r] : 0x7fffffff;
            auto collapse = [&]() {
#pragma unroll
                for (int k = 1; k < NA; ++k) {
                    accs[0].fold(accs[k]);
                    accs[k].reset();
                }
            };
            auto flush = [&]() {
                collapse();
                store_row(r, acc, true);
                acc.reset();
                dirty = false;
                ++r;
                e = (r < m) ? Eb[r] : 0x7fffffff;
            };
          if constexpr (G == 32) {
            while (q < jb) {
                const int cnt = min(U, jb - q);
                unsigned bv[U][NV][VEC];
                T av[U];
                const uint32_t cs = smem_u32(COL) + 4u * (uint32_t)(q - inf.zbase);
                const uint32_t vs = smem_u32(VAL) + 4u * (uint32_t)(q - inf.zbase);
                unsigned cu[U], au[U];
                if (cnt == U && q + U <= e) {  // full batch inside the current row: no row end to check
                    if ((cs & 15u) == 0) {
#pragma unroll
                        for (int u = 0; u < U; u += 4) {
                            const uint4 c4 = lds_u128(cs + 4u * u);
                            const uint4 a4 = lds_u128(vs + 4u * u);
                            cu[u] = c4.x; cu[u + 1] = c4.y; cu[u + 2] = c4.z; cu[u + 3] = c4.w;
                            au[u] = a4.x; au[u + 1] = a4.y; au[u + 2] = a4.z; au[u + 3] = a4.w;
                        }
                    } else {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            cu[u] = lds_u32(cs + 4u * u);
                            au[u] = lds_u32(vs + 4u * u);
                        }
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) gather_full(bv[u], (int)cu[u]);
#pragma unroll
                    for (int u = 0; u < U; ++u) accs[u % NA].mac(from_bits<T>(au[u]), bv[u]);
                    dirty = true;
                    q += U;
                    continue;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    cu[u] = lds_pred(cs + 4u * u, u < cnt);
                    au[u] = lds_pred(vs + 4u * u, u < cnt);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    av[u] = from_bits<T>(au[u]);
                    gather(bv[u], (int)cu[u], u < cnt);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (u < cnt) {
                        while (e <= q + u) flush();  // rows ending before nonzero q+u (rows first on ties)
                        accs[u % NA].mac(av[u], bv[u]);
                        dirty = true;
                    }
                }
                q += cnt;
            }
            while (r < ib) flush();
          } else {
            // folded workers (small n): each G-lane group walks its own equal share of the merge path
            // item by item -- nonzero (gather + FMA) or row end (store C row, reset) -- all groups of
            // the warp in lock-step (equal item counts), item types predicated instead of branched
            constexpr int UF = (U < 8) ? U : 8;
            const int items = d1 - d0;
            const int steps = __reduce_max_sync(FULL, items);
            const uint32_t col_s = smem_u32(COL) - 4u * (uint32_t)inf.zbase;
            const uint32_t val_s = smem_u32(VAL) - 4u * (uint32_t)inf.zbase;
            for (int t0 = 0; t0 < steps; t0 += UF) {
                unsigned bv[UF][NV][VEC];
                unsigned au[UF];
                bool isn[UF], isr[UF];
                const int rstart = r;
#pragma unroll
                for (int u = 0; u < UF; ++u) {
                    const bool active = t0 + u < items;
                    isn[u] = active && (q < e);   // rows first on ties: row r ends before nonzero q if e <= q
                    isr[u] = active && !isn[u];
                    const unsigned c = lds_pred(col_s + 4u * (uint32_t)q, isn[u]);
                    au[u] = lds_pred(val_s + 4u * (uint32_t)q, isn[u]);
                    gather(bv[u], (int)c, isn[u]);
                    q += isn[u] ? 1 : 0;
                    if (isr[u]) {
                        ++r;
                        e = (r < m) ? Eb[r] : 0x7fffffff;
                    }
                }
                int rr = rstart;
#pragma unroll
                for (int u = 0; u < UF; ++u) {
                    if (isn[u]) {
                        acc.mac(from_bits<T>(au[u]), bv[u]);
                        dirty = true;
                    }
                    if (isr[u]) {
                        store_row(rr, acc, true);
                        acc.reset();
                        dirty = false;
                        ++rr;
                    }
                }
            }
          }
            collapse();

            // ---- carry resolution (Alg. 1 line 22): sums worker partials of the same row in ascending
            // worker order; rows whose end item lies in this sub-tile were already written by their
            // owner and get the sum added (RMW); the sub-tile's open row `re` is returned in `open`.
            auto resolve = [&](const T* slots, const int* srow, const int* sflag, T (&open)[4], bool& open_any) {
                open_any = false;
#pragma unroll
                for (int t2 = 0; t2 < 4; ++t2) open[t2] = R::id();
                int w = 0;
                while (w < NWK) {
                    const int row = srow[w];
                    bool any = false;
                    T sacc[4];
#pragma unroll
                    for (int t2 = 0; t2 < 4; ++t2) sacc[t2] = R::id();
                    int w2 = w;
                    while (w2 < NWK && srow[w2] == row) {
                        if (sflag[w2]) {
                            any = true;
#pragma unroll
                            for (int t2 = 0; t2 < 4; ++t2) {
                                const int cc = lane + 32 * t2;
                                if (cc < n) sacc[t2] = R::add(sacc[t2], slots[w2 * n + cc]);
                            }
                        }
                        ++w2;
                    }
                    if (row == re) {
                        open_any = any;
#pragma unroll
                        for (int t2 = 0; t2 < 4; ++t2) open[t2] = sacc[t2];
                    } else if (any && row < m) {
                        T* crow = static_cast<T*>(P.C) + (long long)row * P.ldc;
#pragma unroll
                        for (int t2 = 0; t2 < 4; ++t2) {
                            const int cc = lane + 32 * t2;
                            if (cc < n) crow[cc] = R::add(__ldcg(crow + cc), sacc[t2]);
                        }
                    }
                    w = w2;
                }
            };
            auto write_global_carry = [&](const T (&open)[4], bool open_any) {
                const int row = (re < m) ? re : -1;
                const bool any = (row >= 0) && open_any;
                if (lane == 0) { P.carry_row[inf.range] = row; P.carry_flag[inf.range] = any ? 1 : 0; }
                if (any) {
                    T* cv = static_cast<T*>(P.carry_val) + (long long)inf.range * n;
#pragma unroll
                    for (int t2 = 0; t2 < 4; ++t2) {
                        const int cc = lane + 32 * t2;
                        if (cc < n) cv[cc] = open[t2];
                    }
                }
            };
            auto publish = [&](T* slots, int* srow, int* sflag) {
                if (gl == 0) { srow[wid] = ib; sflag[wid] = dirty ? 1 : 0; }
                if (dirty) {
#pragma unroll
                    for (int v = 0; v < NV; ++v)
#pragma unroll
                        for (int x = 0; x < VEC; ++x) {
                            const int cc = cofs[v] + x;
                            if (colok[v] && cc < n) slots[wid * n + cc] = acc.v[v][x];
                        }
                }
            };

            if ((inf.flags & 3) == 3) {
                // whole range in one tile (2-D merge path): barrier-free -- the last worker to finish
                // resolves the carries, the others move straight on to their next tile
                T* slots = CwS + (size_t)b * NWK * n;
                int* srow = CrowS + b * NWK;
                int* sflag = CflagS + b * NWK;
                publish(slots, srow, sflag);
                // hand-off: __syncwarp orders the warp's slot writes before lane 0's acq_rel atomic
                // (release); the warp whose increment completes the count acquires every earlier
                // release and passes the ordering on to its lanes with __syncwarp
                __syncwarp();
                int last = 0;
                if (lane == 0) last = (smem_atom_add_acq_rel(&Ccnt[b], 1) == TE_CWARPS - 1) ? 1 : 0;
                last = __shfl_sync(FULL, last, 0);
                if (last) {
                    __syncwarp();
                    T open[4];
                    bool open_any;
                    resolve(slots, srow, sflag, open, open_any);
                    write_global_carry(open, open_any);
                    __syncwarp();
                    if (lane == 0) Ccnt[b] = 0;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[b]);  // buffer and slots of stage b are free
                continue;
            }

            // range split over several sub-tiles (1-D nonzero split with many rows): synchronous
            // resolution with a carry forwarded to the next sub-tile's first worker
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[b]);  // done reading this buffer
            publish(Cw, Crow, Cflag);
            named_bar_sync(1, TE_CONSUMERS);
            if (warp == 0) {
                T open[4];
                bool open_any;
                resolve(Cw, Crow, Cflag, open, open_any);
                __syncwarp();
                if (lane == 0) { Crow[NWK] = re; Cflag[NWK] = open_any ? 1 : 0; }
                if (open_any) {
#pragma unroll
                    for (int t2 = 0; t2 < 4; ++t2) {
                        const int cc = lane + 32 * t2;
                        if (cc < n) Cw[NWK * n + cc] = open[t2];
                    }
                }
                if (inf.flags & 2) write_global_carry(open, open_any);
            }
            named_bar_sync(1, TE_CONSUMERS);
        }
    }
}

template <typename T, int SR, int MODE, int VEC, int G, int NV, int U>
__global__ void __launch_bounds__(TE_THREADS, MODE == MODE_MERGE ? TE_MINB_MG : TE_MINB) k_tile(const TileParams P) {
    tile_body<T, SR, MODE, VEC, G, NV, U, false>(P);
}

#ifndef RSP_MAXREG
#define RSP_MAXREG 96  // 9 warps per CTA land 5/4 per SMSP: 2 CTAs per SM need <= 96 registers (64K per SMSP quarter)
#endif
template <typename T, int SR, int VEC, int G, int NV, int U>
__global__ void __maxnreg__(RSP_MAXREG) k_tile_pair(const TileParams P) {
    tile_body<T, SR, MODE_ROWSPLIT, VEC, G, NV, U, true>(P);
}

}  // namespace spmm
