// tiled.cuh -- A/B-tiled SpMM for dense-ish rows (the paper's future work,
// Greiner and Jacob show that once the nonzeros per row exceed m/M (M = fast memory),
// tiling A and B like a dense GEMM beats going across A and gathering B rows).
//
// The gather kernels read one 4n-byte B row from L2 per nonzero.  Above a few percent fill that is
// hundreds of GB of L2 traffic; here every B row is fetched from L2 once per ROW TILE instead:
//   CTA      = a tile of R consecutive rows; each row is owned by a group of G lanes (columns over the
//              lanes, float4) holding RPG rows' accumulators in registers for the whole kernel.
//   K loop   = B streamed through shared memory in blocks of KB rows (cp.async, double-buffered: block
//              kb + 2 loads while block kb is consumed), the B tile of the dense-GEMM analogy.
//   per block, every row advances a cursor over its (sorted) nonzeros: the entries with column < the
//              block end are a prefix of what is left (no search, no format conversion -- the CSR is
//              read once, 8 B per nonzero); a group caches U entries of each of its rows in registers
//              (lane j: entry p + j; the next batch is loaded while the current one is consumed), so a
//              block a row has no entries in costs one ballot; entries are broadcast with shuffles and
//              the B rows gathered from shared memory (LDS.128).
// Requires column indices non-decreasing within each row (checked at plan time) and n % 4 == 0.
#pragma once
#include "common.cuh"
#include "ptx.cuh"
#include "tile.cuh"  // lds_vpred

namespace spmm {

constexpr int TL_THREADS = 256;
#ifndef TL_BUF_BYTES
#define TL_BUF_BYTES 49152  // one B block buffer; two per CTA, two CTAs per SM
#endif

struct TiledParams {
    int m, n, k, nnz;
    const int* ro;
    const int* col;
    const void* val;
    const void* B;
    long long ldb;  // elements
    void* C;
    long long ldc;  // elements
    int kb;         // B rows per block
    int rows_per_cta;
    int b_vec4;     // B base 16-byte aligned and ldb % 4 == 0: 16-byte cp.async, else 4-byte
    int b_tma;      // b_vec4: B blocks arrive by TMA bulk copies (one per block when ldb == n, else one per row)
    int c_vec4;     // C base 16-byte aligned and ldc % 4 == 0: float4 stores, else scalar
    EpiParams epi;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

#ifndef TL_MINB
#define TL_MINB 2  // CTAs per SM the register allocation targets
#endif
#ifndef TL_UMAX
#define TL_UMAX 4  // entries per batch (B rows in flight per row group; 8 spills at 128 registers)
#endif

template <typename T, int SR, int G, int NV, int RPG>
__global__ void __launch_bounds__(TL_THREADS, TL_MINB) k_tiled(const TiledParams P) {
    using R = Ring<T, SR>;
    constexpr int S = 32 / G;          // row groups per warp
    constexpr int U = G < TL_UMAX ? G : TL_UMAX;  // entries per batch (B rows in flight per group)
    extern __shared__ __align__(16) unsigned char tl_smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int slot = lane / G;
    const int gl = lane % G;
    const int gbase = slot * G;  // first lane of this group
    const int n = P.n;
    const int npad = n;          // shared-memory B row pitch (elements; n % 4 == 0)
    const int kb = P.kb;
    const uint32_t sbase = smem_u32(tl_smem);
    const uint32_t buf_bytes = (uint32_t)kb * (uint32_t)npad * 4u;

    // this lane's columns: NV float4 blocks, block v at column (gl + v G) * 4
    int cofs[NV];
    bool colok[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        cofs[v] = (gl + v * G) * 4;
        colok[v] = cofs[v] < n;
    }

    // rows of this group
    const long long row0 = (long long)blockIdx.x * P.rows_per_cta + (long long)(warp * S + slot) * RPG;
    int p[RPG], e[RPG];
#pragma unroll
    for (int i = 0; i < RPG; ++i) {
        const long long r = row0 + i;
        p[i] = (r < P.m) ? __ldg(P.ro + r) : 0;
        e[i] = (r < P.m) ? __ldg(P.ro + r + 1) : 0;
    }
    // the cached batch of each row: lane gl < U holds entry p + gl (INT_MAX past the row end)
    int cc[RPG], off[RPG];
    unsigned ca[RPG];
#pragma unroll
    for (int i = 0; i < RPG; ++i) {
        const int idx = p[i] + gl;
        const bool ok = gl < U && idx < e[i];
        cc[i] = ok ? __ldg(P.col + idx) : 0x7fffffff;
        ca[i] = ok ? __ldg(static_cast<const unsigned*>(P.val) + idx) : 0u;
        off[i] = 0;
    }
    T acc[RPG][NV][4];
#pragma unroll
    for (int i = 0; i < RPG; ++i)
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int x = 0; x < 4; ++x) acc[i][v][x] = R::id();

    const int nblocks = (P.k + kb - 1) / kb;
    const int chunks_per_row = P.b_vec4 ? (n >> 2) : n;
    __shared__ __align__(8) uint64_t full[2];
    if (P.b_tma) {
        if (threadIdx.x == 0) {
            mbar_init(&full[0], 1);
            mbar_init(&full[1], 1);
            fence_mbar_init();
        }
        __syncthreads();
    }
    const uint64_t pol = policy_evict_last();  // B blocks are re-read by every row tile: keep them in L2
    // block b of B (rows [b kb, b kb + kb) ∩ [0, k)) into buffer (b & 1)
    auto load_block = [&](int b) {
        if (P.b_tma) {  // TMA: warp 0 issues, completion as transaction bytes on full[b & 1]
            if (b < nblocks && warp == 0) {
                const int k0 = b * kb;
                const int rows = min(kb, P.k - k0);
                const uint32_t rb = (uint32_t)n * 4u;
                unsigned char* dst0 = tl_smem + (size_t)(b & 1) * buf_bytes;
                const char* src0 = static_cast<const char*>(P.B) + (size_t)k0 * (size_t)P.ldb * 4u;
                if (lane == 0) {
                    fence_proxy_async_smem();
                    mbar_arrive_expect_tx(&full[b & 1], (uint32_t)rows * rb);
                }
                __syncwarp();
                if (P.ldb == n) {
                    if (lane == 0) tma_load_1d(dst0, src0, (uint32_t)rows * rb, &full[b & 1], pol);
                } else {
                    for (int r = lane; r < rows; r += 32)
                        tma_load_1d(dst0 + (size_t)r * rb, src0 + (size_t)r * (size_t)P.ldb * 4u, rb, &full[b & 1], pol);
                }
            }
            return;
        }
        if (b < nblocks) {  // cp.async by every thread, one commit group per block
            const int k0 = b * kb;
            const int rows = min(kb, P.k - k0);
            const uint32_t dst0 = sbase + (uint32_t)(b & 1) * buf_bytes;
            const int total = rows * chunks_per_row;
            for (int t = threadIdx.x; t < total; t += TL_THREADS) {
                const int r = t / chunks_per_row;
                const int c = t - r * chunks_per_row;
                const T* src = static_cast<const T*>(P.B) + (long long)(k0 + r) * P.ldb;
                if (P.b_vec4) cp_async16(dst0 + (uint32_t)(r * npad + c * 4) * 4u, src + c * 4);
                else cp_async4(dst0 + (uint32_t)(r * npad + c) * 4u, src + c);
            }
        }
        cp_async_commit();
    };
    load_block(0);
    load_block(1);
    const int* __restrict__ colg = P.col;
    const unsigned* __restrict__ valg = static_cast<const unsigned*>(P.val);
    for (int b = 0; b < nblocks; ++b) {
        if (P.b_tma) {
            mbar_wait(&full[b & 1], (uint32_t)((b >> 1) & 1));  // block b has landed
        } else {
            cp_async_wait1();  // block b has landed (block b + 1 may still be in flight)
            __syncthreads();
        }
        const int k0 = b * kb;
        const int khi = k0 + kb;
        const uint32_t bs = sbase + (uint32_t)(b & 1) * buf_bytes - (uint32_t)k0 * (uint32_t)npad * 4u;
#pragma unroll
        for (int i = 0; i < RPG; ++i) {
            while (true) {
                // lanes [off, U) of the cached batch are row i's next unconsumed entries; those in this block
                // are a prefix of them (sorted columns)
                const bool mine = gl >= off[i] && gl < U;
                const unsigned inblk = __ballot_sync(FULL, mine && cc[i] < khi);
                const int cnt = __popc((inblk >> gbase) & ((1u << U) - 1u));
                const bool full = off[i] + cnt == U && p[i] + U < e[i];  // batch used up, the row goes on
                int nc = 0x7fffffff;
                unsigned na = 0u;
                if (full) {  // next batch in flight while this one is consumed
                    const int idx = p[i] + U + gl;
                    if (gl < U && idx < e[i]) { nc = __ldg(colg + idx); na = __ldg(valg + idx); }
                }
                if (__any_sync(FULL, cnt > 0)) {
                    unsigned bv[U][NV][4];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int cu = __shfl_sync(FULL, cc[i], gbase + u);
                        const bool take = u >= off[i] && u < off[i] + cnt;
#pragma unroll
                        for (int v = 0; v < NV; ++v)
                            lds_vpred<4>(bv[u][v], bs + ((uint32_t)cu * (uint32_t)npad + (uint32_t)cofs[v]) * 4u,
                                         take && colok[v]);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const T au = from_bits<T>(__shfl_sync(FULL, ca[i], gbase + u));
                        if (u >= off[i] && u < off[i] + cnt) {
#pragma unroll
                            for (int v = 0; v < NV; ++v)
#pragma unroll
                                for (int x = 0; x < 4; ++x) acc[i][v][x] = R::mac(acc[i][v][x], au, from_bits<T>(bv[u][v][x]));
                        }
                    }
                }
                if (full) {
                    p[i] += U;
                    cc[i] = nc;
                    ca[i] = na;
                    off[i] = 0;
                } else {
                    off[i] += cnt;
                }
                if (!__any_sync(FULL, full)) break;  // no group of the warp has more of this block
            }
        }
        __syncthreads();  // every warp is done with buffer (b & 1)
        load_block(b + 2);
    }
    // finished rows -> C (epilogue: accumulate / peer copies when requested)
#pragma unroll
    for (int i = 0; i < RPG; ++i) {
        const long long r = row0 + i;
        if (r >= P.m) continue;
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            if (!colok[v]) continue;
            if (P.c_vec4) {
                unsigned o[4];
#pragma unroll
                for (int x = 0; x < 4; ++x) o[x] = to_bits<T>(acc[i][v][x]);
                epi_store<T, SR, 4>(P.epi, static_cast<T*>(P.C), P.ldc, r, cofs[v], o);
            } else {
#pragma unroll
                for (int x = 0; x < 4; ++x) {
                    unsigned o[1] = {to_bits<T>(acc[i][v][x])};
                    epi_store<T, SR, 1>(P.epi, static_cast<T*>(P.C), P.ldc, r, cofs[v] + x, o);
                }
            }
        }
    }
}

}  // namespace spmm
