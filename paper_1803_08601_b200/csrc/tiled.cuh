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
//              read once, 8 B per nonzero); a group loads G entries at a time (lane j: entry p + j),
//              broadcasts them with shuffles and gathers the B rows from shared memory (LDS.128).
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
    int c_vec4;     // C base 16-byte aligned and ldc % 4 == 0: float4 stores, else scalar
    EpiParams epi;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

template <typename T, int SR, int G, int NV, int RPG>
__global__ void __launch_bounds__(TL_THREADS, 2) k_tiled(const TiledParams P) {
    using R = Ring<T, SR>;
    constexpr int S = 32 / G;          // row groups per warp
    constexpr int U = G < 8 ? G : 8;   // entries per batch (B rows in flight per group)
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
    T acc[RPG][NV][4];
#pragma unroll
    for (int i = 0; i < RPG; ++i)
#pragma unroll
        for (int v = 0; v < NV; ++v)
#pragma unroll
            for (int x = 0; x < 4; ++x) acc[i][v][x] = R::id();

    const int nblocks = (P.k + kb - 1) / kb;
    const int chunks_per_row = P.b_vec4 ? (n >> 2) : n;
    // block b of B (rows [b kb, b kb + kb) ∩ [0, k)) into buffer (b & 1), all threads, one commit group
    auto load_block = [&](int b) {
        if (b < nblocks) {
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
        cp_async_wait1();  // block b has landed (block b + 1 may still be in flight)
        __syncthreads();
        const int k0 = b * kb;
        const int khi = k0 + kb;
        const uint32_t bs = sbase + (uint32_t)(b & 1) * buf_bytes - (uint32_t)k0 * (uint32_t)npad * 4u;
#pragma unroll
        for (int i = 0; i < RPG; ++i) {
            while (true) {
                // the group's next U entries of row i (lane gl < U: entry p + gl)
                const int idx = p[i] + gl;
                const bool ok = gl < U && idx < e[i];
                const int c = ok ? __ldg(colg + idx) : 0x7fffffff;
                const unsigned a = ok ? __ldg(valg + idx) : 0u;
                const unsigned inblk = __ballot_sync(FULL, c < khi);
                // entries of this block are a prefix of the remaining ones (sorted columns)
                const int cnt = __popc((inblk >> gbase) & ((1u << U) - 1u));
                unsigned bv[U][NV][4];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int cu = __shfl_sync(FULL, c, gbase + u);
#pragma unroll
                    for (int v = 0; v < NV; ++v)
                        lds_vpred<4>(bv[u][v], bs + ((uint32_t)cu * (uint32_t)npad + (uint32_t)cofs[v]) * 4u,
                                     u < cnt && colok[v]);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const T au = from_bits<T>(__shfl_sync(FULL, a, gbase + u));
                    if (u < cnt) {
#pragma unroll
                        for (int v = 0; v < NV; ++v)
#pragma unroll
                            for (int x = 0; x < 4; ++x) acc[i][v][x] = R::mac(acc[i][v][x], au, from_bits<T>(bv[u][v][x]));
                    }
                }
                p[i] += cnt;
                if (!__any_sync(FULL, cnt == U)) break;  // no group of the warp has more of this block
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
