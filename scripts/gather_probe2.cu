// gather_probe2.cu -- microbenchmark (not product code): how to keep enough 256-byte B-row gathers in
// flight on B200 for the merge kernel's R-MAT regime (VERDICT r01 "what's weak" 3), and what an L2
// hot/cold policy buys.  Each warp walks a slice of an index stream (R-MAT column marginal: every one of
// L index bits is 1 with probability 0.24, the Graph500 b + d) and sums the gathered 256-byte rows.
//
//   ldg<U>      U gathers (LDG.64, lanes over the 64 floats of a row) in flight per warp, then sum
//   ldgsts<D>   per-warp ring of D batches of 8 rows filled with cp.async (LDGSTS.128, 16 lanes per row),
//               D-1 batches in flight while one is summed from shared memory
//   bulk<D,R>   per-warp ring of D batches of R rows; lane r < R issues one cp.async.bulk (TMA, 256 B)
//               for row r of the batch, completion on one mbarrier per batch
//   policy: 0 default, 1 evict_first on every gather, 2 evict_last on "hot" rows (popcount(idx) <= H)
//           and evict_first on the rest
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gp2 scripts/gather_probe2.cu
// Run:   /tmp/gp2 <levels 22|26> <n_indices>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

__global__ void gen_idx(int* idx, long long n, int levels, uint32_t seed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        uint32_t c = 0;
        for (int l = 0; l < levels; ++l) {
            const uint32_t h = hash32((uint32_t)i * 0x9E3779B1u ^ hash32((uint32_t)(i >> 32) + l * 0x85ebca6bu + seed));
            c = (c << 1) | (h < 1030792151u ? 1u : 0u);  // 0.24 * 2^32
        }
        idx[i] = (int)c;
    }
}

__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p; asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ uint64_t pol_last() {
    uint64_t p; asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p)); return p;
}
__device__ __forceinline__ float2 ldg_pol(const float2* p, uint64_t pol) {
    float2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(p), "l"(pol));
    return v;
}

template <int U, int POL>
__global__ void __launch_bounds__(256) k_ldg(const int* __restrict__ idx, long long n, const float2* __restrict__ B,
                                               float2* out, int hot) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long per = (n + nw - 1) / nw;
    const long long b = warp * per, e = min(n, b + per);
    const uint64_t pf = pol_first(), pl = pol_last();
    float2 acc = make_float2(0.f, 0.f);
    for (long long p = b; p < e; p += 32) {
        const int myidx = (p + lane < e) ? __ldg(idx + p + lane) : 0;
        const int cnt = (int)min(32LL, e - p);
        for (int u0 = 0; u0 < cnt; u0 += U) {
            float2 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = __shfl_sync(0xffffffffu, myidx, (u0 + u) & 31);
                const float2* a = B + (long long)c * 32 + lane;
                if (u0 + u < cnt) {
                    if (POL == 0) v[u] = __ldg(a);
                    else if (POL == 1) v[u] = ldg_pol(a, pf);
                    else v[u] = ldg_pol(a, __popc(c) <= hot ? pl : pf);
                } else {
                    v[u] = make_float2(0.f, 0.f);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; }
        }
    }
    out[warp * 32 + lane] = acc;
}

// ---- LDGSTS ring: 8 rows per batch, D batches per warp; lanes 0-15 copy row 2j, 16-31 row 2j+1 (16 B each)
template <int D, int POL>
__global__ void __launch_bounds__(256) k_ldgsts(const int* __restrict__ idx, long long n, const float2* __restrict__ B,
                                                  float2* out, int hot) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    float2* ring = reinterpret_cast<float2*>(sm) + (size_t)wib * D * 8 * 32;  // [D][8 rows][32 float2]
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long per = (n + nw - 1) / nw;
    const long long b = warp * per, e = min(n, b + per);
    const long long nb = (e > b) ? (e - b + 7) / 8 : 0;
    float2 acc = make_float2(0.f, 0.f);
    const int half = lane >> 4, hl = lane & 15;
    auto issue = [&](long long bi) {
        const int slot = (int)(bi % D);
        const long long p0 = b + bi * 8;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const long long q = p0 + 2 * j + half;
            const int c = (q < e) ? __ldg(idx + q) : 0;
            const float4* src = reinterpret_cast<const float4*>(B + (long long)c * 32) + hl;
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + ((size_t)slot * 8 + 2 * j + half) * 32) + hl * 16;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (long long bi = 0; bi < D - 1; ++bi) {
        if (bi < nb) issue(bi); else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (long long bi = 0; bi < nb; ++bi) {
        if (bi + D - 1 < nb) issue(bi + D - 1); else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        __syncwarp();
        const int slot = (int)(bi % D);
        const int cnt = (int)min(8LL, e - (b + bi * 8));
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            if (r < cnt) {
                const float2 v = ring[((size_t)slot * 8 + r) * 32 + lane];
                acc.x += v.x; acc.y += v.y;
            }
        }
        __syncwarp();
    }
    out[warp * 32 + lane] = acc;
}

// ---- TMA bulk ring: R rows per batch, D batches per warp, one mbarrier per batch
template <int D, int R, int POL>
__global__ void __launch_bounds__(256) k_bulk(const int* __restrict__ idx, long long n, const float2* __restrict__ B,
                                                float2* out, int hot) {
    extern __shared__ __align__(128) unsigned char sm[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int nwb = blockDim.x >> 5;
    float2* ring = reinterpret_cast<float2*>(sm) + (size_t)wib * D * R * 32;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + (size_t)nwb * D * R * 256) + wib * D;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long per = (n + nw - 1) / nw;
    const long long b = warp * per, e = min(n, b + per);
    const long long nb = (e > b) ? (e - b + R - 1) / R : 0;
    const uint64_t pf = pol_first(), pl = pol_last();
    if (lane < D) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(bars + lane)));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    float2 acc = make_float2(0.f, 0.f);
    auto issue = [&](long long bi) {
        const int slot = (int)(bi % D);
        const long long p0 = b + bi * R;
        const int cnt = (int)min((long long)R, e - p0);
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(bars + slot);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(cnt * 256) : "memory");
        __syncwarp();
        if (lane < cnt) {
            const int c = __ldg(idx + p0 + lane);
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + ((size_t)slot * R + lane) * 32);
            const float2* src = B + (long long)c * 32;
            if (POL == 0) {
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                             ::"r"(dst), "l"(src), "r"(bar) : "memory");
            } else {
                const uint64_t pol = (POL == 1) ? pf : (__popc(c) <= hot ? pl : pf);
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], 256, [%2], %3;"
                             ::"r"(dst), "l"(src), "r"(bar), "l"(pol) : "memory");
            }
        }
    };
    for (long long bi = 0; bi < D - 1 && bi < nb; ++bi) issue(bi);
    for (long long bi = 0; bi < nb; ++bi) {
        if (bi + D - 1 < nb) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(bi + D - 1);
        }
        const int slot = (int)(bi % D);
        const uint32_t bar = (uint32_t)__cvta_generic_to_shared(bars + slot);
        const uint32_t par = (uint32_t)((bi / D) & 1);
        uint32_t ok = 0;
        long long spins = 0;
        while (!ok) {
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}"
                         : "=r"(ok) : "r"(bar), "r"(par) : "memory");
            if (++spins > (1LL << 26)) __trap();
        }
        const int cnt = (int)min((long long)R, e - (b + bi * R));
#pragma unroll 8
        for (int r = 0; r < R; ++r) {
            if (r < cnt) {
                const float2 v = ring[((size_t)slot * R + r) * 32 + lane];
                acc.x += v.x; acc.y += v.y;
            }
        }
        __syncwarp();
    }
    out[warp * 32 + lane] = acc;
}

static void* g_flush;
static size_t g_flush_bytes = 1ull << 30;

template <class F>
float timeit(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemsetAsync(g_flush, rep, g_flush_bytes);
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(err)); exit(1); }
    return best;
}

int main(int argc, char** argv) {
    const int levels = argc > 1 ? atoi(argv[1]) : 22;
    const long long n = argc > 2 ? atoll(argv[2]) : 65241671;
    const long long rows = 1LL << levels;
    int* di; float2* B; float2* out;
    cudaMalloc(&di, n * 4);
    cudaMalloc(&B, rows * 256);
    cudaMalloc(&out, 148LL * 64 * 32 * 8 * 4);
    cudaMemset(B, 0, rows * 256);
    cudaMalloc(&g_flush, g_flush_bytes);
    gen_idx<<<148 * 8, 256>>>(di, n, levels, 1803);
    cudaDeviceSynchronize();
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double gb = n * 256.0 / 1e9;
    auto report = [&](const char* name, float ms) {
        printf("%-44s %8.3f ms  %6.2f Gathers/us  %6.2f TB/s of rows\n", name, ms, n / ms / 1e6, gb / ms);
        fflush(stdout);
    };
    int hot = argc > 3 ? atoi(argv[3]) : (levels >= 26 ? 6 : 7);
    char name[128];
    // LDG variants: warps per SM via CTAs per SM (256-thread CTAs)
    for (int cps : {4, 6, 8}) {
        const int grid = sms * cps;
        snprintf(name, sizeof name, "ldg U=8  warps/SM=%d", cps * 8);
        report(name, timeit([&] { k_ldg<8, 0><<<grid, 256>>>(di, n, B, out, hot); }));
        snprintf(name, sizeof name, "ldg U=16 warps/SM=%d", cps * 8);
        report(name, timeit([&] { k_ldg<16, 0><<<grid, 256>>>(di, n, B, out, hot); }));
    }
    for (int cps : {4, 8}) {
        const int grid = sms * cps;
        snprintf(name, sizeof name, "ldg U=8 evict_first warps/SM=%d", cps * 8);
        report(name, timeit([&] { k_ldg<8, 1><<<grid, 256>>>(di, n, B, out, hot); }));
        for (int h = hot - 1; h <= hot + 1; ++h) {
            snprintf(name, sizeof name, "ldg U=8 hot(pc<=%d) last/first warps/SM=%d", h, cps * 8);
            report(name, timeit([&] { k_ldg<8, 2><<<grid, 256>>>(di, n, B, out, h); }));
        }
    }
    // LDGSTS rings
    {
        auto run = [&](auto kern, int D, int cps) {
            const size_t smem = (size_t)8 * D * 8 * 256;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            const int grid = sms * cps;
            snprintf(name, sizeof name, "ldgsts D=%d (%d rows/warp) warps/SM=%d", D, 8 * (D - 1), cps * 8);
            report(name, timeit([&] { kern<<<grid, 256, smem>>>(di, n, B, out, hot); }));
        };
        run(k_ldgsts<3, 0>, 3, 4);
        run(k_ldgsts<4, 0>, 4, 3);
        run(k_ldgsts<4, 0>, 4, 4);
        run(k_ldgsts<6, 0>, 6, 2);
        run(k_ldgsts<6, 0>, 6, 3);
    }
    // TMA bulk rings
    {
        auto run = [&](auto kern, int D, int R, int cps, const char* tag) {
            const size_t smem = (size_t)8 * D * R * 256 + 8 * D * 8;
            if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
                printf("skip bulk D=%d R=%d\n", D, R); cudaGetLastError(); return;
            }
            const int grid = sms * cps;
            snprintf(name, sizeof name, "bulk%s D=%d R=%d (%d rows/warp) warps/SM=%d", tag, D, R, R * (D - 1), cps * 8);
            report(name, timeit([&] { kern<<<grid, 256, smem>>>(di, n, B, out, hot); }));
        };
        run(k_bulk<2, 16, 0>, 2, 16, 2, "");
        run(k_bulk<3, 16, 0>, 3, 16, 2, "");
        run(k_bulk<2, 32, 0>, 2, 32, 1, "");
        run(k_bulk<3, 8, 0>, 3, 8, 4, "");
        run(k_bulk<4, 8, 0>, 4, 8, 3, "");
        run(k_bulk<3, 16, 2>, 3, 16, 2, " hot");
        run(k_bulk<4, 8, 2>, 4, 8, 3, " hot");
    }
    // persisting L2 set-aside + hot policy
    {
        cudaDeviceProp pr; cudaGetDeviceProperties(&pr, 0);
        printf("L2 %d bytes, persisting max %d bytes\n", pr.l2CacheSize, pr.persistingL2CacheMaxSize);
        for (double frac : {0.5, 0.75}) {
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)(pr.persistingL2CacheMaxSize * frac));
            for (int h = hot - 1; h <= hot + 1; ++h) {
                snprintf(name, sizeof name, "ldg U=8 hot(pc<=%d) persist=%.2f warps/SM=32", h, frac);
                report(name, timeit([&] { k_ldg<8, 2><<<sms * 4, 256>>>(di, n, B, out, h); }));
            }
            cudaCtxResetPersistingL2Cache();
        }
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
    }
    return 0;
}
