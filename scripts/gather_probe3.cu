// gather_probe3.cu -- microbenchmark (not product code): the HBM ceiling of the merge kernel's access
// pattern.  Each warp gathers 256-byte rows of B (n = 64 fp32, lanes over columns, LDG.64) at the
// indices of a stream and sums them.  Index streams:
//   seq      i                      (streaming read: the copy-bandwidth reference)
//   uniform  hash(i) mod 2^L        (no reuse beyond chance: B = 2^L x 256 B; L = 26 -> 17.2 GB, so this
//                                    is the random 256-byte-row read bandwidth of HBM)
//   rmat     every one of L bits is 1 with probability 0.24 (Graph500 b + d: R-MAT column marginal)
// U gathers in flight per warp (issued back to back, then summed), warps/SM from CTAs/SM; median of 5
// reps, L2 flushed (1 GB memset) before each.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gp3 scripts/gather_probe3.cu
// Run:   /tmp/gp3 <L> <n_indices>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

__global__ void gen_idx(int* idx, long long n, int levels, int mode, uint32_t seed) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        uint32_t c = 0;
        if (mode == 0) {
            c = (uint32_t)(i & ((1LL << levels) - 1));
        } else if (mode == 1) {
            c = hash32((uint32_t)i * 0x9E3779B1u ^ seed) & (uint32_t)((1LL << levels) - 1);
        } else {
            for (int l = 0; l < levels; ++l) {
                const uint32_t h = hash32((uint32_t)i * 0x9E3779B1u ^ hash32((uint32_t)(i >> 32) + l * 0x85ebca6bu + seed));
                c = (c << 1) | (h < 1030792151u ? 1u : 0u);  // 0.24 * 2^32
            }
        }
        idx[i] = (int)c;
    }
}

__device__ __forceinline__ uint64_t mkpol(int kind) {
    uint64_t p = 0;
    if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    else if (kind == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    else if (kind == 3) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
    else asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float2 ldg_pol(const float2* a, uint64_t pol) {
    float2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(v.x), "=f"(v.y) : "l"(a), "l"(pol));
    return v;
}

// POLICY: 0 none; otherwise rows with popcount(idx) <= hot get policy HOTK, the others COLDK
// (1 evict_last, 2 evict_first, 3 evict_normal)
template <int U, int HOTK, int COLDK>
__global__ void __launch_bounds__(256) k_ldg(const int* __restrict__ idx, long long n, const float2* __restrict__ B,
                                               float2* out, int hot) {
    const uint64_t ph = mkpol(HOTK), pc = mkpol(COLDK);
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long per = (n + nw - 1) / nw;
    const long long b = warp * per, e = min(n, b + per);
    float2 acc = make_float2(0.f, 0.f);
    for (long long p = b; p < e; p += 32) {
        const int myidx = (p + lane < e) ? __ldg(idx + p + lane) : 0;
        const int cnt = (int)min(32LL, e - p);
        for (int u0 = 0; u0 < cnt; u0 += U) {
            float2 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int c = __shfl_sync(0xffffffffu, myidx, (u0 + u) & 31);
                if (u0 + u < cnt) {
                    const float2* a = B + (long long)c * 32 + lane;
                    if (HOTK == 0) v[u] = __ldg(a);
                    else v[u] = ldg_pol(a, __popc(c) <= hot ? ph : pc);
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

static void* g_flush;
static const size_t g_flush_bytes = 1ull << 30;

template <class F>
float timeit(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    std::vector<float> t;
    for (int rep = 0; rep < 6; ++rep) {
        cudaMemsetAsync(g_flush, rep, g_flush_bytes);
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (rep) t.push_back(ms);
    }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(err)); exit(1); }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

int main(int argc, char** argv) {
    const int levels = argc > 1 ? atoi(argv[1]) : 26;
    const long long n = argc > 2 ? atoll(argv[2]) : (1LL << 28);
    const long long rows = 1LL << levels;
    int* di; float2* B; float2* out;
    cudaMalloc(&di, n * 4);
    if (cudaMalloc(&B, rows * 256) != cudaSuccess) { printf("B alloc failed\n"); return 1; }
    cudaMalloc(&out, 148LL * 64 * 32 * 8 * 4);
    cudaMemset(B, 0, rows * 256);
    cudaMalloc(&g_flush, g_flush_bytes);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double gb = n * 256.0 / 1e9;
    printf("L = %d (B = %.2f GB), %lld gathers of 256 B (%.2f GB requested)\n", levels, rows * 256.0 / 1e9, n, gb);
    const char* names[3] = {"seq", "uniform", "rmat"};
    for (int mode = 0; mode < 3 && argc <= 3; ++mode) {  // argv[3]: policy experiment only
        gen_idx<<<sms * 8, 256>>>(di, n, levels, mode, 1803);
        cudaDeviceSynchronize();
        for (int cps : {2, 3, 4, 5, 6, 8}) {
            const int grid = sms * cps;
            const float t8 = timeit([&] { k_ldg<8, 0, 0><<<grid, 256>>>(di, n, B, out, 0); });
            const float t16 = timeit([&] { k_ldg<16, 0, 0><<<grid, 256>>>(di, n, B, out, 0); });
            printf("%-8s warps/SM=%2d  U=8 %8.3f ms %6.2f TB/s   U=16 %8.3f ms %6.2f TB/s\n", names[mode], cps * 8,
                   t8, gb / t8, t16, gb / t16);
            fflush(stdout);
        }
    }
    // L2 priority by popularity (R-MAT marginal: popcount(idx) small = hot), 48 warps/SM, U = 8
    gen_idx<<<sms * 8, 256>>>(di, n, levels, 2, 1803);
    cudaDeviceSynchronize();
    const int grid = sms * 6;
    for (int h = levels / 5; h <= levels / 5 + 3; ++h) {
        long long hot_rows = 0, binom = 1;
        for (int j = 0; j <= h; ++j) { hot_rows += binom; binom = binom * (levels - j) / (j + 1); }
        const float a = timeit([&] { k_ldg<8, 1, 2><<<grid, 256>>>(di, n, B, out, h); });
        const float b = timeit([&] { k_ldg<8, 3, 2><<<grid, 256>>>(di, n, B, out, h); });
        const float c = timeit([&] { k_ldg<8, 1, 3><<<grid, 256>>>(di, n, B, out, h); });
        printf("rmat hot = popcount <= %d (%lld rows, %.1f MB): last/first %8.3f ms  normal/first %8.3f ms  "
               "last/normal %8.3f ms\n", h, hot_rows, hot_rows * 256.0 / 1e6, a, b, c);
        fflush(stdout);
    }
    return 0;
}
