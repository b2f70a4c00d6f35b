// gather_probe.cu -- microbenchmark (not product code): throughput ceiling of the B-row gather pattern
// on this GPU.  Each warp walks a slice of an index array and gathers 256-byte rows of a 1 GiB matrix
// (lanes over the 64 floats of a row, U rows in flight per warp), summing into registers (one store
// per warp at the end), so the only traffic is the gathers themselves.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe gather_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>

template <int U>
__global__ void gather_sum(const int* __restrict__ idx, long long n, const float2* __restrict__ B, float2* out) {
    const int lane = threadIdx.x & 31;
    const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const long long per = (n + nw - 1) / nw;
    const long long b = warp * per, e = min(n, b + per);
    float2 acc = make_float2(0.f, 0.f);
    for (long long p = b; p < e; p += U) {
        float2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const long long q = p + u;
            v[u] = q < e ? __ldg(B + (long long)__ldg(idx + q) * 32 + lane) : make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; }
    }
    out[warp * 32 + lane] = acc;
}

int main(int argc, char** argv) {
    const long long rows = 1 << 22;  // 4M rows x 256 B = 1 GiB
    const long long n = argc > 2 ? atoll(argv[2]) : 65241671;
    const char* mode = argc > 1 ? argv[1] : "uniform";
    std::vector<int> h(n);
    std::mt19937_64 rng(1);
    if (mode[0] == 'u') {
        for (auto& x : h) x = (int)(rng() % rows);
    } else if (mode[0] == 's') {  // sequential rows (each row gathered once, streaming)
        for (long long i = 0; i < n; ++i) h[i] = (int)(i % rows);
    } else {  // power-law: R-MAT-like column popularity (a+c = 0.76 per level)
        for (auto& x : h) {
            int c = 0;
            for (int l = 0; l < 22; ++l) {
                const double r = (rng() >> 11) * (1.0 / 9007199254740992.0);
                c = (c << 1) | (r >= 0.76 ? 1 : 0);
            }
            x = c;
        }
    }
    int* di; float2* B; float2* out;
    cudaMalloc(&di, n * 4);
    cudaMalloc(&B, rows * 256);
    cudaMalloc(&out, 1 << 26);
    cudaMemcpy(di, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaMemset(B, 0, rows * 256);
    void* flush; cudaMalloc(&flush, 512 << 20);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int blocks[] = {148 * 4, 148 * 8, 148 * 16};
    for (int bi = 0; bi < 3; ++bi) {
        for (int u : {8, 16, 32}) {
            float best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                cudaMemset(flush, rep, 512 << 20);
                cudaEventRecord(e0);
                if (u == 8) gather_sum<8><<<blocks[bi], 256>>>(di, n, B, out);
                if (u == 16) gather_sum<16><<<blocks[bi], 256>>>(di, n, B, out);
                if (u == 32) gather_sum<32><<<blocks[bi], 256>>>(di, n, B, out);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("%s blocks=%d U=%d: %.3f ms  gathers %.1f G/s  %.2f TB/s of rows\n", mode, blocks[bi], u, best,
                   n / best / 1e6, n * 256.0 / best / 1e9);
        }
    }
    return 0;
}
