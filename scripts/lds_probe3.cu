// brute force (tuning only): per-group block offsets o_g (blk = (v + o_g) & 3) for 8 groups of 4 lanes
// reading 64-byte blocks of different 256-byte rows; find assignments that make LDS.128 conflict-free.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(unsigned code, int iters, float* out) {
    __shared__ __align__(16) float buf[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = i * 0.5f;
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 2, gl = lane & 3;
    const int og = (code >> (2 * g)) & 3;
    float4 acc = make_float4(0, 0, 0, 0);
    const unsigned base = (unsigned)__cvta_generic_to_shared(buf);
    for (int it = 0; it < iters; ++it) {
        const int blk = ((it & 3) + og) & 3;
        const int row = (g * 5 + it * 3) & 31;
        const unsigned a = base + row * 256 + blk * 64 + gl * 16;
        float4 x;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(a));
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    if (acc.x == 12345.f) out[threadIdx.x] = acc.y + acc.z + acc.w;
}
int main() {
    float* out; cudaMalloc(&out, 4096);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e9; unsigned bc = 0;
    int hist[40] = {0};
    for (unsigned code = 0; code < (1u << 14); ++code) {
        const unsigned c = code << 2;  // o_0 = 0
        cudaEventRecord(e0);
        probe<<<148 * 2, 512>>>(c, 512, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double cyc = ms * 1e-3 * 1.9e9 / (2.0 * 16 * 512);
        int b = (int)(cyc * 4); if (b > 39) b = 39; hist[b]++;
        if (cyc < best) { best = cyc; bc = c; }
    }
    printf("best %.2f cycles/LDS.128, offsets:", best);
    for (int g = 0; g < 8; ++g) printf(" %u", (bc >> (2 * g)) & 3);
    printf("\nhistogram (quarter cycles):");
    for (int i = 0; i < 40; ++i) if (hist[i]) printf(" %.2f:%d", i / 4.0, hist[i]);
    printf("\n");
    return 0;
}
