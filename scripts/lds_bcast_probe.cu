// probe (tuning only): LDS.128 cost when the 4 groups of 8 lanes of a warp read the SAME 128-byte block
// (shared-memory broadcast across quarter-warps) vs 2 or 4 different blocks.  Prints ns per warp-LDS per SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int mode, int iters, float* out) {
    __shared__ __align__(16) float buf[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = i * 0.5f;
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 3, gl = lane & 7;
    const int w = threadIdx.x >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    const unsigned base = (unsigned)__cvta_generic_to_shared(buf);
    // mode 0: 4 distinct rows; 1: all groups the same row; 2: two distinct rows (groups 0,1 / 2,3)
    const int gsel = mode == 0 ? g : (mode == 1 ? 0 : (g >> 1));
    for (int it = 0; it < iters; ++it) {
        const int row = (gsel * 5 + it * 3 + w * 7) & 31;
        const unsigned a = base + row * 256 + gl * 16;
        float4 x;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(a));
        acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    if (acc.x == 12345.f) out[threadIdx.x] = acc.y + acc.z + acc.w;
}
int main() {
    float* out; cudaMalloc(&out, 4096);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 1 << 16, threads = 512, ctas = sms * 4;
    for (int mode = 0; mode < 3; ++mode) {
        probe<<<ctas, threads>>>(mode, iters, out);
        cudaEventRecord(e0);
        probe<<<ctas, threads>>>(mode, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double lds_per_sm = (double)iters * (threads / 32) * (ctas / sms);
        printf("mode %d (%s): %.3f ms, %.3f ns per warp LDS.128 per SM (%.2f clk at 1.965 GHz)\n", mode,
               mode == 0 ? "4 distinct 128B blocks" : mode == 1 ? "1 block, broadcast" : "2 blocks",
               ms, ms * 1e6 / lds_per_sm, ms * 1e6 / lds_per_sm * 1.965);
    }
    return 0;
}
