// probe (tuning only): does a SHFL occupy the same shared-memory / LSU data pipe as an LDS?  Warps
// issue 2 LDS.128 per iteration (B-row-like traffic, 4 cycles each) plus either nothing, 2 LDS.32 or
// 2 SHFL.IDX; prints ns per iteration per SM.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int mode, int iters, float* out) {
    __shared__ __align__(16) float buf[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = i * 0.5f;
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 3, gl = lane & 7;
    const int w = threadIdx.x >> 5;
    float4 acc = make_float4(0, 0, 0, 0);
    float sacc = 0.f;
    unsigned sidx = lane;
    const unsigned base = (unsigned)__cvta_generic_to_shared(buf);
    for (int it = 0; it < iters; ++it) {
        const int row = (g * 5 + it * 3 + w * 7) & 31;
        const unsigned a = base + row * 256 + gl * 16;
        float4 x, y;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w) : "r"(a));
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(y.x), "=f"(y.y), "=f"(y.z), "=f"(y.w) : "r"(a + 128));
        acc.x += x.x * y.x; acc.y += x.y * y.y; acc.z += x.z * y.z; acc.w += x.w * y.w;
        if (mode == 1) {
            float u, v;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(u) : "r"(base + 4 * ((sidx + it) & 1023)));
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(base + 4 * ((sidx + 2 * it) & 1023)));
            sacc += u * v;
        } else if (mode == 2) {
            const float u = __shfl_sync(0xffffffffu, acc.x, (lane & 24) | (it & 7));
            const float v = __shfl_sync(0xffffffffu, acc.y, (lane & 24) | ((it + 3) & 7));
            sacc += u * v;
        }
    }
    if (acc.x + sacc == 12345.f) out[threadIdx.x] = acc.y + acc.z + acc.w;
}
int main() {
    float* out; cudaMalloc(&out, 4096);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 1 << 15, threads = 512, ctas = sms * 4;
    const char* names[3] = {"2 LDS.128", "2 LDS.128 + 2 LDS.32", "2 LDS.128 + 2 SHFL.IDX"};
    for (int mode = 0; mode < 3; ++mode) {
        probe<<<ctas, threads>>>(mode, iters, out);
        cudaEventRecord(e0);
        probe<<<ctas, threads>>>(mode, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double per_sm = (double)iters * (threads / 32) * (ctas / sms);
        printf("mode %d (%s): %.3f ms, %.3f clk per warp-iteration per SM at 1.965 GHz\n", mode, names[mode], ms,
               ms * 1e6 / per_sm * 1.965);
    }
    return 0;
}
