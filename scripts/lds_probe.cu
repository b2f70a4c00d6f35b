// LDS.128 wavefront probe: do the 4 row groups of a warp (8 lanes x 16 B each) that read the SAME
// 128-byte B row cost one shared-memory wavefront (broadcast) or four (quarter-warp phases)?
// mode 0: group g reads chunk g (512 distinct bytes per instruction)
// mode 1: all groups read chunk 0 (128 distinct bytes per instruction)
// mode 2: all 32 lanes read the same 16 bytes
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int mode, int iters, float* out) {
    __shared__ __align__(16) float buf[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = i * 0.5f;
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 3, gl = lane & 7;
    int base = (mode == 0) ? (g * 32 + gl * 4) : (mode == 1 ? gl * 4 : 0);
    base += (threadIdx.x >> 5) * 128;  // warps read different rows
    float4 acc = make_float4(0, 0, 0, 0);
    unsigned a = (unsigned)__cvta_generic_to_shared(buf) + base * 4;
    for (int it = 0; it < iters; ++it) {
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a + ((it & 7) << 11)));
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    if (acc.x == 12345.f) out[threadIdx.x] = acc.y + acc.z + acc.w;
}
int main() {
    float* out; cudaMalloc(&out, 4096);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
        probe<<<148 * 4, 512>>>(mode, 4096, out);
        cudaEventRecord(e0);
        probe<<<148 * 4, 512>>>(mode, 4096, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double instr = 148.0 * 4 * 16 * 4096;  // warp-level LDS.128
        printf("mode %d: %.3f ms, %.2f cycles/LDS.128 per SM @1.9GHz\n", mode, ms, ms * 1e-3 * 1.9e9 / (instr / 148));
    }
    return 0;
}
