// LDS.128 bank-pattern probe (tuning, not product code): 8 row groups of 4 lanes per warp, each group
// reading a 64-byte column block of a different 256-byte B row (row pitch 256 B), block index chosen
// by a per-group rotation rule.  Prints cycles per LDS.128 per SM (4.0 = conflict-free).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(int rule, int iters, float* out) {
    __shared__ __align__(16) float buf[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = i * 0.5f;
    __syncthreads();
    const int lane = threadIdx.x & 31, g = lane >> 2, gl = lane & 3;
    float4 acc = make_float4(0, 0, 0, 0);
    const unsigned base = (unsigned)__cvta_generic_to_shared(buf);
    for (int it = 0; it < iters; ++it) {
        const int v = it & 3;
        int blk;
        if (rule == 0) blk = v;                       // no rotation
        else if (rule == 1) blk = (v + g) & 3;        // rotate by group
        else if (rule == 2) blk = (v + (g >> 1)) & 3; // rotate by group pair
        else blk = v ^ (g & 3);                       // xor
        const int row = (g * 5 + it * 3) & 31;        // 8 different rows per instruction
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
    const char* names[] = {"none", "rot_g", "rot_gpair", "xor"};
    for (int r = 0; r < 4; ++r) {
        probe<<<148 * 4, 512>>>(r, 4096, out);
        cudaEventRecord(e0);
        probe<<<148 * 4, 512>>>(r, 4096, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double instr = 148.0 * 4 * 16 * 4096;
        printf("rule %-10s: %.2f cycles/LDS.128 per SM @1.9GHz\n", names[r], ms * 1e-3 * 1.9e9 / (instr / 148));
    }
    return 0;
}
