// ptx.cuh -- thin inline-PTX wrappers for the sm_100a features the tile engine uses:
// mbarrier (transaction-count barriers), 1-D TMA bulk copies global->shared, proxy fences,
// named barriers and packed fp32x2 FMA.
#pragma once
#include <stdint.h>

namespace spmm {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// arrive (count 1) and add `tx` expected transaction bytes
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// TMA 1-D bulk copy: `bytes` (multiple of 16) from 16B-aligned global `src` to 16B-aligned smem `dst`,
// completion signalled as transaction bytes on `bar`.  L2 evict-first hint: the A stream is read once.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// TMA bulk prefetch of a contiguous global range into L2 (no shared-memory destination)
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}

__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

// predicated shared-memory load (no branch); 0 when !pred
__device__ __forceinline__ unsigned lds_pred(uint32_t saddr, bool pred) {
    unsigned v;
    asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; mov.b32 %0, 0; @q ld.shared.b32 %0, [%1];}"
                 : "=r"(v) : "r"(saddr), "r"((int)pred));
    return v;
}
__device__ __forceinline__ unsigned lds_u32(uint32_t saddr) {
    unsigned v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(saddr));
    return v;
}
__device__ __forceinline__ uint2 lds_u64(uint32_t saddr) {
    uint2 v;
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(saddr));
    return v;
}
__device__ __forceinline__ uint4 lds_u128(uint32_t saddr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(saddr));
    return v;
}
// predicated streaming global load
__device__ __forceinline__ unsigned ldg_stream_pred(const void* p, bool pred) {
    unsigned v;
    asm volatile("{.reg .pred q; setp.ne.b32 q, %2, 0; mov.b32 %0, 0; @q ld.global.nc.L1::no_allocate.b32 %0, [%1];}"
                 : "=r"(v) : "l"(p), "r"((int)pred));
    return v;
}
// opaque 64-bit copy: keeps a per-lane base address in one register pair so that address
// arithmetic folds into a single IMAD.WIDE.U32
__device__ __forceinline__ const char* opaque_ptr(const char* p) {
    const char* q;
    asm("mov.b64 %0, %1;" : "=l"(q) : "l"(p));
    return q;
}

template <int VEC> __device__ __forceinline__ void lds_vec(unsigned (&o)[VEC], uint32_t saddr);
template <> __device__ __forceinline__ void lds_vec<1>(unsigned (&o)[1], uint32_t a) {
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(o[0]) : "r"(a));
}
template <> __device__ __forceinline__ void lds_vec<2>(unsigned (&o)[2], uint32_t a) {
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(o[0]), "=r"(o[1]) : "r"(a));
}
template <> __device__ __forceinline__ void lds_vec<4>(unsigned (&o)[4], uint32_t a) {
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]) : "r"(a));
}

// d = a * b + c on two packed fp32 lanes (sm_100 FFMA2)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    uint64_t d;
    uint64_t ua = *reinterpret_cast<uint64_t*>(&a);
    uint64_t ub = *reinterpret_cast<uint64_t*>(&b);
    uint64_t uc = *reinterpret_cast<uint64_t*>(&c);
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(ua), "l"(ub), "l"(uc));
    return *reinterpret_cast<float2*>(&d);
}

}  // namespace spmm
