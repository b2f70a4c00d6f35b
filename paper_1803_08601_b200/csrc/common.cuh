// common.cuh -- semiring arithmetic, vector gathers and cache-hinted memory ops shared by the
// sm_100a SpMM kernels (row split, merge path, carry fix-up).  Product code; shares nothing with
// oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace spmm {

constexpr unsigned FULL = 0xffffffffu;
constexpr int WARPS_PER_CTA = 8;          // 256-thread CTAs everywhere
constexpr int THREADS = 32 * WARPS_PER_CTA;

enum : int { SR_PLUS_TIMES = 0, SR_MIN_PLUS = 1 };

// ---------------------------------------------------------------------------------------------
// Semirings (GrB_mxm framing).  mac(acc, a, b) = acc (+) (a (x) b); add = (+).
// int32 arithmetic is done in uint32 so overflow wraps (SURVEY.md §8(c) ambiguity 19).
// ---------------------------------------------------------------------------------------------
template <typename T, int SR> struct Ring;

template <> struct Ring<float, SR_PLUS_TIMES> {
    __device__ __forceinline__ static float id() { return 0.0f; }
    __device__ __forceinline__ static float mac(float acc, float a, float b) { return __fmaf_rn(a, b, acc); }
    __device__ __forceinline__ static float add(float x, float y) { return __fadd_rn(x, y); }
};
template <> struct Ring<int, SR_PLUS_TIMES> {
    __device__ __forceinline__ static int id() { return 0; }
    __device__ __forceinline__ static int mac(int acc, int a, int b) {
        return (int)((unsigned)acc + (unsigned)a * (unsigned)b);
    }
    __device__ __forceinline__ static int add(int x, int y) { return (int)((unsigned)x + (unsigned)y); }
};
template <> struct Ring<float, SR_MIN_PLUS> {
    __device__ __forceinline__ static float id() { return __int_as_float(0x7f800000); }
    __device__ __forceinline__ static float mac(float acc, float a, float b) { return fminf(acc, __fadd_rn(a, b)); }
    __device__ __forceinline__ static float add(float x, float y) { return fminf(x, y); }
};
template <> struct Ring<int, SR_MIN_PLUS> {
    __device__ __forceinline__ static int id() { return 0x7fffffff; }
    __device__ __forceinline__ static int mac(int acc, int a, int b) {
        return min(acc, (int)((unsigned)a + (unsigned)b));
    }
    __device__ __forceinline__ static int add(int x, int y) { return min(x, y); }
};

// ---------------------------------------------------------------------------------------------
// bit casts
// ---------------------------------------------------------------------------------------------
template <typename T> __device__ __forceinline__ T from_bits(unsigned u);
template <> __device__ __forceinline__ float from_bits<float>(unsigned u) { return __uint_as_float(u); }
template <> __device__ __forceinline__ int from_bits<int>(unsigned u) { return (int)u; }
template <typename T> __device__ __forceinline__ unsigned to_bits(T v);
template <> __device__ __forceinline__ unsigned to_bits<float>(float v) { return __float_as_uint(v); }
template <> __device__ __forceinline__ unsigned to_bits<int>(int v) { return (unsigned)v; }

// ---------------------------------------------------------------------------------------------
// Memory ops.
//   A stream (col_indices, values, row_offsets): read once -> no L1 allocation.
//   B gathers: read-only path (L1 + L2 cached); B rows are the reused operand.
//   C rows: written once -> streaming store (evict-first).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ int ld_stream(const int* p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
// gather VEC consecutive elements of a B row (VEC in {1,2,4}); p must be VEC*4-byte aligned
template <int VEC> __device__ __forceinline__ void ldg_vec(unsigned (&o)[VEC], const void* p);
template <> __device__ __forceinline__ void ldg_vec<1>(unsigned (&o)[1], const void* p) {
    o[0] = __ldg(reinterpret_cast<const unsigned*>(p));
}
template <> __device__ __forceinline__ void ldg_vec<2>(unsigned (&o)[2], const void* p) {
    uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    o[0] = v.x; o[1] = v.y;
}
template <> __device__ __forceinline__ void ldg_vec<4>(unsigned (&o)[4], const void* p) {
    uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}

template <int VEC> __device__ __forceinline__ void st_vec(void* p, const unsigned (&o)[VEC]);
template <> __device__ __forceinline__ void st_vec<1>(void* p, const unsigned (&o)[1]) {
    __stcs(reinterpret_cast<unsigned*>(p), o[0]);
}
template <> __device__ __forceinline__ void st_vec<2>(void* p, const unsigned (&o)[2]) {
    __stcs(reinterpret_cast<uint2*>(p), make_uint2(o[0], o[1]));
}
template <> __device__ __forceinline__ void st_vec<4>(void* p, const unsigned (&o)[4]) {
    __stcs(reinterpret_cast<uint4*>(p), make_uint4(o[0], o[1], o[2], o[3]));
}

// ---------------------------------------------------------------------------------------------
// Epilogue of every finished row of C (spmm_exec_opts): C = C (+) result when accumulating (the
// diagonal / off-diagonal split of the iterative distributed SpMM), and the
// same row also stored into up to 7 peer copies of C (the all-gather of C fused into the SpMM, NEXT-1:
// peer pointers are P2P / IPC mappings of other GPUs' C, so the store travels over NVLink).
// ---------------------------------------------------------------------------------------------
constexpr int EPI_MAX_PEERS = 7;
struct EpiParams {
    int accumulate;
    int npeers;
    long long peer_row0;  // row r of this C is row r + peer_row0 of each peer C
    long long peer_ldc;
    void* peer[EPI_MAX_PEERS];
};

template <int VEC> __device__ __forceinline__ void ld_vec(unsigned (&o)[VEC], const void* p);
template <> __device__ __forceinline__ void ld_vec<1>(unsigned (&o)[1], const void* p) {
    o[0] = *reinterpret_cast<const volatile unsigned*>(p);
}
template <> __device__ __forceinline__ void ld_vec<2>(unsigned (&o)[2], const void* p) {
    const uint2 v = *reinterpret_cast<const uint2*>(p);
    o[0] = v.x; o[1] = v.y;
}
template <> __device__ __forceinline__ void ld_vec<4>(unsigned (&o)[4], const void* p) {
    const uint4 v = *reinterpret_cast<const uint4*>(p);
    o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
}

// the epilogue's accumulate / peer path
template <typename T, int SR, int VEC>
__device__ __forceinline__ void epi_store_ext(const EpiParams& E, T* p, long long row, int col, unsigned (&o)[VEC]) {
    if (E.accumulate) {
        unsigned old[VEC];
        ld_vec<VEC>(old, p);
#pragma unroll
        for (int x = 0; x < VEC; ++x) o[x] = to_bits<T>(Ring<T, SR>::add(from_bits<T>(old[x]), from_bits<T>(o[x])));
    }
    st_vec<VEC>(p, o);
    for (int i = 0; i < E.npeers; ++i)
        st_vec<VEC>(static_cast<T*>(E.peer[i]) + (row + E.peer_row0) * E.peer_ldc + col, o);
}

// store VEC values (bit patterns in o) of row `row`, columns [col, col + VEC), through the epilogue
template <typename T, int SR, int VEC>
__device__ __forceinline__ void epi_store(const EpiParams& E, T* C, long long ldc, long long row, int col,
                                          unsigned (&o)[VEC]) {
    T* p = C + row * ldc + col;
    if (E.accumulate | E.npeers) epi_store_ext<T, SR, VEC>(E, p, row, col, o);
    else st_vec<VEC>(p, o);
}

}  // namespace spmm
