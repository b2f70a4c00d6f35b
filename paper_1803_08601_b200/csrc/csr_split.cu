// csr_split.cu -- spmm_csr_split_columns (include/spmm.h): split every row of a CSR matrix into the
// entries whose column lies in [c0, c1) (column rebased by -c0) and all other entries (global column),
// keeping each row's storage order.  Set-up for the iterative distributed SpMM (SURVEY.md §8(f) NEXT-3,
// PAPER.md:13): a rank's row block A_r = [A_rr | A_r,other] is split once, so each iteration computes
// the diagonal block A_rr X_r while the other ranks' blocks of X are still being gathered, then
// accumulates A_r,other X (spmm_csr_execute_ex, accumulate = 1).  Not on the per-call SpMM path.
#include <cuda_runtime.h>

#include <algorithm>

#include <cub/cub.cuh>

#include "../../include/spmm.h"

namespace {

constexpr int kThreads = 256;

// warp per row: in-range / out-of-range entry counts
__global__ void k_split_count(const int* __restrict__ ro, const int* __restrict__ col, long long m, int c0, int c1,
                              int* __restrict__ cnt_in, int* __restrict__ cnt_out) {
    const int lane = threadIdx.x & 31;
    const long long nw = (long long)gridDim.x * (blockDim.x / 32);
    for (long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < m; r += nw) {
        const int s = ro[r], e = ro[r + 1];
        int c = 0;
        for (int p = s + lane; p < e; p += 32) {
            const int x = col[p];
            c += (x >= c0 && x < c1) ? 1 : 0;
        }
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) {
            cnt_in[r] = c;
            cnt_out[r] = (e - s) - c;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        cnt_in[m] = 0;
        cnt_out[m] = 0;
    }
}

// warp per row: stable compaction of the row's entries into the two outputs
__global__ void k_split_scatter(const int* __restrict__ ro, const int* __restrict__ col,
                                const unsigned* __restrict__ val, long long m, int c0, int c1,
                                const int* __restrict__ ro_in, int* __restrict__ col_in, unsigned* __restrict__ val_in,
                                const int* __restrict__ ro_out, int* __restrict__ col_out,
                                unsigned* __restrict__ val_out) {
    const int lane = threadIdx.x & 31;
    const unsigned below = (1u << lane) - 1u;
    const long long nw = (long long)gridDim.x * (blockDim.x / 32);
    for (long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < m; r += nw) {
        const int s = ro[r], e = ro[r + 1];
        int pin = ro_in[r], pout = ro_out[r];
        for (int p0 = s; p0 < e; p0 += 32) {
            const int p = p0 + lane;
            const bool ok = p < e;
            const int x = ok ? col[p] : 0;
            const unsigned v = ok ? val[p] : 0u;
            const bool in = ok && x >= c0 && x < c1;
            const unsigned bin = __ballot_sync(0xffffffffu, in);
            const unsigned bout = __ballot_sync(0xffffffffu, ok && !in);
            if (in) {
                const int q = pin + __popc(bin & below);
                col_in[q] = x - c0;
                val_in[q] = v;
            } else if (ok) {
                const int q = pout + __popc(bout & below);
                col_out[q] = x;
                val_out[q] = v;
            }
            pin += __popc(bin);
            pout += __popc(bout);
        }
    }
}

}  // namespace

extern "C" spmm_status spmm_csr_split_columns(const int32_t* row_offsets, const int32_t* col_indices,
                                              const void* values, int64_t m, int64_t nnz, int32_t c0, int32_t c1,
                                              spmm_dtype dtype, int32_t* ro_in, int32_t* col_in, void* val_in,
                                              int32_t* ro_out, int32_t* col_out, void* val_out, int64_t* nnz_in,
                                              void* stream) {
    if (!nnz_in || !ro_in || !ro_out) return SPMM_ERR_NULL_POINTER;
    *nnz_in = 0;
    if (m < 0 || nnz < 0 || m >= 0x7fffffffLL || nnz >= 0x7fffffffLL || c1 < c0) return SPMM_ERR_INVALID_ARG;
    if (dtype != SPMM_F32 && dtype != SPMM_I32) return SPMM_ERR_INVALID_ARG;
    if (m > 0 && !row_offsets) return SPMM_ERR_NULL_POINTER;
    if (nnz > 0 && (!col_indices || !values || !col_in || !val_in || !col_out || !val_out)) return SPMM_ERR_NULL_POINTER;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (m == 0) {
        if (cudaMemsetAsync(ro_in, 0, sizeof(int32_t), st) != cudaSuccess) return SPMM_ERR_CUDA;
        if (cudaMemsetAsync(ro_out, 0, sizeof(int32_t), st) != cudaSuccess) return SPMM_ERR_CUDA;
        return SPMM_OK;
    }
    // counts go to the output offset arrays, then an in-place exclusive scan over m + 1 entries
    const int grid = (int)std::min<long long>((m * 32 + kThreads - 1) / kThreads, 148LL * 16);
    k_split_count<<<grid, kThreads, 0, st>>>(row_offsets, col_indices, m, c0, c1, ro_in, ro_out);
    if (cudaGetLastError() != cudaSuccess) return SPMM_ERR_CUDA;
    size_t tmp_bytes = 0;
    if (cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, ro_in, ro_in, (int)(m + 1), st) != cudaSuccess)
        return SPMM_ERR_CUDA;
    void* tmp = nullptr;
    if (cudaMallocAsync(&tmp, tmp_bytes, st) != cudaSuccess) return SPMM_ERR_CUDA;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, ro_in, ro_in, (int)(m + 1), st);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, ro_out, ro_out, (int)(m + 1), st);
    cudaFreeAsync(tmp, st);
    if (e != cudaSuccess) return SPMM_ERR_CUDA;
    if (nnz > 0) {
        k_split_scatter<<<grid, kThreads, 0, st>>>(row_offsets, col_indices, static_cast<const unsigned*>(values), m, c0,
                                                   c1, ro_in, col_in, static_cast<unsigned*>(val_in), ro_out, col_out,
                                                   static_cast<unsigned*>(val_out));
        if (cudaGetLastError() != cudaSuccess) return SPMM_ERR_CUDA;
    }
    int32_t tot = 0;
    if (cudaMemcpyAsync(&tot, ro_in + m, sizeof(int32_t), cudaMemcpyDeviceToHost, st) != cudaSuccess) return SPMM_ERR_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return SPMM_ERR_CUDA;
    *nnz_in = tot;
    return SPMM_OK;
}
