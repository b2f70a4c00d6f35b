// kernels.h -- host-side interface between the C ABI (spmm_api.cu) and the kernel translation units
// (inst_*.cu, one per value type x semiring, compiled in parallel): launch configuration types, the
// compile-time tuning constants of the kernels, and the per-kind launch entry points.
#pragma once
#include <cuda_runtime.h>

#include "common.cuh"
#include "merge_f.cuh"
#include "merge_w.cuh"
#include "tile.cuh"
#include "tiled.cuh"

#ifndef RS_U
#define RS_U 8  // row split: B rows gathered back to back per row group
#endif
#ifndef RS_U4
#define RS_U4 4  // row split, 4 float4 blocks per lane (n > 96): B rows gathered back to back per row group
#endif
#ifndef MW_U
#define MW_U 8  // merge: B rows gathered per batch (row of <= 2 values per lane)
#endif
#ifndef MW_U4
#define MW_U4 4  // merge: B rows per batch when a lane holds 3-4 values of a row (n > 64)
#endif
#ifndef MW_MINB
#define MW_MINB 5  // merge: 256-thread CTAs per SM (40 warps, <= 48 registers; 6 x 40 registers spills)
#endif
#ifndef MW_MINB1
#define MW_MINB1 6  // merge, one value per lane (n <= 32): 48 warps (40 registers; spills only outside the
                    // gather loop; R-MAT 22 n = 32 1.18 -> 1.09 ms, profiles/r02_s3_experiments.txt)
#endif
#ifndef MW_TPW
#define MW_TPW 1  // merge: tasks per resident warp (1: one static task per warp; > 1: tasks from a queue)
#endif
#ifndef MW_TPW_SKEW
#define MW_TPW_SKEW 8  // merge, AUTO policy, skewed row lengths: tasks per warp, from the queue
#endif
#ifndef TL_MIN_D
#define TL_MIN_D 1000000000.0  // AUTO picks the tiled kernel from this mean row length (set from the sweep)
#endif
#ifndef TL_TMA
#define TL_TMA 1  // tiled: B blocks by TMA bulk copies (1) or cp.async from every thread (0)
#endif
#ifndef TL_RPG
#define TL_RPG 4  // tiled: rows per row group (accumulators held across the whole K loop)
#endif
#ifndef MW_MIN_ITEMS_DYN
#define MW_MIN_ITEMS_DYN 1024  // merge, tasks from the queue: fewest items per task
#endif
#ifndef MF_MAX_N
#define MF_MAX_N 16  // merge: lane-folded workers (k_merge_f) for n <= MF_MAX_N
#endif
#ifndef MF_L
#define MF_L 8  // merge, folded: items per slot per chunk
#endif
#ifndef MF_MINB
#define MF_MINB 8  // merge, folded: 128-thread CTAs per SM the register allocation targets (VEC = 1)
#endif
#ifndef MF_L_NARROW
#define MF_L_NARROW 4  // merge, folded, 1-2 lanes per slot: items per slot per chunk
#endif
#ifndef MF_MINB_NARROW
#define MF_MINB_NARROW 12  // merge, folded, 1-2 lanes per slot: CTAs per SM (48 warps)
#endif
#ifndef MF_L_NARROW4
#define MF_L_NARROW4 6  // merge, folded, float4, 1-2 lanes per slot: items per slot per chunk (n = 8 R-MAT 22
                        // 721 -> 637 us vs L = 4; with scalar / float2 slots L > 4 is slower)
#endif
#ifndef MF_MINB4_NARROW
#define MF_MINB4_NARROW 8  // merge, folded, float4, 1-2 lanes per slot (4 values per gather: 64 registers)
#endif
#ifndef MF_MINB4
#define MF_MINB4 6  // merge, folded, VEC = 4 (8 gathers x 4 values in flight per lane)
#endif
#ifndef MW_MINB4
#define MW_MINB4 4  // merge, 2-4 values of a row per lane (64 registers: no spills)
#endif

namespace spmm {

constexpr int kNumSMs = 148;

// vector shape of a launch: VEC elements per lane access, G lanes per row group (row split) / per
// worker slot (merge), NV vector blocks per lane
struct VecCfg {
    int vec, G, NV;
};

inline int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        int v = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = kNumSMs;
        sms = v;
    }
    return sms;
}

// k_tile<ROWSPLIT> for this vector shape (cudaErrorNotSupported if no instance)
template <typename T, int SR> cudaError_t rowsplit_kernel(VecCfg cfg, const TileParams& P, cudaStream_t st);
// k_merge_w (cfg.G == 32) / k_merge_f (lane-folded) for this vector shape; M == nullptr: only report
// the resident warps per SM in *per_sm_out
template <typename T, int SR>
cudaError_t merge_w_launch(VecCfg cfg, const MergeParams* M, cudaStream_t st, int* per_sm_out);
template <typename T, int SR>
cudaError_t merge_f_launch(VecCfg cfg, const MergeParams* M, cudaStream_t st, int* per_sm_out);
// k_tiled (NEXT-4) for row groups of cfg.G lanes x cfg.NV float4 blocks
template <typename T, int SR> cudaError_t tiled_launch(VecCfg cfg, const TiledParams& P, cudaStream_t st);

#define SPMM_EXTERN_KIND(T, SR)                                                                             \
    extern template cudaError_t rowsplit_kernel<T, SR>(VecCfg, const TileParams&, cudaStream_t);            \
    extern template cudaError_t merge_w_launch<T, SR>(VecCfg, const MergeParams*, cudaStream_t, int*);     \
    extern template cudaError_t merge_f_launch<T, SR>(VecCfg, const MergeParams*, cudaStream_t, int*);     \
    extern template cudaError_t tiled_launch<T, SR>(VecCfg, const TiledParams&, cudaStream_t);
SPMM_EXTERN_KIND(float, SR_PLUS_TIMES)
SPMM_EXTERN_KIND(float, SR_MIN_PLUS)
SPMM_EXTERN_KIND(int, SR_PLUS_TIMES)
SPMM_EXTERN_KIND(int, SR_MIN_PLUS)
#undef SPMM_EXTERN_KIND

}  // namespace spmm
