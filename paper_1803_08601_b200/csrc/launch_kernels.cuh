// launch_kernels.cuh -- definitions of the per-kind launch entry points declared in kernels.h: kernel
// attribute / occupancy caching, grid sizing (persistent CTAs: resident CTAs per SM x SMs) and the
// switch over the template instances.  Included only by the inst_*.cu translation units.
#pragma once
#include <algorithm>
#include <mutex>

#include "kernels.h"

namespace spmm {

// Kernel attributes are set and the occupancy is queried once per (kernel instance, device, shared
// memory size) -- not on every execute (host overhead on the launch-bound small configs).
struct LaunchCache {
    int dev = -1;
    size_t smem_set = 0;   // largest dynamic shared memory size set so far on `dev`
    size_t smem_q = 0;     // shared memory size of the cached occupancy query
    int per_sm = 0;
};

template <typename T, int SR, int MODE, int V, int G, int NV, int U>
cudaError_t launch_tile(const TileParams& P, cudaStream_t st) {
    void (*kfn)(const TileParams) = k_tile<T, SR, MODE, V, G, NV, U>;
    static std::mutex mu;
    static LaunchCache cache[8];
    const size_t smem = te_smem_bytes(P.capr, P.capz, (int)sizeof(T), P.stages, P.capb);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    {
        std::lock_guard<std::mutex> lock(mu);
        LaunchCache& c = cache[dev & 7];
        if (c.dev != dev) c = LaunchCache{dev, 0, 0, 0};
        if (smem > c.smem_set) {
            e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            c.smem_set = smem;
        }
        if (c.per_sm == 0 || c.smem_q != smem) {
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c.per_sm, kfn, TE_THREADS, smem);
            if (e != cudaSuccess) { c.per_sm = 0; return e; }
            c.smem_q = smem;
        }
        per_sm = c.per_sm;
    }
    if (per_sm <= 0) return cudaErrorInvalidConfiguration;
    const long long grid = std::min<long long>(P.num_ranges, (long long)per_sm * num_sms());
    if (grid <= 0) return cudaSuccess;
    kfn<<<(unsigned)grid, TE_THREADS, smem, st>>>(P);
    return cudaGetLastError();
}

template <typename T, int SR>
cudaError_t rowsplit_kernel(VecCfg cfg, const TileParams& P, cudaStream_t st) {
#define RS_CASE_U(V, G_, NV_, U_) \
    case (V)*1000 + (G_)*10 + (NV_): return launch_tile<T, SR, MODE_ROWSPLIT, V, G_, NV_, U_>(P, st);
#define RS_CASE(V, G_, NV_) RS_CASE_U(V, G_, NV_, RS_U)
    switch (cfg.vec * 1000 + cfg.G * 10 + cfg.NV) {
        RS_CASE(4, 1, 1) RS_CASE(4, 2, 1) RS_CASE(4, 4, 1) RS_CASE(4, 8, 1) RS_CASE(4, 8, 2) RS_CASE(4, 16, 2)
        RS_CASE(4, 4, 4) RS_CASE_U(4, 8, 4, RS_U4)
        RS_CASE(2, 1, 1) RS_CASE(2, 2, 1) RS_CASE(2, 4, 1) RS_CASE(2, 8, 1) RS_CASE(2, 8, 2) RS_CASE(2, 16, 2)
        RS_CASE(2, 32, 2)
        RS_CASE(1, 1, 1) RS_CASE(1, 2, 1) RS_CASE(1, 4, 1) RS_CASE(1, 8, 1) RS_CASE(1, 8, 2) RS_CASE(1, 16, 2)
        RS_CASE(1, 32, 2) RS_CASE(1, 32, 3) RS_CASE(1, 32, 4)
        default: return cudaErrorNotSupported;
    }
#undef RS_CASE
#undef RS_CASE_U
}

// launch of a warp-task merge kernel (k_merge_w / k_merge_f): persistent grid of resident CTAs x SMs,
// capped at one warp per task.  With M == nullptr only the resident CTAs per SM are returned in
// *per_sm_out (plan sizes the merge-path tasks from it: one task per resident warp by default).
template <void (*KFN)(const MergeParams), int NT>
cudaError_t launch_warp_tasks(const MergeParams* M, cudaStream_t st, int* per_sm_out) {
    static std::mutex mu;
    static int per_sm_cache[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    int per_sm;
    {
        std::lock_guard<std::mutex> lock(mu);
        int& c = per_sm_cache[dev & 7];
        if (c == 0) {
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&c, KFN, NT, 0);
            if (e != cudaSuccess) { c = 0; return e; }
        }
        per_sm = c;
    }
    if (per_sm <= 0) return cudaErrorInvalidConfiguration;
    if (per_sm_out) *per_sm_out = per_sm * (NT / 32);  // resident warps per SM
    if (!M) return cudaSuccess;
    const long long grid = std::min<long long>((M->num_tasks + NT / 32 - 1) / (NT / 32), (long long)per_sm * num_sms());
    if (grid <= 0) return cudaSuccess;
    KFN<<<(unsigned)grid, NT, 0, st>>>(*M);
    return cudaGetLastError();
}

// dispatch over the k_merge_w instances by vector shape (pick_vec with G = 32)
template <typename T, int SR>
cudaError_t merge_w_launch(VecCfg cfg, const MergeParams* M, cudaStream_t st, int* per_sm_out) {
#define MW_CASE(V, NV_, U_, MB_) \
    case (V)*10 + (NV_):                                                                                   \
        return epi ? launch_warp_tasks<k_merge_w<T, SR, V, NV_, U_, MB_, true>, MW_THREADS>(M, st, per_sm_out)  \
                   : launch_warp_tasks<k_merge_w<T, SR, V, NV_, U_, MB_, false>, MW_THREADS>(M, st, per_sm_out);
    const bool epi = M && (M->epi.accumulate || M->epi.npeers);  // epilogue instances only when requested
    switch (cfg.vec * 10 + cfg.NV) {
        MW_CASE(4, 1, MW_U4, MW_MINB4) MW_CASE(2, 1, MW_U, MW_MINB) MW_CASE(2, 2, MW_U4, MW_MINB4)
        MW_CASE(1, 1, MW_U, MW_MINB1) MW_CASE(1, 2, MW_U, MW_MINB4) MW_CASE(1, 3, MW_U4, MW_MINB4)
        MW_CASE(1, 4, MW_U4, MW_MINB4)
        default: return cudaErrorNotSupported;
    }
#undef MW_CASE
}

// dispatch over the k_merge_f instances (lane-folded merge, n <= MF_MAX_N): VEC in {1, 2, 4}, G lanes per slot
template <typename T, int SR>
cudaError_t merge_f_launch(VecCfg cfg, const MergeParams* M, cudaStream_t st, int* per_sm_out) {
#define MF_CASE(V, G_, L_, MB_) \
    case (V)*100 + (G_):                                                                                   \
        return epi ? launch_warp_tasks<k_merge_f<T, SR, V, G_, L_, MB_, true>, MF_THREADS>(M, st, per_sm_out)  \
                   : launch_warp_tasks<k_merge_f<T, SR, V, G_, L_, MB_, false>, MF_THREADS>(M, st, per_sm_out);
    const bool epi = M && (M->epi.accumulate || M->epi.npeers);
    // 1-2 lanes per slot (n <= 2, or n <= 8 with float4): short chunks (L = 4; 6 with float4, which has
    // the registers for it) and more resident warps; wider slots: L = 8 (profiles/r02_fold_tuning.txt,
    // r02_s3_experiments.txt)
    switch (cfg.vec * 100 + cfg.G) {
        MF_CASE(4, 1, MF_L_NARROW4, MF_MINB4_NARROW) MF_CASE(4, 2, MF_L_NARROW4, MF_MINB4_NARROW) MF_CASE(4, 4, MF_L, MF_MINB4)
        MF_CASE(2, 1, MF_L_NARROW, MF_MINB_NARROW) MF_CASE(2, 2, MF_L_NARROW, MF_MINB_NARROW) MF_CASE(2, 4, MF_L, MF_MINB)
        MF_CASE(2, 8, MF_L, MF_MINB)
        MF_CASE(1, 1, MF_L_NARROW, MF_MINB_NARROW) MF_CASE(1, 2, MF_L_NARROW, MF_MINB_NARROW) MF_CASE(1, 4, MF_L, MF_MINB)
        MF_CASE(1, 8, MF_L, MF_MINB) MF_CASE(1, 16, MF_L, MF_MINB)
        default: return cudaErrorNotSupported;
    }
#undef MF_CASE
}

// A/B-tiled kernel (NEXT-4): G lanes x NV float4 blocks per row group, RPG rows per group
template <typename T, int SR, int G, int NV>
cudaError_t launch_tiled(const TiledParams& P, cudaStream_t st) {
    void (*kfn)(const TiledParams) = k_tiled<T, SR, G, NV, TL_RPG>;
    const size_t smem = 2 * (size_t)P.kb * (size_t)P.n * sizeof(T);
    static std::mutex mu;
    static size_t smem_set[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (smem > smem_set[dev & 7]) {
            e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            smem_set[dev & 7] = smem;
        }
    }
    const long long grid = ((long long)P.m + P.rows_per_cta - 1) / P.rows_per_cta;
    if (grid <= 0) return cudaSuccess;
    kfn<<<(unsigned)grid, TL_THREADS, smem, st>>>(P);
    return cudaGetLastError();
}

template <typename T, int SR>
cudaError_t tiled_launch(VecCfg cfg, const TiledParams& P, cudaStream_t st) {
    switch (cfg.G * 10 + cfg.NV) {
        case 81: return launch_tiled<T, SR, 8, 1>(P, st);
        case 82: return launch_tiled<T, SR, 8, 2>(P, st);
        case 162: return launch_tiled<T, SR, 16, 2>(P, st);
        default: return cudaErrorNotSupported;
    }
}

#define SPMM_INSTANTIATE_KIND(T, SR)                                                                        \
    template cudaError_t rowsplit_kernel<T, SR>(VecCfg, const TileParams&, cudaStream_t);                   \
    template cudaError_t merge_w_launch<T, SR>(VecCfg, const MergeParams*, cudaStream_t, int*);            \
    template cudaError_t merge_f_launch<T, SR>(VecCfg, const MergeParams*, cudaStream_t, int*);            \
    template cudaError_t tiled_launch<T, SR>(VecCfg, const TiledParams&, cudaStream_t);

}  // namespace spmm
