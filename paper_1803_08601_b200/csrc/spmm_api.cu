// spmm_api.cu -- the C ABI of libspmm.so (include/spmm.h): handle, planner, §5.4 heuristic,
// workspace sizing, argument checks and kernel dispatch for the sm_100a CSR SpMM kernels.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>

#include "../../include/spmm.h"
#include "common.cuh"
#include "kernels.h"
#include "merge.cuh"

namespace {
// NVTX range around each C-ABI call (create / plan / execute / multiply_host), visible to nsys / ncu
// --nvtx; header-only NVTX v3: a no-op function-pointer call when no tool is attached
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

using namespace spmm;

struct spmm_csr_s {
    int64_t m = 0, k = 0, nnz = 0;
    const int32_t* ro = nullptr;
    const int32_t* col = nullptr;
    const void* val = nullptr;
    spmm_dtype dtype = SPMM_F32;
    // plan
    bool planned = false;
    int32_t n = 0;
    spmm_algo chosen = SPMM_ALGO_ROWSPLIT;
    spmm_semiring sr = SPMM_PLUS_TIMES;
    spmm_plan_opts opts{};
    double threshold = 9.35;
    int64_t max_row = -1;
    int64_t num_ctas = 0;
    int32_t items = 2048;
    int32_t rows_per_tile = 128;  // row split: rows per tile
    int32_t capz = 4104;          // row split: staged nonzeros per tile (+8 slack)
    int32_t capb = 0;             // row split: bytes of staged B row span per stage (0 = gather B from global)
    bool rs_dyn = false;          // row split: tiles from a queue in the workspace (irregular row lengths)
    bool mfold = false;           // merge: lane-folded workers (k_merge_f) instead of whole warps (k_merge_w)
    bool mdyn = false;            // merge: warps take tasks from a queue in the workspace
    double bspan_compact = -1.0;  // fraction of nonzeros in row tiles whose B span is compact (plan-time)
    int32_t tl_kb = 0;            // tiled: B rows per shared-memory block
    int sorted = -1;              // column indices non-decreasing within rows: -1 unknown, 0 no, 1 yes
    size_t ws_bytes = 0;
    int* d_scratch = nullptr;  // 32 bytes: plan-time reductions / validation flags (stream-ordered allocation)
    cudaStream_t st_alloc = nullptr;  // stream d_scratch was allocated on (freed on it: no device sync)
    int64_t hint_max_row = -1;        // longest row when known on the host (skips plan's device reduction)
    cudaEvent_t ev[8] = {};    // optional per-kernel timing events (spmm_csr_set_timing_events)
    int32_t nev = 0;
    std::string err;
};

namespace {

#ifndef RS_DYN_SKEW
#define RS_DYN_SKEW 4.0  // row split takes tiles from a queue when (AUTO) max row > RS_DYN_SKEW x mean row
#endif
#ifndef RS_G8_MAX_D
#define RS_G8_MAX_D 64.0  // row split, n > 96: 8-lane groups up to this mean row length, 16 lanes above
#endif
#ifndef RS_GDIV
#define RS_GDIV 2  // row split, 16..32 vector lanes per row: split the row over lanes/RS_GDIV lanes
#endif
#ifndef RS_STAGES
#define RS_STAGES 3
#endif
#ifndef RS_TILE_NNZ
#define RS_TILE_NNZ 2048  // row split: target nonzeros per row tile
#endif
#ifndef RS_CAPZ_MAX
#define RS_CAPZ_MAX 8200  // row split: most nonzeros a staged tile slice holds (+8 slack)
#endif
#ifndef RS_ZF
#define RS_ZF 12  // row split: staged capacity = RS_ZF/10 x the tile's expected nonzeros
#endif
#ifndef MG_ITEMS
#define MG_ITEMS 0  // merge-path items per task; 0 = sized at plan time (about 16 tasks per resident warp)
#endif
constexpr int kDefaultItems = MG_ITEMS;
#ifndef RS_BSTAGE
#define RS_BSTAGE 1  // row split: stage compact B row spans into shared memory with TMA (plan-time measured)
#endif
#ifndef RS_BSTAGE_MIN_ROW
#define RS_BSTAGE_MIN_ROW 256  // stage B only for rows of >= 256 bytes (n >= 64 fp32); below, L1 serves
#endif                         // the short rows better (measured: banded n=16/32 slower when staged)
#ifndef RS_BSTAGE_MIN
#define RS_BSTAGE_MIN 0.5  // stage B when at least this fraction of the nonzeros lies in compact tiles
#endif
#ifndef RS_BSTAGE_SMEM
#define RS_BSTAGE_SMEM 110000  // shared-memory budget per CTA with B staging (2 CTAs per SM)
#endif
spmm_status fail(spmm_csr_t h, spmm_status s, const std::string& msg) {
    if (h) h->err = msg;
    return s;
}

spmm_status cuda_fail(spmm_csr_t h, cudaError_t e, const char* where) {
    if (h) h->err = std::string(where) + ": " + cudaGetErrorString(e);
    return SPMM_ERR_CUDA;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

inline void mark(const spmm_csr_s* h, int i, cudaStream_t st) {
    if (i < h->nev && h->ev[i]) cudaEventRecord(h->ev[i], st);
}

// ------------------------------------------------------------------------------------------------
// device helpers for create/plan
// ------------------------------------------------------------------------------------------------
__global__ void k_max_row(const int* __restrict__ ro, long long m, int* __restrict__ out) {
    int best = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
        best = max(best, ro[i + 1] - ro[i]);
    best = __reduce_max_sync(FULL, best);
    if ((threadIdx.x & 31) == 0) atomicMax(out, best);
}

// B-span compactness for the row-split kernel's B staging: warp per row tile of R rows; a tile is
// compact when its column span [lo, hi] holds at most 2 B rows per nonzero and fits capb bytes at
// row_bytes per row.  out[0] += nonzeros of compact tiles; out[1] = max bytes of a compact span.
__global__ void k_tile_span(const int* __restrict__ ro, const int* __restrict__ col, long long m, int R,
                            long long row_bytes, long long capb, unsigned long long* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const long long tiles = (m + R - 1) / R;
    const long long nw = (long long)gridDim.x * (blockDim.x / 32);
    unsigned long long acc = 0, mx = 0;
    for (long long t = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32; t < tiles; t += nw) {
        const long long rs = t * R, re = min(m, rs + R);
        const int zs = ro[rs], ze = ro[re];
        int lo = 0x7fffffff, hi = -1;
        for (int p = zs + lane; p < ze; p += 32) {
            const int c = col[p];
            lo = min(lo, c);
            hi = max(hi, c);
        }
        lo = __reduce_min_sync(FULL, lo);
        hi = __reduce_max_sync(FULL, hi);
        const long long cnt = ze - zs, span = (long long)hi - lo + 1;
        if (cnt > 0 && span <= 2 * cnt && span * row_bytes <= capb) {
            acc += (unsigned long long)cnt;
            mx = max(mx, (unsigned long long)(span * row_bytes));
        }
    }
    if (lane == 0 && acc) {
        atomicAdd(out, acc);
        atomicMax(out + 1, mx);
    }
}

// plan-time check, warp per row: column indices non-decreasing within every row (flag = 1 otherwise)
__global__ void k_check_sorted(const int* __restrict__ ro, const int* __restrict__ col, long long m,
                               int* __restrict__ flag) {
    const int lane = threadIdx.x & 31;
    const long long nw = (long long)gridDim.x * (blockDim.x / 32);
    int bad = 0;
    for (long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32; r < m; r += nw) {
        const int s = ro[r], e = ro[r + 1];
        for (int q = s + 1 + lane; q < e; q += 32) bad |= (col[q] < col[q - 1]) ? 1 : 0;
    }
    if (__any_sync(FULL, bad) && lane == 0) atomicOr(flag, 1);
}

// flags: bit0 ro[0] != 0, bit1 decreasing offsets, bit2 ro[m] != nnz, bit3 column out of range
__global__ void k_validate(const int* __restrict__ ro, long long m, long long nnz, const int* __restrict__ col,
                           long long k, int* __restrict__ flags) {
    int f = 0;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long step = (long long)gridDim.x * blockDim.x;
    if (tid == 0) {
        if (ro[0] != 0) f |= 1;
        if ((long long)ro[m] != nnz) f |= 4;
    }
    for (long long i = tid; i < m; i += step)
        if (ro[i + 1] < ro[i]) f |= 2;
    for (long long p = tid; p < nnz; p += step) {
        const int c = col[p];
        if (c < 0 || (long long)c >= k) f |= 8;
    }
    if (f) atomicOr(flags, f);
}

int pow2ceil(int x) {
    int p = 1;
    while (p < x) p <<= 1;
    return p;
}

VecCfg pick_vec(int n, const void* B, int64_t ldb, const void* C, int64_t ldc, bool folded, double d = 0.0) {
    const uintptr_t pb = (uintptr_t)B, pc = (uintptr_t)C;
    int vec = 1;
    if (n % 4 == 0 && ldb % 4 == 0 && ldc % 4 == 0 && pb % 16 == 0 && pc % 16 == 0) vec = 4;
    else if (n % 2 == 0 && ldb % 2 == 0 && ldc % 2 == 0 && pb % 8 == 0 && pc % 8 == 0) vec = 2;
    const int lanes = (n + vec - 1) / vec;
    VecCfg c;
    c.vec = vec;
    if (folded) {
        // row groups of G lanes; for 16..32 lanes split the row over half as many lanes with two
        // column blocks each (n = 64: 8 lanes x 2 float4) -- more rows per warp, fewer broadcast loads
        const int G0 = std::min(32, pow2ceil(lanes));
        if (lanes <= 32 && G0 >= 16) {
            // n = 97..128 with float4 and rows of <= 64 entries (d = mean row length): 8 lanes x 4 blocks
            // (4 rows per warp; banded n = 128 3% faster than 16 x 2, short rows up to 1.7x; rows of
            // 256+ entries 1.7-1.8x slower, profiles/r02_s3_experiments.txt); n = 64: 8 lanes x 2 blocks
            c.G = (G0 == 32 && vec == 4 && lanes > 24 && d <= RS_G8_MAX_D) ? 8 : G0 / RS_GDIV;
            c.NV = (lanes + c.G - 1) / c.G;
        } else {
            c.G = G0;
            c.NV = (lanes + 31) / 32;
        }
    } else {  // merge: one worker per warp, narrowest vector that covers n with 32 lanes
        const int want = n <= 32 ? 1 : (n <= 64 ? 2 : 4);
        if (want < vec) c.vec = want;
        const int l2 = (n + c.vec - 1) / c.vec;
        c.G = 32;
        c.NV = (l2 + 31) / 32;
    }
    return c;
}

inline double mean_row(const spmm_csr_s* h) { return h->m > 0 ? (double)h->nnz / (double)h->m : 0.0; }

template <typename T, int SR>
cudaError_t launch_rowsplit(const spmm_csr_s* h, VecCfg cfg, TileParams P, cudaStream_t st) {
    P.num_ranges = (int)((h->m + h->rows_per_tile - 1) / h->rows_per_tile);
    P.rows_per_tile = h->rows_per_tile;
    P.capr = h->rows_per_tile + 8;
    P.capz = h->capz;
    P.stages = RS_STAGES;
    // B staging needs 16-byte aligned B rows (TMA bulk copy source)
    P.capb = (h->capb > 0 && ((uintptr_t)P.B % 16) == 0 && (P.ldb_bytes % 16) == 0) ? h->capb : 0;
    cudaError_t e;
    mark(h, 0, st);
    int ev = 1;
    if (h->rs_dyn) {
        // irregular row lengths: row tiles from a queue in the workspace, zeroed here;
        // counted as launch 0 of the execute (spmm_plan_info.launches_per_execute / compute_launch)
        e = cudaMemsetAsync(P.tile_ctr, 0, sizeof(int), st);
        if (e != cudaSuccess) return e;
        mark(h, ev++, st);
    } else {
        P.tile_ctr = nullptr;
    }
    e = rowsplit_kernel<T, SR>(cfg, P, st);
    mark(h, ev, st);
    return e;
}


// lane-folded merge workers (k_merge_f): VEC = 4 when n, ldb, ldc and the B / C bases allow 16-byte
// vectors, else 1; G = lanes per slot covering n columns
VecCfg pick_fold(int n, const void* B, int64_t ldb, const void* C, int64_t ldc) {
    const uintptr_t pb = (uintptr_t)B, pc = (uintptr_t)C;
    VecCfg c;
    // float4 when n, ldb, ldc and the bases allow it, else float2 (n = 2: one lane per slot, 32 slots --
    // half the chunk overhead of two scalar lanes), else scalar
    if (n % 4 == 0 && ldb % 4 == 0 && ldc % 4 == 0 && pb % 16 == 0 && pc % 16 == 0) c.vec = 4;
    else if (n % 2 == 0 && ldb % 2 == 0 && ldc % 2 == 0 && pb % 8 == 0 && pc % 8 == 0) c.vec = 2;
    else c.vec = 1;
    c.G = pow2ceil((n + c.vec - 1) / c.vec);
    c.NV = 1;
    return c;
}

// tiled kernel row groups: float4 over n (n % 4 == 0), G lanes x NV blocks as the row split picks them
VecCfg tiled_cfg(int n) {  // the tiled kernel keeps 16-lane groups at n > 96
    VecCfg c = pick_vec(n, nullptr, 4, nullptr, 4, true);
    if (c.G == 8 && c.NV == 4) { c.G = 16; c.NV = 2; }
    return c;
}
bool tiled_shape_ok(int n) {
    if (n % 4 != 0 || n < 32 || n > 128) return false;
    const VecCfg c = tiled_cfg(n);
    return c.vec == 4 && ((c.G == 8 && (c.NV == 1 || c.NV == 2)) || (c.G == 16 && c.NV == 2));
}

// resident warps per SM of the merge kernel instance used for this shape (0 on error)
int merge_per_sm_warps(spmm_dtype dt, spmm_semiring sr, VecCfg cfg, bool folded) {
    int per_sm = 0;
    cudaError_t e;
    if (folded) {
        if (dt == SPMM_F32) e = sr == SPMM_PLUS_TIMES ? merge_f_launch<float, SR_PLUS_TIMES>(cfg, nullptr, nullptr, &per_sm)
                                                      : merge_f_launch<float, SR_MIN_PLUS>(cfg, nullptr, nullptr, &per_sm);
        else e = sr == SPMM_PLUS_TIMES ? merge_f_launch<int, SR_PLUS_TIMES>(cfg, nullptr, nullptr, &per_sm)
                                       : merge_f_launch<int, SR_MIN_PLUS>(cfg, nullptr, nullptr, &per_sm);
    } else {
        if (dt == SPMM_F32) e = sr == SPMM_PLUS_TIMES ? merge_w_launch<float, SR_PLUS_TIMES>(cfg, nullptr, nullptr, &per_sm)
                                                      : merge_w_launch<float, SR_MIN_PLUS>(cfg, nullptr, nullptr, &per_sm);
        else e = sr == SPMM_PLUS_TIMES ? merge_w_launch<int, SR_PLUS_TIMES>(cfg, nullptr, nullptr, &per_sm)
                                       : merge_w_launch<int, SR_MIN_PLUS>(cfg, nullptr, nullptr, &per_sm);
    }
    return e == cudaSuccess ? per_sm : 0;
}

template <typename T, int SR>
cudaError_t launch_merge(const spmm_csr_s* h, VecCfg cfg, TileParams P, unsigned char* ws, cudaStream_t st) {
    const long long NC = h->num_ctas;
    if (NC <= 0) return cudaSuccess;
    int* states = reinterpret_cast<int*>(ws);
    size_t off = align256(sizeof(int) * 2 * (NC + 1));
    int* carry_row = reinterpret_cast<int*>(ws + off);
    off += align256(sizeof(int) * NC);
    int* carry_flag = reinterpret_cast<int*>(ws + off);
    off += align256(sizeof(int) * NC);
    T* carry_val = reinterpret_cast<T*>(ws + off);
    off += align256(sizeof(T) * (size_t)NC * h->n);
    int* task_ctr = h->mdyn ? reinterpret_cast<int*>(ws + off) : nullptr;  // zeroed by k_partition
    const int items = h->items;
    // phase 1: PartitionSpmm (Alg. 1 line 2)
    mark(h, 0, st);
    k_partition<<<partition_grid(h->m), THREADS, 0, st>>>(h->ro, (int)h->m, (int)h->nnz, items, h->opts.partition, (int)NC,
                                                     states, task_ctr);
    mark(h, 1, st);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // phase 2: per-task compute + carry-out (Alg. 1 lines 3-23)
    MergeParams M{};
    M.m = P.m; M.n = P.n; M.nnz = P.nnz;
    M.ro = P.ro; M.col = P.col; M.val = P.val;
    M.B = P.B; M.ldb_bytes = P.ldb_bytes; M.C = P.C; M.ldc = P.ldc;
    M.states = states;
    M.num_tasks = (int)NC;
    M.carry_row = carry_row;
    M.carry_flag = carry_flag;
    M.carry_val = carry_val;
    M.task_ctr = task_ctr;
    M.epi = P.epi;
    e = h->mfold ? merge_f_launch<T, SR>(cfg, &M, st, nullptr) : merge_w_launch<T, SR>(cfg, &M, st, nullptr);
    mark(h, 2, st);
    if (e != cudaSuccess) return e;
    // phase 3: FixCarryOut (Alg. 1 line 24)
    k_fixup<T, SR><<<fixup_grid(NC), THREADS, 0, st>>>((int)NC, h->n, carry_row, carry_flag, carry_val,
                                                        static_cast<T*>(P.C), P.ldc, P.epi);
    mark(h, 3, st);
    return cudaGetLastError();
}

template <typename T, int SR>
cudaError_t run(const spmm_csr_s* h, const void* Bv, long long ldb, void* Cv, long long ldc, void* ws,
                const EpiParams& epi, cudaStream_t st) {
    TileParams P{};
    P.m = (int)h->m;
    P.n = h->n;
    P.nnz = (int)h->nnz;
    P.ro = h->ro;
    P.col = h->col;
    P.val = h->val;
    P.B = Bv;
    P.ldb_bytes = (unsigned)(ldb * (long long)sizeof(T));
    P.C = Cv;
    P.ldc = ldc;
    P.epi = epi;
#ifndef PF_OFF
    // L2 prefetch of gathered B rows: needs 16B-aligned rows; prefetch whole 16-byte granules only
    if (((uintptr_t)Bv % 16) == 0 && (P.ldb_bytes % 16) == 0 && h->n * sizeof(T) >= 16)
        P.pf_bytes = (unsigned)((h->n * sizeof(T)) & ~(size_t)15);
#endif
    if (h->chosen == SPMM_ALGO_TILED) {
        TiledParams Q{};
        Q.m = P.m; Q.n = P.n; Q.k = (int)h->k; Q.nnz = P.nnz;
        Q.ro = P.ro; Q.col = P.col; Q.val = P.val;
        Q.B = Bv; Q.ldb = ldb; Q.C = Cv; Q.ldc = ldc;
        Q.kb = h->tl_kb;
        Q.rows_per_cta = h->rows_per_tile;
        Q.b_vec4 = ((uintptr_t)Bv % 16) == 0 && ldb % 4 == 0;
        Q.b_tma = Q.b_vec4 && TL_TMA;
        Q.c_vec4 = ((uintptr_t)Cv % 16) == 0 && ldc % 4 == 0;
        Q.epi = P.epi;
        mark(h, 0, st);
        const cudaError_t e = tiled_launch<T, SR>(tiled_cfg(h->n), Q, st);
        mark(h, 1, st);
        return e;
    }
    if (h->chosen == SPMM_ALGO_ROWSPLIT) {
        P.tile_ctr = static_cast<int*>(ws);
        return launch_rowsplit<T, SR>(h, pick_vec(h->n, Bv, ldb, Cv, ldc, true, mean_row(h)), P, st);
    }
    const VecCfg mc = h->mfold ? pick_fold(h->n, Bv, ldb, Cv, ldc) : pick_vec(h->n, Bv, ldb, Cv, ldc, false);
    return launch_merge<T, SR>(h, mc, P, static_cast<unsigned char*>(ws), st);
}

}  // namespace

// plan-time O(m) device reduction: the longest row (AUTO policy guards, row-split tile queue)
static spmm_status measure_max_row(spmm_csr_t h, void* stream) {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int hmax = 0;
    cudaError_t e = cudaMemsetAsync(h->d_scratch, 0, sizeof(int), st);
    if (e == cudaSuccess) {
        const int grid = (int)std::min<long long>((h->m + THREADS - 1) / THREADS, 8LL * kNumSMs);
        k_max_row<<<std::max(grid, 1), THREADS, 0, st>>>(h->ro, h->m, h->d_scratch);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hmax, h->d_scratch, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(h, e, "plan: max row length");
    h->max_row = hmax;
    return SPMM_OK;
}

// plan-time O(nnz) device check for the tiled kernel: are column indices non-decreasing within rows?
static spmm_status measure_sorted(spmm_csr_t h, void* stream) {
    if (h->sorted >= 0) return SPMM_OK;  // A is immutable while the handle lives: checked once
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int flag = 0;
    cudaError_t e = cudaMemsetAsync(h->d_scratch, 0, sizeof(int), st);
    if (e == cudaSuccess && h->m > 0) {
        const int grid = (int)std::min<long long>((h->m * 32 + THREADS - 1) / THREADS, 16LL * kNumSMs);
        k_check_sorted<<<std::max(grid, 1), THREADS, 0, st>>>(h->ro, h->col, h->m, h->d_scratch);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(&flag, h->d_scratch, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(h, e, "plan: sortedness check");
    h->sorted = flag ? 0 : 1;
    return SPMM_OK;
}

// ================================================================================================
// C ABI
// ================================================================================================
extern "C" {

int32_t spmm_abi_version(void) { return SPMM_ABI_VERSION; }

const char* spmm_status_string(spmm_status s) {
    switch (s) {
        case SPMM_OK: return "SPMM_OK";
        case SPMM_ERR_NULL_POINTER: return "SPMM_ERR_NULL_POINTER: a required pointer argument is NULL";
        case SPMM_ERR_INVALID_ARG: return "SPMM_ERR_INVALID_ARG: invalid size, leading dimension or enum";
        case SPMM_ERR_INVALID_CSR: return "SPMM_ERR_INVALID_CSR: CSR invariant violated";
        case SPMM_ERR_NOT_PLANNED: return "SPMM_ERR_NOT_PLANNED: execute before plan";
        case SPMM_ERR_WORKSPACE_TOO_SMALL: return "SPMM_ERR_WORKSPACE_TOO_SMALL";
        case SPMM_ERR_UNSUPPORTED: return "SPMM_ERR_UNSUPPORTED: configuration not implemented (n > 128?)";
        case SPMM_ERR_CUDA: return "SPMM_ERR_CUDA: CUDA runtime error";
    }
    return "unknown spmm_status";
}

const char* spmm_csr_last_error(spmm_csr_t h) {
    if (!h) return "null handle";
    return h->err.c_str();
}

spmm_status spmm_csr_create(spmm_csr_t* out, int64_t m, int64_t k, int64_t nnz, const int32_t* row_offsets,
                            const int32_t* col_indices, const void* values, spmm_dtype dtype, uint32_t flags,
                            void* stream) {
    NvtxRange nvtx_range("spmm_csr_create");
    if (!out) return SPMM_ERR_NULL_POINTER;
    *out = nullptr;
    if (m < 0 || k < 0 || nnz < 0 || m >= 0x7fffffffLL || k >= 0x7fffffffLL || nnz >= 0x7fffffffLL ||
        m + nnz >= 0x7fffffffLL)
        return SPMM_ERR_INVALID_ARG;
    if (k == 0 && nnz != 0) return SPMM_ERR_INVALID_ARG;
    if (dtype != SPMM_F32 && dtype != SPMM_I32) return SPMM_ERR_INVALID_ARG;
    if ((flags & ~SPMM_FLAG_VALIDATE) != 0u) return SPMM_ERR_INVALID_ARG;
    if (m > 0 && !row_offsets) return SPMM_ERR_NULL_POINTER;
    if (nnz > 0 && (!col_indices || !values)) return SPMM_ERR_NULL_POINTER;
    spmm_csr_s* h = new (std::nothrow) spmm_csr_s();
    if (!h) return SPMM_ERR_CUDA;
    h->m = m; h->k = k; h->nnz = nnz;
    h->ro = row_offsets; h->col = col_indices; h->val = values; h->dtype = dtype;
    h->st_alloc = static_cast<cudaStream_t>(stream);
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&h->d_scratch), 32, h->st_alloc);
    if (e != cudaSuccess) { delete h; return SPMM_ERR_CUDA; }
    if ((flags & SPMM_FLAG_VALIDATE) && m > 0) {
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        int hflags = 0;
        e = cudaMemsetAsync(h->d_scratch, 0, 16, st);
        if (e == cudaSuccess) {
            const long long work = std::max<long long>(m, nnz);
            const int grid = (int)std::min<long long>((work + THREADS - 1) / THREADS, 8LL * kNumSMs);
            k_validate<<<std::max(grid, 1), THREADS, 0, st>>>(row_offsets, m, nnz, col_indices, k, h->d_scratch);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(&hflags, h->d_scratch, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) {
            cudaFreeAsync(h->d_scratch, h->st_alloc);
            delete h;
            return SPMM_ERR_CUDA;
        }
        if (hflags) {
            cudaFreeAsync(h->d_scratch, h->st_alloc);
            delete h;
            return SPMM_ERR_INVALID_CSR;
        }
    }
    *out = h;
    return SPMM_OK;
}

spmm_status spmm_csr_destroy(spmm_csr_t h) {
    if (!h) return SPMM_OK;
    if (h->d_scratch) cudaFreeAsync(h->d_scratch, h->st_alloc);  // stream-ordered: no device-wide sync
    delete h;
    return SPMM_OK;
}

int64_t spmm_merge_num_ctas(int64_t m, int64_t nnz, int32_t items_per_cta, int32_t partition) {
    if (items_per_cta <= 0 || m < 0 || nnz < 0) return -1;
    if (m + nnz == 0) return 0;
    if (partition == SPMM_PARTITION_NONZERO_SPLIT) return std::max<int64_t>(1, (nnz + items_per_cta - 1) / items_per_cta);
    return (m + nnz + items_per_cta - 1) / items_per_cta;
}

spmm_status spmm_csr_plan_ex(spmm_csr_t h, int32_t n, spmm_algo algo, spmm_semiring sr, double threshold,
                             const spmm_plan_opts* opts, void* stream, size_t* workspace_bytes, spmm_algo* chosen) {
    NvtxRange nvtx_range("spmm_csr_plan");
    if (!h) return SPMM_ERR_NULL_POINTER;
    h->planned = false;
    if (n < 1) return fail(h, SPMM_ERR_INVALID_ARG, "n must be >= 1");
    if (n > 128) return fail(h, SPMM_ERR_UNSUPPORTED, "n > 128 is not implemented (SURVEY.md §8(b))");
    if (algo != SPMM_ALGO_AUTO && algo != SPMM_ALGO_ROWSPLIT && algo != SPMM_ALGO_MERGE && algo != SPMM_ALGO_TILED)
        return fail(h, SPMM_ERR_INVALID_ARG, "bad algo");
    if (sr != SPMM_PLUS_TIMES && sr != SPMM_MIN_PLUS) return fail(h, SPMM_ERR_INVALID_ARG, "bad semiring");
    spmm_plan_opts o{};
    if (opts) o = *opts;
    for (int i = 0; i < 3; ++i)
        if (o.reserved[i] != 0) return fail(h, SPMM_ERR_INVALID_ARG, "reserved plan option fields must be 0");
    if (o.merge_worker < 0 || o.merge_worker > 2) return fail(h, SPMM_ERR_INVALID_ARG, "bad merge_worker");
    if (o.tasks_per_warp < 0 || o.tasks_per_warp > 64) return fail(h, SPMM_ERR_INVALID_ARG, "tasks_per_warp must be in [0, 64]");
    if (o.policy != SPMM_POLICY_AUTO && o.policy != SPMM_POLICY_PAPER) return fail(h, SPMM_ERR_INVALID_ARG, "bad policy");
    if (o.partition != SPMM_PARTITION_MERGE_PATH && o.partition != SPMM_PARTITION_NONZERO_SPLIT)
        return fail(h, SPMM_ERR_INVALID_ARG, "bad partition");
    int items = o.items_per_cta ? o.items_per_cta : kDefaultItems;
    // merge worker: lane-folded slots for narrow B (Type-2 waste of a whole warp per worker at small n,
    // PAPER.md:64), else a whole warp over B's columns
    const bool fold = o.merge_worker == SPMM_MERGE_WORKER_FOLDED ||
                      (o.merge_worker == SPMM_MERGE_WORKER_AUTO && n <= MF_MAX_N);
    if (fold && n > 16) return fail(h, SPMM_ERR_UNSUPPORTED, "lane-folded merge workers need n <= 16");
    if (items != 0 && (items < 32 || items > (1 << 30) || items % 32 != 0))
        return fail(h, SPMM_ERR_INVALID_ARG, "items_per_cta must be a multiple of 32 in [32, 2^30]");
    h->threshold = threshold > 0 ? threshold : 9.35;
    h->n = n;
    h->sr = sr;
    h->mfold = fold;
    h->mdyn = false;
    h->max_row = h->hint_max_row;  // -1 unless the caller already knows it (spmm_csr_multiply_host)
    h->capb = 0;
    h->bspan_compact = -1.0;
    h->rs_dyn = false;
    const double d = h->m > 0 ? (double)h->nnz / (double)h->m : 0.0;  // PAPER.md:267, mean row length
    spmm_algo pick = algo;
    if (algo == SPMM_ALGO_AUTO) {
        if (o.policy == SPMM_POLICY_PAPER || h->m == 0) {
            // §5.4: "use merge-based on datasets whose mean row length is less than 9.35, and row split
            // otherwise"
            pick = (d < h->threshold) ? SPMM_ALGO_MERGE : SPMM_ALGO_ROWSPLIT;
        } else {
            // AUTO (B200 refit of §5.4, profiles/r01_config4_*): on this GPU the row-split
            // kernel handles short rows well, so the row-length threshold is replaced by the two causes of
            // Type 1 imbalance that merge path removes: a skewed row-length
            // distribution, or too few rows to fill the GPU's row groups.
            if (h->max_row < 0) {
                const spmm_status ms = measure_max_row(h, stream);
                if (ms != SPMM_OK) return ms;
            }
            const long long hmax = h->max_row;
            const bool skewed = (double)hmax > 16.0 * d && hmax >= 1024;
            const VecCfg rc = pick_vec(n, nullptr, n % 4 == 0 ? 4 : 1, nullptr, n % 4 == 0 ? 4 : 1, true, d);
            const long long groups = (long long)num_sms() * 2 * TE_CWARPS * (32 / rc.G);  // resident row groups
            // (only when there is enough work for idle row groups to matter: a small matrix is
            // launch-bound, and the single row-split launch beats merge's three -- config 0: 15 vs 51 us)
            const bool few_rows = h->m < 2 * groups && h->nnz >= (1LL << 20);
            // rows so long that even a 16-row tile overflows the staged CSR slice: the row-split kernel
            // would stream A from global per row group (measured 2.5x slower than merge at d = 1000,
            // profiles/r01_density_sweep.txt), while merge path stages fixed-size slices at any d
            const bool long_rows = RS_ZF / 10.0 * 16.0 * d > (double)(RS_CAPZ_MAX - 8);
            // (round 2 refit on the config-3 sweep, profiles/r02_config3_summary.txt, with the task queue
            // and the lane-folded workers): merge path also wins for mildly skewed rows (max row above 16 d
            // but under the 1024 floor) once B rows are >= 64 bytes, and for very short rows with wide B
            // (the row-split tiles then carry 1-2 nonzeros per row of per-row overhead; d = 3-4 at n > 96
            // went back to row split with its 8-lane x 4-block groups, profiles/r02_config3_summary.txt)
            const bool mild_skew = (double)hmax > 16.0 * d && hmax >= 256 && n >= 16;
            const bool short_rows = d < 3.0 && n >= 32;
            pick = (skewed || few_rows || long_rows || mild_skew || short_rows) ? SPMM_ALGO_MERGE : SPMM_ALGO_ROWSPLIT;
            // dense-ish rows (NEXT-4): B streamed once per row tile beats a B-row gather
            // per nonzero once d is large (measured crossover)
            if (d >= TL_MIN_D && !skewed && tiled_shape_ok(n)) {
                const spmm_status ss = measure_sorted(h, stream);
                if (ss != SPMM_OK) return ss;
                if (h->sorted == 1) pick = SPMM_ALGO_TILED;
            }
        }
    }
    if (pick == SPMM_ALGO_TILED) {
        if (!tiled_shape_ok(n)) return fail(h, SPMM_ERR_UNSUPPORTED, "tiled kernel needs n % 4 == 0 and 32 <= n <= 128");
        const spmm_status ss = measure_sorted(h, stream);
        if (ss != SPMM_OK) return ss;
        if (h->sorted != 1)
            return fail(h, SPMM_ERR_UNSUPPORTED, "tiled kernel needs column indices non-decreasing within rows");
    }
    h->chosen = pick;
    h->ws_bytes = 0;
    h->num_ctas = 0;
    if (pick == SPMM_ALGO_TILED) {
        const VecCfg tc = tiled_cfg(n);
        const size_t elem = h->dtype == SPMM_F32 ? sizeof(float) : sizeof(int);
        h->tl_kb = (int)std::max<size_t>(1, TL_BUF_BYTES / ((size_t)n * elem));
        h->rows_per_tile = (TL_THREADS / 32) * (32 / tc.G) * TL_RPG;
        h->num_ctas = (h->m + h->rows_per_tile - 1) / h->rows_per_tile;
        h->items = items ? items : 256;  // unused
        o.items_per_cta = h->items;
    } else if (pick == SPMM_ALGO_MERGE) {
        // tasks per warp: AUTO takes tasks from a queue on skewed row lengths (R-MAT: the cost of equal
        // merge-path slices varies with their B rows' cache behaviour; measured -12% on R-MAT 22), and
        // one static task per warp otherwise (uniform costs: the queue's smaller tasks only add work)
        int tpw = o.tasks_per_warp;
        if (tpw == 0) {
            tpw = MW_TPW;
            if (o.policy == SPMM_POLICY_AUTO && h->m > 0) {
                if (h->max_row < 0) {
                    const spmm_status ms = measure_max_row(h, stream);
                    if (ms != SPMM_OK) return ms;
                }
                if ((double)h->max_row > 16.0 * d && h->max_row >= 1024) tpw = MW_TPW_SKEW;
            }
        }
        h->mdyn = tpw > 1;
        if (items == 0) {
            // merge-path items per task (the partition granularity, Alg. 1 line 2): tpw tasks per
            // resident merge warp of the kernel instance this n uses with aligned B / C, so every warp
            // streams contiguous, equal slices of the path
            const int l4 = n % 4 == 0 ? 4 : (n % 2 == 0 ? 2 : 1);
            const VecCfg mc = fold ? pick_fold(n, nullptr, l4, nullptr, l4) : pick_vec(n, nullptr, l4, nullptr, l4, false);
            int per_sm = merge_per_sm_warps(h->dtype, sr, mc, fold);
            if (per_sm <= 0) per_sm = 32;
            const long long workers = (long long)num_sms() * per_sm * tpw;
            const long long path = o.partition == SPMM_PARTITION_NONZERO_SPLIT ? h->nnz : h->m + h->nnz;
            long long it = (path + workers - 1) / workers;
            // queued tasks are kept >= MW_MIN_ITEMS_DYN items: smaller ones cost more in queue and carry
            // traffic than they recover in balance (R-MAT 20, n = 1: 300-item tasks 24% slower)
            it = std::max<long long>(tpw > 1 ? MW_MIN_ITEMS_DYN : 256, (it + 31) / 32 * 32);
            items = (int)std::min<long long>(it, 1LL << 30);
        }
        o.items_per_cta = items;
        o.tasks_per_warp = tpw;
        h->items = items;
        const int64_t NC = spmm_merge_num_ctas(h->m, h->nnz, items, o.partition);
        h->num_ctas = NC;
        if (NC > 0) {
            const size_t elem = h->dtype == SPMM_F32 ? sizeof(float) : sizeof(int);
            h->ws_bytes = align256(sizeof(int) * 2 * (NC + 1)) + 2 * align256(sizeof(int) * NC) +
                          align256(elem * (size_t)NC * n) + (h->mdyn ? 256 : 0);
        }
    } else {
        h->items = items ? items : 256;  // unused by row split
        o.items_per_cta = h->items;
        // row tiles of R rows sized so a typical tile's nonzeros fit the staged shared-memory slice
        const double dd = std::max(1.0, d);
        int R = 1;
        while (R * 2 <= 4096 && R * 2 * dd <= (double)RS_TILE_NNZ) R *= 2;
        R = std::max(16, std::min(R, 1024));
#ifdef RS_R_FORCE
        R = RS_R_FORCE;  // tuning knob: fixed tile height
#endif
        auto capz_for = [&](int rows) {
            long long z = (long long)std::ceil(RS_ZF / 10.0 * rows * dd);
            z = std::max<long long>(1024, std::min<long long>(z, RS_CAPZ_MAX - 8));
            return (int)(((z + 3) & ~3LL) + 8);
        };
        h->rows_per_tile = R;
        h->capz = capz_for(R);
        h->capb = 0;
        h->bspan_compact = -1.0;
        const size_t elem = h->dtype == SPMM_F32 ? sizeof(float) : sizeof(int);
        if (RS_BSTAGE && h->nnz > 0 && (n * elem) % 16 == 0 && n * elem >= RS_BSTAGE_MIN_ROW) {
            // B staging: the largest tile height R_b <= R whose tiles' B row spans fit
            // the shared memory left next to the CSR slice (3 stages x 2 CTAs per SM) for at least
            // RS_BSTAGE_MIN of the nonzeros; the per-stage B slot is then sized to the largest
            // compact span measured.  The B row pitch is assumed to be n (execute re-checks per tile).
            const long long row_bytes = (long long)(n * elem);
            cudaStream_t st = static_cast<cudaStream_t>(stream);
            unsigned long long* dc = reinterpret_cast<unsigned long long*>(h->d_scratch + 4);
            for (int Rb = R; Rb >= 16; Rb /= 2) {
                const long long csr = (long long)te_buf_bytes(Rb + 8, capz_for(Rb), (int)elem, 0);
                const long long capb_try = ((RS_BSTAGE_SMEM / RS_STAGES - csr) / 16) * 16;
                if (capb_try < 16 * row_bytes) continue;
                unsigned long long cnt[2] = {0, 0};
                cudaError_t e = cudaMemsetAsync(dc, 0, sizeof(cnt), st);
                if (e == cudaSuccess) {
                    const long long tiles = (h->m + Rb - 1) / Rb;
                    const int grid = (int)std::min<long long>((tiles + WARPS_PER_CTA - 1) / WARPS_PER_CTA, 8LL * kNumSMs);
                    k_tile_span<<<std::max(grid, 1), THREADS, 0, st>>>(h->ro, h->col, h->m, Rb, row_bytes, capb_try, dc);
                    e = cudaGetLastError();
                }
                if (e == cudaSuccess) e = cudaMemcpyAsync(cnt, dc, sizeof(cnt), cudaMemcpyDeviceToHost, st);
                if (e == cudaSuccess) e = cudaStreamSynchronize(st);
                if (e != cudaSuccess) return cuda_fail(h, e, "plan: B span");
                const double frac = (double)cnt[0] / (double)h->nnz;
                h->bspan_compact = std::max(h->bspan_compact, frac);
                if (frac >= RS_BSTAGE_MIN) {
                    h->rows_per_tile = Rb;
                    h->capz = capz_for(Rb);
                    h->capb = (int)std::min<long long>(capb_try, (long long)((cnt[1] + 15) & ~15ULL));
                    break;
                }
            }
        }
        R = h->rows_per_tile;
        h->num_ctas = (h->m + R - 1) / R;
        // irregular (but not merge-skewed) row lengths: uneven tile costs, so the persistent CTAs take
        // row tiles from a queue (measured: lognormal d = 7.9 -14%; regular matrices keep the static
        // round robin, which the queue's extra latency slows)
        if (o.policy == SPMM_POLICY_AUTO && h->max_row < 0 && h->m > 0) {  // forced ROWSPLIT under AUTO policy
            const spmm_status ms = measure_max_row(h, stream);
            if (ms != SPMM_OK) return ms;
        }
        h->rs_dyn = o.policy == SPMM_POLICY_AUTO && h->max_row >= 0 &&
                    (double)h->max_row > RS_DYN_SKEW * std::max(1.0, d);
        if (h->rs_dyn) h->ws_bytes = 256;
    }
    h->opts = o;
    h->planned = true;
    if (workspace_bytes) *workspace_bytes = h->ws_bytes;
    if (chosen) *chosen = pick;
    return SPMM_OK;
}

spmm_status spmm_csr_plan(spmm_csr_t h, int32_t n, spmm_algo algo, spmm_semiring sr, double threshold, void* stream,
                          size_t* workspace_bytes, spmm_algo* chosen) {
    return spmm_csr_plan_ex(h, n, algo, sr, threshold, nullptr, stream, workspace_bytes, chosen);
}

spmm_status spmm_csr_get_plan_info(spmm_csr_t h, spmm_plan_info* out) {
    if (!h || !out) return SPMM_ERR_NULL_POINTER;
    if (!h->planned) return fail(h, SPMM_ERR_NOT_PLANNED, "not planned");
    std::memset(out, 0, sizeof(*out));
    out->m = h->m; out->k = h->k; out->nnz = h->nnz; out->n = h->n;
    out->chosen = h->chosen; out->semiring = h->sr; out->dtype = h->dtype;
    out->policy = h->opts.policy; out->partition = h->opts.partition;
    out->mean_row_length = h->m > 0 ? (double)h->nnz / (double)h->m : 0.0;
    out->max_row_length = h->max_row;
    out->threshold = h->threshold;
    out->num_ctas = (int32_t)h->num_ctas;
    out->items_per_cta = h->chosen == SPMM_ALGO_MERGE ? h->items : 0;
    const bool rsq = h->chosen == SPMM_ALGO_ROWSPLIT && h->rs_dyn;
    out->launches_per_execute = (h->m == 0) ? 0 : (h->chosen == SPMM_ALGO_MERGE ? 3 : (rsq ? 2 : 1));
    out->compute_launch = (h->chosen == SPMM_ALGO_MERGE || rsq) ? 1 : 0;
    out->b_staging = (h->chosen == SPMM_ALGO_ROWSPLIT && h->capb > 0) ? 1 : 0;
    out->rows_per_tile = (h->chosen == SPMM_ALGO_ROWSPLIT || h->chosen == SPMM_ALGO_TILED) ? h->rows_per_tile : 0;
    out->bspan_compact = h->bspan_compact;
    out->tasks_per_warp = h->chosen == SPMM_ALGO_MERGE ? h->opts.tasks_per_warp : 0;
    out->merge_worker_lanes = h->chosen == SPMM_ALGO_MERGE ? (h->mfold ? pick_fold(h->n, nullptr, h->n % 4 == 0 ? 4 : 1, nullptr, h->n % 4 == 0 ? 4 : 1).G : 32) : 0;
    out->workspace_bytes = h->ws_bytes;
    return SPMM_OK;
}

spmm_status spmm_csr_execute_ex(spmm_csr_t h, const void* B, int64_t ldb, void* C, int64_t ldc, int32_t n,
                                void* workspace, size_t workspace_bytes, const spmm_exec_opts* opts, void* stream) {
    NvtxRange nvtx_range("spmm_csr_execute");
    if (!h) return SPMM_ERR_NULL_POINTER;
    if (!h->planned) return fail(h, SPMM_ERR_NOT_PLANNED, "execute before plan");
    if (n != h->n) return fail(h, SPMM_ERR_INVALID_ARG, "n differs from the planned n");
    if (ldb < n || ldc < n) return fail(h, SPMM_ERR_INVALID_ARG, "ldb and ldc must be >= n");
    EpiParams epi{};
    if (opts) {
        for (int i = 0; i < 4; ++i)
            if (opts->reserved[i] != 0) return fail(h, SPMM_ERR_INVALID_ARG, "reserved exec option fields must be 0");
        if (opts->accumulate != 0 && opts->accumulate != 1) return fail(h, SPMM_ERR_INVALID_ARG, "accumulate must be 0 or 1");
        if (opts->num_peers < 0 || opts->num_peers > SPMM_MAX_PEERS)
            return fail(h, SPMM_ERR_INVALID_ARG, "num_peers must be in [0, 7]");
        if (opts->num_peers > 0) {
            if (opts->peer_ldc != ldc) return fail(h, SPMM_ERR_INVALID_ARG, "peer_ldc must equal ldc");
            if (opts->peer_row_offset < 0) return fail(h, SPMM_ERR_INVALID_ARG, "peer_row_offset must be >= 0");
            for (int i = 0; i < opts->num_peers; ++i) {
                if (!opts->peer_C[i]) return fail(h, SPMM_ERR_NULL_POINTER, "peer_C[i] is NULL");
                if (((uintptr_t)opts->peer_C[i] % 16) != 0) return fail(h, SPMM_ERR_INVALID_ARG, "peer_C must be 16-byte aligned");
            }
        }
        epi.accumulate = opts->accumulate;
        epi.npeers = opts->num_peers;
        epi.peer_row0 = opts->peer_row_offset;
        epi.peer_ldc = opts->peer_ldc;
        for (int i = 0; i < opts->num_peers; ++i) epi.peer[i] = opts->peer_C[i];
    }
    if (h->m == 0) return SPMM_OK;
    if (!C) return fail(h, SPMM_ERR_NULL_POINTER, "C is NULL");
    if (h->nnz > 0 && !B) return fail(h, SPMM_ERR_NULL_POINTER, "B is NULL");
    if (workspace_bytes < h->ws_bytes) return fail(h, SPMM_ERR_WORKSPACE_TOO_SMALL, "workspace too small");
    if (h->ws_bytes > 0 && !workspace) return fail(h, SPMM_ERR_NULL_POINTER, "workspace is NULL");
    if (h->ws_bytes > 0 && ((uintptr_t)workspace % 16) != 0)
        return fail(h, SPMM_ERR_INVALID_ARG, "workspace must be 16-byte aligned");
    if ((long long)h->m * ldc >= (1LL << 40) || (long long)h->k * ldb >= (1LL << 40) || ldb >= (1LL << 29))
        return fail(h, SPMM_ERR_UNSUPPORTED, "matrix too large");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    if (h->dtype == SPMM_F32) {
        e = (h->sr == SPMM_PLUS_TIMES) ? run<float, SR_PLUS_TIMES>(h, B, ldb, C, ldc, workspace, epi, st)
                                       : run<float, SR_MIN_PLUS>(h, B, ldb, C, ldc, workspace, epi, st);
    } else {
        e = (h->sr == SPMM_PLUS_TIMES) ? run<int, SR_PLUS_TIMES>(h, B, ldb, C, ldc, workspace, epi, st)
                                       : run<int, SR_MIN_PLUS>(h, B, ldb, C, ldc, workspace, epi, st);
    }
    if (e == cudaErrorNotSupported) return fail(h, SPMM_ERR_UNSUPPORTED, "no kernel instance for this n / alignment");
    if (e != cudaSuccess) return cuda_fail(h, e, "execute");
    return SPMM_OK;
}

spmm_status spmm_csr_execute(spmm_csr_t h, const void* B, int64_t ldb, void* C, int64_t ldc, int32_t n,
                             void* workspace, size_t workspace_bytes, void* stream) {
    return spmm_csr_execute_ex(h, B, ldb, C, ldc, n, workspace, workspace_bytes, nullptr, stream);
}

// ---- device buffers shareable across processes (CUDA IPC), for the peer copies of C (NEXT-1) ----
static_assert(sizeof(cudaIpcMemHandle_t) == SPMM_IPC_HANDLE_BYTES, "IPC handle size");
static_assert(SPMM_MAX_PEERS == EPI_MAX_PEERS, "peer count");
spmm_status spmm_ipc_alloc(size_t bytes, void** ptr, void* handle_out) {
    if (!ptr || !handle_out) return SPMM_ERR_NULL_POINTER;
    *ptr = nullptr;
    if (bytes == 0) return SPMM_ERR_INVALID_ARG;
    void* p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) return SPMM_ERR_CUDA;
    cudaIpcMemHandle_t hd;
    if (cudaIpcGetMemHandle(&hd, p) != cudaSuccess) {
        cudaFree(p);
        return SPMM_ERR_CUDA;
    }
    std::memcpy(handle_out, &hd, sizeof(hd));
    *ptr = p;
    return SPMM_OK;
}

spmm_status spmm_ipc_free(void* ptr) {
    if (!ptr) return SPMM_OK;
    return cudaFree(ptr) == cudaSuccess ? SPMM_OK : SPMM_ERR_CUDA;
}

spmm_status spmm_ipc_open(const void* handle, void** ptr) {
    if (!handle || !ptr) return SPMM_ERR_NULL_POINTER;
    *ptr = nullptr;
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, handle, sizeof(hd));
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        return SPMM_ERR_CUDA;
    }
    *ptr = p;
    return SPMM_OK;
}

spmm_status spmm_ipc_close(void* ptr) {
    if (!ptr) return SPMM_OK;
    return cudaIpcCloseMemHandle(ptr) == cudaSuccess ? SPMM_OK : SPMM_ERR_CUDA;
}

spmm_status spmm_csr_set_timing_events(spmm_csr_t h, void* const* events, int32_t count) {
    if (!h) return SPMM_ERR_NULL_POINTER;
    if (count < 0 || count > 8) return fail(h, SPMM_ERR_INVALID_ARG, "timing event count must be in [0, 8]");
    if (count > 0 && !events) return fail(h, SPMM_ERR_NULL_POINTER, "events is NULL");
    for (int i = 0; i < 8; ++i) h->ev[i] = (i < count) ? static_cast<cudaEvent_t>(events[i]) : nullptr;
    h->nev = count;
    return SPMM_OK;
}

spmm_status spmm_merge_partition(const int32_t* row_offsets, int64_t m, int64_t nnz, int32_t items_per_cta,
                                 int32_t partition, int64_t num_ctas, int32_t* states_out, void* stream) {
    if (!states_out || (m > 0 && !row_offsets)) return SPMM_ERR_NULL_POINTER;
    if (partition != SPMM_PARTITION_MERGE_PATH && partition != SPMM_PARTITION_NONZERO_SPLIT) return SPMM_ERR_INVALID_ARG;
    if (items_per_cta <= 0 || m < 0 || nnz < 0 || m + nnz >= 0x7fffffffLL) return SPMM_ERR_INVALID_ARG;
    if (num_ctas != spmm_merge_num_ctas(m, nnz, items_per_cta, partition)) return SPMM_ERR_INVALID_ARG;
    if (num_ctas == 0) return SPMM_OK;
    k_partition<<<partition_grid(m), THREADS, 0, static_cast<cudaStream_t>(stream)>>>(
        row_offsets, (int)m, (int)nnz, items_per_cta, partition, (int)num_ctas, states_out, nullptr);
    return cudaGetLastError() == cudaSuccess ? SPMM_OK : SPMM_ERR_CUDA;
}

// library-owned stream-ordered memory pool for spmm_csr_multiply_host (one per device, kept across
// calls: a release threshold of "never" so repeated calls reuse the same device memory)
static cudaMemPool_t host_api_pool() {
    static std::mutex mu;
    static cudaMemPool_t pools[8] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    cudaMemPool_t& p = pools[dev & 7];
    if (!p) {
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.handleTypes = cudaMemHandleTypeNone;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&p, &props) != cudaSuccess) { p = nullptr; return nullptr; }
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
        // never make a call on one stream wait for memory another stream is still using: the pool grows
        // to one buffer set per stream in flight instead, and calls on different streams overlap
        int no = 0;
        cudaMemPoolSetAttribute(p, cudaMemPoolReuseAllowInternalDependencies, &no);
    }
    return p;
}

spmm_status spmm_csr_multiply_host(int64_t m, int64_t k, int64_t nnz, const int32_t* h_ro, const int32_t* h_col,
                                   const void* h_val, spmm_dtype dtype, const void* h_B, int64_t ldb, void* h_C,
                                   int64_t ldc, int32_t n, spmm_algo algo, spmm_semiring sr, uint32_t flags,
                                   void* stream) {
    NvtxRange nvtx_range("spmm_csr_multiply_host");
    if (m < 0 || k < 0 || nnz < 0 || n < 1 || ldb < n || ldc < n) return SPMM_ERR_INVALID_ARG;
    if ((flags & ~SPMM_HOST_SYNC) != 0u) return SPMM_ERR_INVALID_ARG;
    if (dtype != SPMM_F32 && dtype != SPMM_I32) return SPMM_ERR_INVALID_ARG;
    if (m == 0) return SPMM_OK;
    if (!h_ro || !h_C || (nnz > 0 && (!h_col || !h_val || !h_B))) return SPMM_ERR_NULL_POINTER;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t e4 = 4;
    int32_t *d_ro = nullptr, *d_col = nullptr;
    void *d_val = nullptr, *d_B = nullptr, *d_C = nullptr, *d_ws = nullptr;
    spmm_csr_t h = nullptr;
    spmm_status rc = SPMM_OK;
    auto ok = [&](cudaError_t e) {
        if (e != cudaSuccess && rc == SPMM_OK) rc = SPMM_ERR_CUDA;
        return rc == SPMM_OK;
    };
    // stream-ordered device buffers from the library's pool (kept across calls: no device-wide sync)
    cudaMemPool_t pool = host_api_pool();
    if (!pool) return SPMM_ERR_CUDA;
    auto dalloc = [&](void** ptr, size_t bytes) { return cudaMallocFromPoolAsync(ptr, bytes, pool, st); };
    const size_t kk = (size_t)std::max<int64_t>(k, 1), zz = (size_t)std::max<int64_t>(nnz, 1);
    if (ok(dalloc(reinterpret_cast<void**>(&d_ro), e4 * (size_t)(m + 1))) &&
        ok(dalloc(reinterpret_cast<void**>(&d_col), e4 * zz)) && ok(dalloc(&d_val, e4 * zz)) &&
        ok(dalloc(&d_B, e4 * kk * (size_t)n)) && ok(dalloc(&d_C, e4 * (size_t)m * (size_t)n)) &&
        ok(cudaMemcpyAsync(d_ro, h_ro, e4 * (size_t)(m + 1), cudaMemcpyHostToDevice, st)) &&
        (nnz == 0 || (ok(cudaMemcpyAsync(d_col, h_col, e4 * (size_t)nnz, cudaMemcpyHostToDevice, st)) &&
                      ok(cudaMemcpyAsync(d_val, h_val, e4 * (size_t)nnz, cudaMemcpyHostToDevice, st)) &&
                      ok(ldb == n ? cudaMemcpyAsync(d_B, h_B, e4 * (size_t)k * (size_t)n, cudaMemcpyHostToDevice, st)
                                  : cudaMemcpy2DAsync(d_B, e4 * (size_t)n, h_B, e4 * (size_t)ldb, e4 * (size_t)n,
                                                      (size_t)k, cudaMemcpyHostToDevice, st))))) {
        rc = spmm_csr_create(&h, m, k, nnz, d_ro, d_col, d_val, dtype, 0u, stream);
        // the longest row from the host copy (while the copies above are in flight): plan then needs no
        // device reduction + read-back, so the call does not wait on this stream's copies
        if (rc == SPMM_OK) {
            int32_t mx = 0;
            for (int64_t i = 0; i < m; ++i) mx = std::max(mx, h_ro[i + 1] - h_ro[i]);
            h->hint_max_row = mx;
        }
        size_t ws = 0;
        spmm_algo chosen;
        if (rc == SPMM_OK) rc = spmm_csr_plan(h, n, algo, sr, 0.0, stream, &ws, &chosen);
        if (rc == SPMM_OK && ws > 0) ok(dalloc(&d_ws, ws));
        if (rc == SPMM_OK) rc = spmm_csr_execute(h, d_B, n, d_C, n, n, d_ws, ws, stream);
        if (rc == SPMM_OK)  // columns [0, n) of C only: the host C's padding columns stay untouched
            ok(ldc == n ? cudaMemcpyAsync(h_C, d_C, e4 * (size_t)m * (size_t)n, cudaMemcpyDeviceToHost, st)
                        : cudaMemcpy2DAsync(h_C, e4 * (size_t)ldc, d_C, e4 * (size_t)n, e4 * (size_t)n, (size_t)m,
                                            cudaMemcpyDeviceToHost, st));
        if (h) spmm_csr_destroy(h);
    }
    for (void* p : {static_cast<void*>(d_ro), static_cast<void*>(d_col), d_val, d_B, d_C, d_ws})
        if (p) cudaFreeAsync(p, st);
    if (rc == SPMM_OK && (flags & SPMM_HOST_SYNC)) ok(cudaStreamSynchronize(st));
    return rc;
}

spmm_status spmm_partition_rows(const int32_t* host_row_offsets, int64_t m, int32_t parts, int32_t mode,
                                int64_t* row_bounds) {
    if (!row_bounds || (m > 0 && !host_row_offsets)) return SPMM_ERR_NULL_POINTER;
    if (parts < 1 || m < 0 || (mode != 0 && mode != 1)) return SPMM_ERR_INVALID_ARG;
    const int64_t nnz = m > 0 ? host_row_offsets[m] : 0;
    row_bounds[0] = 0;
    for (int p = 1; p < parts; ++p) {
        int64_t b;
        if (mode == 0) {
            // nnz-balanced: first row r with ro[r] >= p*nnz/parts (lower_bound)
            const long double target = (long double)nnz * p / parts;
            int64_t lo = 0, hi = m;
            while (lo < hi) {
                const int64_t mid = (lo + hi) / 2;
                if ((long double)host_row_offsets[mid] < target) lo = mid + 1; else hi = mid;
            }
            b = lo;
        } else {
            // merge-path balanced: row coordinate of diagonal D = p*(m+nnz)/parts
            const int64_t D = (int64_t)((long double)(m + nnz) * p / parts);
            int64_t lo = std::max<int64_t>(0, D - nnz), hi = std::min<int64_t>(D, m);
            while (lo < hi) {
                const int64_t mid = (lo + hi) / 2;
                if ((int64_t)host_row_offsets[mid + 1] <= D - mid - 1) lo = mid + 1; else hi = mid;
            }
            b = lo;
        }
        row_bounds[p] = std::max(b, row_bounds[p - 1]);
    }
    row_bounds[parts] = m;
    for (int p = 1; p < parts; ++p) row_bounds[p] = std::min(row_bounds[p], m);
    return SPMM_OK;
}

}  // extern "C"
