/*
 * spmm.h -- C ABI of libspmm.so: CSR sparse x tall-skinny row-major dense SpMM on B200 (sm_100a).
 *
 * The operation (§1, arXiv 1803.08601): "Given an m-by-k sparse matrix A and a k-by-n
 * dense matrix B, SpMM computes an m-by-n dense matrix C = AB", A in CSR (§2.2: row
 * offsets, column indices, values -- used as given, no format conversion), B and C
 * dense row-major (Fig. 3 caption :107), n small (tall-skinny B).
 * Generalised to the semirings plus-times and min-plus (GraphBLAS GrB_mxm framing).
 *
 * Two kernels and a selector:
 *   SPMM_ALGO_ROWSPLIT  row splitting, §4.1 (Fig. 3, Table 1)
 *   SPMM_ALGO_MERGE     merge-based, §4.2 Algorithm 1: PartitionSpmm (line 2),
 *                       per-CTA compute with carry-out (lines 3-23), FixCarryOut (line 24)
 *   SPMM_ALGO_AUTO      §5.4 heuristic: policy PAPER = merge iff mean row length d = nnz/m < threshold
 *                       (default 9.35); policy AUTO = B200 refit, see spmm_plan_opts.
 *
 * Conventions (all entry points):
 *   - Every pointer named row_offsets / col_indices / values / B / C / workspace is a DEVICE pointer
 *     (cudaMalloc / torch CUDA memory) unless its name starts with host_.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Indices are int32 (m, k, nnz < 2^31); sizes are int64 for ABI stability.
 *   - Errors are returned as spmm_status; no C++ exception crosses the ABI.  Kernel launch errors are
 *     reported by the call that launched (SPMM_ERR_CUDA); asynchronous device faults surface at the
 *     caller's next synchronisation of `stream`.
 *   - Thread safety: a handle may be used from several host threads / streams concurrently only for
 *     execute() with distinct workspaces; create/plan/destroy must not race with other calls on it.
 */
#ifndef SPMM_B200_H
#define SPMM_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SPMM_API __attribute__((visibility("default")))
#else
#define SPMM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ABI history: 2 = round 1; 3 = row pairing removed (the plan option field is reserved), merge
 * items are per warp task, spmm_plan_info.compute_launch added, row split under the AUTO policy may
 * need a 256-byte workspace (tile queue) -- callers must size the workspace from plan(); 4 = plan
 * option merge_worker (was reserved0), plan option tasks_per_warp (was reserved[0]) and
 * spmm_plan_info.merge_worker_lanes / tasks_per_warp (lane-folded merge, task queue),
 * spmm_csr_execute_ex (accumulate, peer copies of C) and the spmm_ipc_* buffers, SPMM_ALGO_TILED,
 * spmm_csr_multiply_host (host buffers). */
#define SPMM_ABI_VERSION 4

typedef struct spmm_csr_s* spmm_csr_t;

typedef enum {
    SPMM_OK = 0,
    SPMM_ERR_NULL_POINTER = 1,        /* a required pointer argument is NULL                        */
    SPMM_ERR_INVALID_ARG = 2,         /* bad size / leading dimension / enum / n != planned n        */
    SPMM_ERR_INVALID_CSR = 3,         /* SPMM_FLAG_VALIDATE found a broken CSR invariant             */
    SPMM_ERR_NOT_PLANNED = 4,         /* execute() before a successful plan()                        */
    SPMM_ERR_WORKSPACE_TOO_SMALL = 5, /* workspace_bytes < the size plan() reported                 */
    SPMM_ERR_UNSUPPORTED = 6,         /* n > 128, or a configuration this build does not implement  */
    SPMM_ERR_CUDA = 7                 /* a CUDA runtime call or kernel launch failed                */
} spmm_status;

/* TILED (NEXT-4): A/B tiling for dense-ish rows -- needs n % 4 == 0, 32 <= n <= 128
 * and column indices non-decreasing within rows (checked at plan: UNSUPPORTED otherwise). */
typedef enum { SPMM_ALGO_AUTO = 0, SPMM_ALGO_ROWSPLIT = 1, SPMM_ALGO_MERGE = 2, SPMM_ALGO_TILED = 3 } spmm_algo;
typedef enum { SPMM_F32 = 0, SPMM_I32 = 1 } spmm_dtype;                /* dtype of values, B and C */
typedef enum { SPMM_PLUS_TIMES = 0, SPMM_MIN_PLUS = 1 } spmm_semiring;
enum { SPMM_FLAG_VALIDATE = 1u };                                       /* one checking pass at create */

typedef enum { SPMM_POLICY_AUTO = 0, SPMM_POLICY_PAPER = 1 } spmm_policy;
typedef enum { SPMM_PARTITION_MERGE_PATH = 0, SPMM_PARTITION_NONZERO_SPLIT = 1 } spmm_partition;
typedef enum { SPMM_MERGE_WORKER_AUTO = 0, SPMM_MERGE_WORKER_WARP = 1, SPMM_MERGE_WORKER_FOLDED = 2 } spmm_merge_worker;

/* Optional planner knobs (spmm_csr_plan_ex).  Zero-initialised = defaults. */
typedef struct {
    int32_t policy;          /* spmm_policy.  PAPER: merge iff d < threshold.
                                AUTO (default): B200 refit of §5.4 -- merge iff the row
                                lengths are skewed (max row > 16 d and >= 1024), there are too few
                                rows to fill the row-split kernel (m < 2 x resident row groups, with
                                nnz >= 2^20), or
                                the rows are too long to stage a 16-row tile (1.2 x 16 d > 8192),
                                or (round-2 refit) mildly skewed rows (max row > 16 d, >= 256) with
                                n >= 16, or very short rows with wide B (d < 3 and n >= 32);
                                costs one O(m) device reduction + stream sync at plan time.  */
    int32_t partition;       /* spmm_partition for the merge kernel: 2-D merge path over (row ends,
                                nonzeros) (default) or the paper's 1-D nonzero split
                                (PAPER.md:80, :89).                                                  */
    int32_t items_per_cta;   /* merge-path items (rows + nonzeros) per merge task, the partition
                                granularity of Alg. 1 line 2; 0 = sized at plan time (256..2048, about
                                16 tasks per resident worker).  Must be a multiple of 32 in [32, 8192]. */
    int32_t merge_worker;    /* spmm_merge_worker: who walks a merge task.  AUTO (0): lane-folded slots
                                for n <= 16, else a whole warp.  WARP (1): a whole warp with lanes
                                over B's columns (k_merge_w).  FOLDED (2): the warp split into 32/G
                                slots of G lanes (G x VEC >= n), each walking its own piece of the
                                task's merge path (k_merge_f); n <= 16 only (else
                                plan returns UNSUPPORTED).                                             */
    int32_t tasks_per_warp;  /* merge: tasks per resident warp when items_per_cta is 0.  0 = default;
                                1 = one task per warp, walked in a static order; k > 1 = k tasks per
                                warp taken from a queue in the workspace (zeroed by the partition
                                kernel) so warps that finish early take more.  At most 64.          */
    int32_t reserved[3];     /* must be zero */
} spmm_plan_opts;

/* Read-only description of the current plan (spmm_csr_get_plan_info). */
typedef struct {
    int64_t m, k, nnz;
    int32_t n;
    int32_t chosen;          /* spmm_algo actually used by execute (ROWSPLIT or MERGE) */
    int32_t semiring, dtype, policy, partition;
    double mean_row_length;  /* d = nnz/m */
    int64_t max_row_length;  /* -1 unless computed (AUTO policy) */
    double threshold;
    int32_t num_ctas;        /* row split: row tiles; merge: merge-path tasks */
    int32_t items_per_cta;   /* merge only: items per task */
    int32_t launches_per_execute;  /* operations one execute() enqueues: merge 3 (partition, compute,
                                      fix-up); row split 1, or 2 when its tile queue is reset first */
    int32_t compute_launch;  /* 0-based index of the compute kernel among them (timing events i..i+1) */
    size_t workspace_bytes;
    int32_t b_staging;       /* 1 if the row-split kernel stages compact B row spans in shared memory
                                (TMA); measured at plan time, applied per tile at execute when B and
                                ldb allow 16-byte aligned rows                          */
    int32_t rows_per_tile;   /* row split: rows per tile                                               */
    double bspan_compact;    /* fraction of nonzeros in tiles whose B span is compact (-1: not measured) */
    int32_t merge_worker_lanes; /* merge: lanes per merge worker (32 = whole warp, G < 32 = lane-folded
                                   slots, with 16-byte aligned B / C); 0 for row split              */
    int32_t tasks_per_warp;  /* merge: tasks per resident warp the plan sized (> 1: taken from a queue) */
} spmm_plan_info;

/*
 * spmm_csr_create -- record a CSR matrix A (m x k, nnz stored entries).  a0 in SURVEY.md §8(a).
 *   row_offsets[m+1], col_indices[nnz], values[nnz]: device arrays, BORROWED (never copied or
 *   converted); they must stay valid and unmodified until spmm_csr_destroy.
 *   values has the element type `dtype` (float or int32).  Column indices need not be sorted or
 *   unique within a row (duplicates are summed in storage order).
 *   flags: SPMM_FLAG_VALIDATE runs one synchronous device pass checking row_offsets[0] == 0,
 *   non-decreasing offsets, row_offsets[m] == nnz and 0 <= col < k (else SPMM_ERR_INVALID_CSR).
 *   Without it the CSR is trusted.  m == 0 or nnz == 0 is allowed (pointers may then be NULL
 *   except row_offsets when m > 0).  k == 0 requires nnz == 0.
 *   The three arrays may be views at any 4-byte offset (e.g. a row block of a larger CSR): the kernels
 *   stage them with TMA by address, reading at most to the enclosing 16-byte granules.
 *   *out receives a new handle (owned by the caller, free with spmm_csr_destroy).
 */
SPMM_API spmm_status spmm_csr_create(spmm_csr_t* out, int64_t m, int64_t k, int64_t nnz,
                            const int32_t* row_offsets, const int32_t* col_indices, const void* values,
                            spmm_dtype dtype, uint32_t flags, void* stream);

/*
 * spmm_csr_plan -- choose the kernel for B with n columns (1 <= n <= 128) and size the workspace.
 *   algo_or_auto: force ROWSPLIT / MERGE, or AUTO (§5.4 heuristic).
 *   threshold <= 0 -> 9.35.  *workspace_bytes receives the device workspace size
 *   execute() needs (row split: 0, or 256 bytes for its tile queue when AUTO finds irregular row lengths);
 *   *chosen receives ROWSPLIT or MERGE.  Either out pointer may
 *   be NULL.  Plan enqueues small measurement kernels on `stream` and synchronises it: the maximum
 *   row length (AUTO policy) and, for the row-split kernel with n * 4 >= 256 bytes, the compactness
 *   of the row tiles' B spans (B staging, see spmm_plan_info.b_staging).  Plan once, execute often.
 */
SPMM_API spmm_status spmm_csr_plan(spmm_csr_t h, int32_t n, spmm_algo algo_or_auto, spmm_semiring sr,
                          double threshold, void* stream, size_t* workspace_bytes, spmm_algo* chosen);

/* spmm_csr_plan with explicit planner options (opts may be NULL = defaults). */
SPMM_API spmm_status spmm_csr_plan_ex(spmm_csr_t h, int32_t n, spmm_algo algo_or_auto, spmm_semiring sr,
                             double threshold, const spmm_plan_opts* opts, void* stream,
                             size_t* workspace_bytes, spmm_algo* chosen);

/*
 * spmm_csr_execute -- C = A (x) B over the planned semiring, enqueued on `stream`, no host sync,
 * no allocation.
 *   B: device, k rows x ldb (row-major, element = dtype); only columns [0, n) are read, and only
 *      rows named by col_indices.  C: device, m rows x ldc; columns [0, n) of every row are
 *      OVERWRITTEN (no alpha/beta: the paper computes C = AB); columns [n, ldc) are
 *      untouched.  Empty rows receive the semiring identity (0, +inf or INT32_MAX).
 *   Requires ldb >= n, ldc >= n, n == planned n.  B and C must not overlap.  16-byte aligned B/C
 *   with ldb/ldc multiples of 4 take the float4 path; anything else takes a narrower vector or
 *   scalar path with bit-identical results for int32 / min-plus.
 *   workspace: device buffer of at least the planned workspace_bytes (may be NULL if 0), 16-byte
 *   aligned, caller-owned, not shared by concurrent executes.
 */
SPMM_API spmm_status spmm_csr_execute(spmm_csr_t h, const void* B, int64_t ldb, void* C, int64_t ldc, int32_t n,
                             void* workspace, size_t workspace_bytes, void* stream);

/* Optional epilogue of execute (spmm_csr_execute_ex).  Zero-initialised = plain execute. */
#define SPMM_MAX_PEERS 7
typedef struct {
    int32_t accumulate;       /* 0: C = A (x) B (overwrite).  1: C = C (+) A (x) B -- rows of C are read
                                 and combined with the product (plus-times: +, min-plus: min); empty
                                 rows of A leave C unchanged.  Used by the iterative distributed SpMM
                                 (dist.IterativeRowBlockSpmm: diagonal block first, then the
                                 off-diagonal block accumulated).           */
    int32_t num_peers;        /* 0..SPMM_MAX_PEERS: every finished row of C is ALSO stored, with the same
                                 value, into each peer_C[i] at row (row + peer_row_offset) -- the
                                 all-gather of C fused into the SpMM (NEXT-1).  peer_C are device
                                 pointers valid on this device (CUDA IPC / P2P mappings of other
                                 GPUs' full C, e.g. from spmm_ipc_open), 16-byte aligned, with
                                 peer_ldc == ldc.  The peer copies are complete when this execute's
                                 stream work has completed; the caller orders that with the peers
                                 (e.g. stream sync + process-group barrier).                        */
    int64_t peer_row_offset;  /* first global row of this C block in the peer Cs (>= 0)              */
    int64_t peer_ldc;         /* leading dimension of the peer Cs (must equal ldc)                   */
    void* peer_C[SPMM_MAX_PEERS];
    int32_t reserved[4];      /* must be zero                                                        */
} spmm_exec_opts;

/*
 * spmm_csr_execute_ex -- spmm_csr_execute with the epilogue options above (opts may be NULL).
 * Errors: INVALID_ARG for accumulate not in {0,1}, num_peers outside [0, 7], peer_ldc != ldc,
 * negative peer_row_offset, misaligned peer pointers or non-zero reserved fields; NULL_POINTER for a
 * NULL peer pointer; otherwise as spmm_csr_execute.
 */
SPMM_API spmm_status spmm_csr_execute_ex(spmm_csr_t h, const void* B, int64_t ldb, void* C, int64_t ldc, int32_t n,
                                         void* workspace, size_t workspace_bytes, const spmm_exec_opts* opts,
                                         void* stream);

/*
 * CUDA IPC buffers for the peer copies of C (NEXT-1).  The handle is SPMM_IPC_HANDLE_BYTES opaque
 * bytes (a cudaIpcMemHandle_t) that another process on the same node passes to spmm_ipc_open.
 *   spmm_ipc_alloc: cudaMalloc `bytes` on the current device (*ptr) and export its handle.
 *   spmm_ipc_free:  free a buffer from spmm_ipc_alloc (after every peer closed it).
 *   spmm_ipc_open:  map another process's buffer into this one (*ptr, peer access enabled lazily);
 *                   fails (SPMM_ERR_CUDA) for a handle exported by the calling process itself.
 *   spmm_ipc_close: unmap a pointer from spmm_ipc_open.
 */
/*
 * spmm_csr_multiply_host -- one-shot C = A (x) B on HOST buffers (the whole path behind one call):
 * stream-ordered device buffers from a library-owned memory pool per device (kept across calls, so
 * repeated calls reuse the memory and never synchronise the device), host->device copies of the CSR arrays and of columns [0, n) of B, create + plan
 * (the given algo / semiring, AUTO policy) + execute, device->host copy of columns [0, n) of C (the
 * host C's columns [n, ldc) are untouched), buffers released on the stream.  Host arrays: row_offsets
 * [m+1], col_indices / values [nnz], B k x ldb, C m x ldc, row-major, 4-byte elements; pinned (page-
 * locked) memory makes the copies asynchronous.  Plan synchronises `stream` once (the AUTO reduction);
 * flags: SPMM_HOST_SYNC (1) also synchronises before return -- otherwise C is valid once `stream`
 * completes, and the host arrays must stay valid until then.  Errors as create / plan / execute, plus
 * SPMM_ERR_CUDA for a failed allocation or copy.
 */
enum { SPMM_HOST_SYNC = 1u };
SPMM_API spmm_status spmm_csr_multiply_host(int64_t m, int64_t k, int64_t nnz, const int32_t* row_offsets,
                                            const int32_t* col_indices, const void* values, spmm_dtype dtype,
                                            const void* B, int64_t ldb, void* C, int64_t ldc, int32_t n,
                                            spmm_algo algo, spmm_semiring semiring, uint32_t flags, void* stream);

/*
 * spmm_csr_split_columns -- set-up for the iterative distributed SpMM (NEXT-3): split every row of
 * A (m x ?, CSR, device) into the entries whose column lies in [c0, c1) and the others, keeping
 * each row's storage order.  Outputs (device, caller-allocated): ro_in[m+1], col_in / val_in (>= nnz
 * entries; columns rebased to col - c0) and ro_out[m+1], col_out / val_out (>= nnz entries; global
 * columns).  *nnz_in (host) receives the number of in-range entries (the rest, nnz - *nnz_in, are
 * in the "out" part).  Synchronises `stream` (one 4-byte read-back).  Values are copied bit for
 * bit (dtype only names their 4-byte type).  Errors: INVALID_ARG for c1 < c0 or sizes >= 2^31,
 * NULL_POINTER for missing arrays, CUDA on a runtime error.
 */
SPMM_API spmm_status spmm_csr_split_columns(const int32_t* row_offsets, const int32_t* col_indices, const void* values,
                                            int64_t m, int64_t nnz, int32_t c0, int32_t c1, spmm_dtype dtype,
                                            int32_t* ro_in, int32_t* col_in, void* val_in, int32_t* ro_out,
                                            int32_t* col_out, void* val_out, int64_t* nnz_in, void* stream);

#define SPMM_IPC_HANDLE_BYTES 64
SPMM_API spmm_status spmm_ipc_alloc(size_t bytes, void** ptr, void* handle_out);
SPMM_API spmm_status spmm_ipc_free(void* ptr);
SPMM_API spmm_status spmm_ipc_open(const void* handle, void** ptr);
SPMM_API spmm_status spmm_ipc_close(void* ptr);

/* spmm_csr_destroy -- free the handle (not the borrowed CSR arrays).  NULL is a no-op. */
SPMM_API spmm_status spmm_csr_destroy(spmm_csr_t h);

/* Fill *out with the current plan (SPMM_ERR_NOT_PLANNED before plan). */
SPMM_API spmm_status spmm_csr_get_plan_info(spmm_csr_t h, spmm_plan_info* out);

/*
 * spmm_csr_set_timing_events -- diagnostic: if count > 0, every later execute() records
 * events[0] (cudaEvent_t) on its stream before its first kernel and events[i+1] after its i-th
 * kernel (i < count-1), so the caller can time each kernel of the path separately (the bench's
 * roofline uses the dominant kernel's own duration).  count == 0 disables.  The events are borrowed.
 */
SPMM_API spmm_status spmm_csr_set_timing_events(spmm_csr_t h, void* const* events, int32_t count);

/* Static strings; never NULL. */
SPMM_API const char* spmm_status_string(spmm_status s);
SPMM_API const char* spmm_csr_last_error(spmm_csr_t h);   /* per-handle detail message of the last failure */
SPMM_API int32_t spmm_abi_version(void);

/*
 * spmm_merge_partition -- the merge kernel's phase 1 (Alg. 1 line 2 "PartitionSpmm")
 * on its own, exported for verification.  For each c in [0, num_ctas] writes the merge-path state
 * (row, nonzero) at which CTA c starts (c == num_ctas: the end state (m, nnz)):
 *   partition == MERGE_PATH: state on diagonal min(c*items_per_cta, m+nnz) of the merge of row-end
 *       offsets with nonzero indices, rows first on ties (Fig. 2(c));
 *   partition == NONZERO_SPLIT: (largest r with row_offsets[r] <= c*items_per_cta, c*items_per_cta),
 *       row 0 for c == 0 (SURVEY.md §8(c) ambiguity 20b).
 * num_ctas must equal spmm_merge_num_ctas(m, nnz, items_per_cta, partition).
 * row_offsets: device int32[m+1]; states_out: device int32[2*(num_ctas+1)] as (row, nz) pairs.
 */
SPMM_API int64_t spmm_merge_num_ctas(int64_t m, int64_t nnz, int32_t items_per_cta, int32_t partition);
SPMM_API spmm_status spmm_merge_partition(const int32_t* row_offsets, int64_t m, int64_t nnz, int32_t items_per_cta,
                                 int32_t partition, int64_t num_ctas, int32_t* states_out, void* stream);

/*
 * spmm_partition_rows -- host-side 1-D row-block partition for multi-GPU SpMM (north_star;
 * SURVEY.md §8(e)).  host_row_offsets: HOST int32[m+1].  Writes parts+1 row bounds (int64, host):
 * bounds[0] = 0, bounds[parts] = m, non-decreasing; part p owns rows [bounds[p], bounds[p+1]).
 *   mode 0: nnz-balanced, bounds[p] = first row r with row_offsets[r] >= p*nnz/parts (lower_bound);
 *   mode 1: merge-path balanced, bounds[p] = row coordinate of diagonal p*(m+nnz)/parts.
 * A row is never split across parts.
 */
SPMM_API spmm_status spmm_partition_rows(const int32_t* host_row_offsets, int64_t m, int32_t parts, int32_t mode,
                                int64_t* row_bounds);

#ifdef __cplusplus
}
#endif
#endif /* SPMM_B200_H */
