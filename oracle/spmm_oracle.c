/*
 * oracle/spmm_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the CSR SpMM hot path of
 * Yang, Buluc, Owens, "Design Principles for Sparse Matrix Multiplication on the GPU" (arXiv 1803.08601).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it.
 * It shares no code, header, table or helper with the CUDA path (paper_1803_08601_b200/csrc/).
 *
 * What is computed (§1): "Given an m-by-k sparse matrix A and a k-by-n dense matrix B,
 * SpMM computes an m-by-n dense matrix C = AB."  A is CSR (§2.2: row offsets, column
 * indices, values); B and C are row-major.  Both of the paper's kernels
 * (row split §4.1, merge-based Alg. 1 §4.2) reach exactly this result up to the order of the fp32
 * sums, so the oracle is the definition written out:
 *
 *     for i in [0,m): for j in [0,n):
 *         acc = 0(semiring)
 *         for p in [ro[i], ro[i+1]):  acc = acc (+) values[p] (x) B[col[p]*ldb + j]
 *         C[i*n + j] = acc
 *
 * Semirings (GraphBLAS GrB_mxm framing):
 *   f32 plus-times : products and sums in fp64 (each fp32*fp32 product is exact in fp64), plus the
 *                    elementwise error scale bound_ij = sum |a|*|b| used by the 1e-5 tolerance.
 *   i32 plus-times : uint32 arithmetic, i.e. two's-complement wrap mod 2^32 (order independent).
 *   f32 min-plus   : acc = fminf(acc, a + b) with the add done in fp32 (one rounding), identity +inf.
 *   i32 min-plus   : acc = min(acc, (int32)(uint32)a + (uint32)b), identity INT32_MAX.
 * Partition oracles (Alg. 1 line 2 "PartitionSpmm"; §4(2a)/(2b)):
 *   merge_path_walk : brute-force sequential walk of the merge path of row-end offsets against
 *                     nonzero indices (Merrill-Garland, Fig. 2(c)), rows first on ties.
 *   nonzero_split   : Baxter's 1-D split: start row of block c = largest r with
 *                     ro[r] <= c*G, found by linear scan, with row_0 = 0
 *                     (SURVEY.md §8(c) ambiguity 20b).
 *
 * Rows are independent, so the OpenMP loop over rows gives bit-identical output for any thread count.
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared (no -ffast-math: fp order preserved).
 */
#include <stdint.h>
#include <stddef.h>
#include <math.h>

#define ORACLE_API __attribute__((visibility("default")))

static inline int64_t row_of(const int64_t* rows, int64_t r) { return rows ? rows[r] : r; }

/* f32 plus-times: C (fp64) and bound (fp64), both nrows x n.  rows == NULL -> all m rows. */
ORACLE_API int oracle_spmm_f32_plus_times(int64_t m, int64_t k, int64_t n,
                                          const int32_t* ro, const int32_t* col, const float* val,
                                          const float* B, int64_t ldb,
                                          const int64_t* rows, int64_t nrows,
                                          double* C, double* bound) {
    if (!rows) nrows = m;
    (void)k;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = row_of(rows, r);
        for (int64_t j = 0; j < n; ++j) {
            double acc = 0.0, bnd = 0.0;
            for (int64_t p = ro[i]; p < ro[i + 1]; ++p) {
                double a = (double)val[p];
                double b = (double)B[(int64_t)col[p] * ldb + j];
                acc += a * b;
                bnd += fabs(a) * fabs(b);
            }
            C[r * n + j] = acc;
            bound[r * n + j] = bnd;
        }
    }
    return 0;
}

/* i32 plus-times with wrap-around (mod 2^32). */
ORACLE_API int oracle_spmm_i32_plus_times(int64_t m, int64_t k, int64_t n,
                                          const int32_t* ro, const int32_t* col, const int32_t* val,
                                          const int32_t* B, int64_t ldb,
                                          const int64_t* rows, int64_t nrows, int32_t* C) {
    if (!rows) nrows = m;
    (void)k;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = row_of(rows, r);
        for (int64_t j = 0; j < n; ++j) {
            uint32_t acc = 0u;
            for (int64_t p = ro[i]; p < ro[i + 1]; ++p) {
                uint32_t a = (uint32_t)val[p];
                uint32_t b = (uint32_t)B[(int64_t)col[p] * ldb + j];
                acc += a * b;
            }
            C[r * n + j] = (int32_t)acc;
        }
    }
    return 0;
}

/* f32 min-plus: acc = min(acc, a + b), identity +inf; the add is one fp32 rounding. */
ORACLE_API int oracle_spmm_f32_min_plus(int64_t m, int64_t k, int64_t n,
                                        const int32_t* ro, const int32_t* col, const float* val,
                                        const float* B, int64_t ldb,
                                        const int64_t* rows, int64_t nrows, float* C) {
    if (!rows) nrows = m;
    (void)k;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = row_of(rows, r);
        for (int64_t j = 0; j < n; ++j) {
            float acc = INFINITY;
            for (int64_t p = ro[i]; p < ro[i + 1]; ++p) {
                volatile float s = val[p] + B[(int64_t)col[p] * ldb + j];
                acc = fminf(acc, s);
            }
            C[r * n + j] = acc;
        }
    }
    return 0;
}

/* i32 min-plus: acc = min(acc, a + b) with the add wrapping mod 2^32, identity INT32_MAX. */
ORACLE_API int oracle_spmm_i32_min_plus(int64_t m, int64_t k, int64_t n,
                                        const int32_t* ro, const int32_t* col, const int32_t* val,
                                        const int32_t* B, int64_t ldb,
                                        const int64_t* rows, int64_t nrows, int32_t* C) {
    if (!rows) nrows = m;
    (void)k;
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = row_of(rows, r);
        for (int64_t j = 0; j < n; ++j) {
            int32_t acc = INT32_MAX;
            for (int64_t p = ro[i]; p < ro[i + 1]; ++p) {
                int32_t s = (int32_t)((uint32_t)val[p] + (uint32_t)B[(int64_t)col[p] * ldb + j]);
                if (s < acc) acc = s;
            }
            C[r * n + j] = acc;
        }
    }
    return 0;
}

/*
 * Brute-force merge-path walk (§4(2b), Fig. 2(c); Merrill & Garland [14]).
 * The path merges the list of row-end offsets ro[1..m] with the list of nonzero indices 0..nnz-1.
 * From state (i, j) -- i row ends and j nonzeros consumed -- the next item is the row end of row i
 * if i < m and ro[i+1] <= j (rows first on ties), otherwise nonzero j.
 * diags[] must be ascending, each in [0, m+nnz]; out_i/out_j receive the state after diags[t] items.
 */
ORACLE_API int oracle_merge_path_walk(const int32_t* ro, int64_t m, int64_t nnz,
                                      const int64_t* diags, int64_t nd, int64_t* out_i, int64_t* out_j) {
    int64_t i = 0, j = 0, steps = 0, t = 0;
    while (t < nd) {
        if (diags[t] < steps || diags[t] > m + nnz) return 1;
        while (steps < diags[t]) {
            if (i < m && (int64_t)ro[i + 1] <= j) ++i;
            else ++j;
            ++steps;
        }
        out_i[t] = i;
        out_j[t] = j;
        ++t;
    }
    return 0;
}

/*
 * Baxter's nonzero split (§4(2a)): block c covers nonzeros [c*G, min((c+1)*G, nnz));
 * its start row is the largest r with ro[r] <= c*G (linear scan), except block 0 which
 * starts at row 0 so that leading empty rows are covered (SURVEY.md §8(c) ambiguity 20b).
 * out_rows has nblocks entries.
 */
ORACLE_API int oracle_nonzero_split(const int32_t* ro, int64_t m, int64_t G, int64_t nblocks, int64_t* out_rows) {
    for (int64_t c = 0; c < nblocks; ++c) {
        if (c == 0) { out_rows[c] = 0; continue; }
        int64_t target = c * G, r = 0;
        for (int64_t q = 0; q <= m; ++q)
            if ((int64_t)ro[q] <= target) r = q;
        out_rows[c] = r;
    }
    return 0;
}
