/* abi_smoke.c -- a plain C program that uses libspmm.so only through include/spmm.h (no Python, no
 * torch): C = A*B for a permutation matrix A (one nonzero per row, so the result is exact in fp32 and
 * must equal P*B bit for bit -- a closed form) plus one empty row (semiring identity),
 * through AUTO, ROWSPLIT and MERGE, fp32 plus-times and int32 min-plus.  Exit code 0 = pass.
 * Build: gcc -std=c11 -I include -I $CUDA/include tests/c/abi_smoke.c -L paper_1803_08601_b200 -lspmm
 *        -L $CUDA/lib64 -lcudart -Wl,-rpath,... */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "spmm.h"

#define M 1000
#define K 1200
#define N 64

static int fail(const char* what, int code) {
    fprintf(stderr, "abi_smoke: %s (%d)\n", what, code);
    return 1;
}

int main(void) {
    int32_t ro[M + 1], col[M];
    float valf[M];
    int32_t vali[M];
    int nnz = 0;
    ro[0] = 0;
    for (int i = 0; i < M; ++i) {
        if (i != 500) {  /* row 500 is empty */
            col[nnz] = (int32_t)((i * 7 + 3) % K);
            valf[nnz] = (float)((i % 5) - 2);  /* small integers: exact products */
            vali[nnz] = (i % 9) + 1;
            ++nnz;
        }
        ro[i + 1] = nnz;
    }
    float* Bf = malloc(sizeof(float) * K * N);
    int32_t* Bi = malloc(sizeof(int32_t) * K * N);
    for (int r = 0; r < K; ++r)
        for (int j = 0; j < N; ++j) {
            Bf[r * N + j] = (float)((r * 31 + j * 17) % 101) * 0.25f;
            Bi[r * N + j] = (r * 13 + j * 7) % 1000;
        }
    int32_t *dro, *dcol;
    void *dval, *dB, *dC, *ws = NULL;
    if (cudaMalloc((void**)&dro, sizeof(ro)) || cudaMalloc((void**)&dcol, sizeof(col)) ||
        cudaMalloc(&dval, sizeof(valf)) || cudaMalloc(&dB, sizeof(float) * K * N) || cudaMalloc(&dC, sizeof(float) * M * N))
        return fail("cudaMalloc", 0);
    cudaMemcpy(dro, ro, sizeof(ro), cudaMemcpyHostToDevice);
    cudaMemcpy(dcol, col, sizeof(col), cudaMemcpyHostToDevice);
    float* Cf = malloc(sizeof(float) * M * N);
    int32_t* Ci = malloc(sizeof(int32_t) * M * N);
    if (spmm_abi_version() != SPMM_ABI_VERSION) return fail("ABI version mismatch", spmm_abi_version());
    for (int kind = 0; kind < 2; ++kind) {
        const spmm_dtype dt = kind == 0 ? SPMM_F32 : SPMM_I32;
        const spmm_semiring sr = kind == 0 ? SPMM_PLUS_TIMES : SPMM_MIN_PLUS;
        cudaMemcpy(dval, kind == 0 ? (void*)valf : (void*)vali, sizeof(valf), cudaMemcpyHostToDevice);
        cudaMemcpy(dB, kind == 0 ? (void*)Bf : (void*)Bi, sizeof(float) * K * N, cudaMemcpyHostToDevice);
        spmm_csr_t h = NULL;
        spmm_status st = spmm_csr_create(&h, M, K, nnz, dro, dcol, dval, dt, SPMM_FLAG_VALIDATE, NULL);
        if (st != SPMM_OK) return fail(spmm_status_string(st), st);
        const spmm_algo algos[3] = {SPMM_ALGO_AUTO, SPMM_ALGO_ROWSPLIT, SPMM_ALGO_MERGE};
        for (int a = 0; a < 3; ++a) {
            size_t wsb = 0;
            spmm_algo chosen;
            st = spmm_csr_plan(h, N, algos[a], sr, 0.0, NULL, &wsb, &chosen);
            if (st != SPMM_OK) return fail(spmm_csr_last_error(h), st);
            if (ws) cudaFree(ws);
            ws = NULL;
            if (wsb && cudaMalloc(&ws, wsb)) return fail("workspace", (int)wsb);
            cudaMemset(dC, 0xff, sizeof(float) * M * N);  /* poison */
            st = spmm_csr_execute(h, dB, N, dC, N, N, ws, wsb, NULL);
            if (st != SPMM_OK) return fail(spmm_csr_last_error(h), st);
            if (cudaDeviceSynchronize() != cudaSuccess) return fail("kernel fault", a);
            cudaMemcpy(kind == 0 ? (void*)Cf : (void*)Ci, dC, sizeof(float) * M * N, cudaMemcpyDeviceToHost);
            for (int i = 0; i < M; ++i) {
                const int p = ro[i];
                const int empty = ro[i + 1] == p;
                for (int j = 0; j < N; ++j) {
                    if (kind == 0) {
                        const float want = empty ? 0.0f : 0.0f + valf[p] * Bf[col[p] * N + j];  /* 0 + (-0) = +0 */
                        if (memcmp(&Cf[i * N + j], &want, 4) != 0)
                            return fail("fp32 plus-times mismatch", i * N + j);
                    } else {
                        const int32_t want = empty ? INT32_MAX : vali[p] + Bi[col[p] * N + j];
                        if (Ci[i * N + j] != want) return fail("int32 min-plus mismatch", i * N + j);
                    }
                }
            }
        }
        /* errors come back as status codes */
        if (spmm_csr_execute(h, dB, N, dC, N, N + 1, ws, 0, NULL) != SPMM_ERR_INVALID_ARG) return fail("bad n accepted", 0);
        spmm_csr_destroy(h);
    }
    printf("abi_smoke ok\n");
    return 0;
}
