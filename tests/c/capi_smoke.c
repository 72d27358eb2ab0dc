/* Plain-C client of include/split3.h (no Python, no torch): the boundary as a C user sees it.
 *   capi_smoke cpu   -> only host-side checks (no GPU needed): status strings, sizes, errors
 *   capi_smoke gpu   -> full call sequence on device 0: create, workspace, sgemm (3/4/1 terms),
 *                       host-buffer entry, destroy; C must equal the exact integer product. */
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "split3.h"

#define CHECK(cond, msg)                                   \
    do {                                                   \
        if (!(cond)) {                                     \
            fprintf(stderr, "FAIL: %s (line %d)\n", msg, __LINE__); \
            return 1;                                      \
        }                                                  \
    } while (0)

static int cpu_checks(void) {
    CHECK(strcmp(split3_status_string(SPLIT3_OK), "SPLIT3_OK") == 0, "status string");
    CHECK(split3_sgemm_workspace_size(100, 60, 33, 0) > 0, "workspace size");
    CHECK(split3_sgemm(NULL, 1, 1, 1, NULL, 1, NULL, 1, NULL, 1, 0) == SPLIT3_ERR_INVALID_VALUE, "null handle");
    CHECK(split3_sgemm_destroy(NULL) == SPLIT3_OK, "destroy NULL");
    CHECK(split3_set_fold(NULL, 1) == SPLIT3_ERR_INVALID_VALUE, "fold NULL handle");
    CHECK(split3_set_fused_split_a(NULL, 1, 0) == SPLIT3_ERR_INVALID_VALUE, "fused A NULL handle");
    CHECK(split3_last_path(NULL) == 0, "path NULL handle");
    printf("cpu ok\n");
    return 0;
}

static int gpu_checks(void) {
    const int64_t M = 300, N = 200, K = 1000;
    split3_handle_t h = NULL;
    int st = split3_sgemm_create(&h, 0, NULL);
    CHECK(st == SPLIT3_OK, split3_status_string(st));
    float *hA = malloc(M * K * 4), *hB = malloc(K * N * 4), *hC = malloc(M * N * 4);
    double *ref = calloc(M * N, sizeof(double));
    srand(7);
    for (int64_t i = 0; i < M * K; i++) hA[i] = (float)(rand() % 5 - 2);
    for (int64_t i = 0; i < K * N; i++) hB[i] = (float)(rand() % 5 - 2);
    for (int64_t i = 0; i < M; i++)
        for (int64_t k = 0; k < K; k++)
            for (int64_t j = 0; j < N; j++) ref[i * N + j] += (double)hA[i * K + k] * hB[k * N + j];
    float *A, *B, *C;
    void* ws;
    size_t wsb = split3_sgemm_host_workspace_size(M, N, K, SPLIT3_FOUR_TERM);
    CHECK(cudaMalloc((void**)&A, M * K * 4) == cudaSuccess && cudaMalloc((void**)&B, K * N * 4) == cudaSuccess &&
          cudaMalloc((void**)&C, M * N * 4) == cudaSuccess && cudaMalloc(&ws, wsb) == cudaSuccess, "cudaMalloc");
    cudaMemcpy(A, hA, M * K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, K * N * 4, cudaMemcpyHostToDevice);
    CHECK(split3_sgemm(h, M, N, K, A, K, B, N, C, N, 0) == SPLIT3_ERR_WORKSPACE, "workspace missing");
    CHECK(split3_sgemm_set_workspace(h, ws, wsb) == SPLIT3_OK, "set workspace");
    const uint32_t flags[3] = {SPLIT3_THREE_TERM, SPLIT3_FOUR_TERM, SPLIT3_ONE_TERM};
    for (int f = 0; f < 3; f++) {
        CHECK(split3_sgemm(h, M, N, K, A, K, B, N, C, N, flags[f]) == SPLIT3_OK, "sgemm");
        CHECK(cudaMemcpy(hC, C, M * N * 4, cudaMemcpyDeviceToHost) == cudaSuccess, "copy back");
        for (int64_t i = 0; i < M * N; i++) CHECK((double)hC[i] == ref[i], "integer product exact");
    }
    /* round-2 knobs: the folded accumulator (every 3-/4-term call) and fused A (C = (B^T A^T)^T):
       integer inputs stay exact whatever the path */
    CHECK(split3_set_fold(h, 3) == SPLIT3_ERR_INVALID_VALUE && split3_set_fold(h, 2) == SPLIT3_OK, "fold mode");
    CHECK(split3_set_fused_split_a(h, 2, 0) == SPLIT3_OK, "fused A mode");
    for (int f = 0; f < 2; f++) {
        CHECK(split3_sgemm(h, M, N, K, A, K, B, N, C, N, flags[f]) == SPLIT3_OK, "sgemm (fold, fused A)");
        CHECK((split3_last_path(h) & (SPLIT3_PATH_FOLD | SPLIT3_PATH_FUSED_A)) ==
                  (f == 0 ? (SPLIT3_PATH_FOLD | SPLIT3_PATH_FUSED_A) : SPLIT3_PATH_FOLD), "path bits");
        CHECK(cudaMemcpy(hC, C, M * N * 4, cudaMemcpyDeviceToHost) == cudaSuccess, "copy back");
        for (int64_t i = 0; i < M * N; i++) CHECK((double)hC[i] == ref[i], "integer product exact (fold)");
    }
    CHECK(split3_set_fold(h, 1) == SPLIT3_OK && split3_set_fused_split_a(h, 0, 0) == SPLIT3_OK, "defaults");
    memset(hC, 0, M * N * 4);
    CHECK(split3_sgemm_host(h, M, N, K, hA, hB, hC, 0) == SPLIT3_OK, "host entry");
    for (int64_t i = 0; i < M * N; i++) CHECK((double)hC[i] == ref[i], "host entry exact");
    CHECK(split3_sgemm(h, M, N, K, A, K - 1, B, N, C, N, 0) == SPLIT3_ERR_INVALID_VALUE, "lda < K");
    CHECK(split3_sgemm_destroy(h) == SPLIT3_OK, "destroy");
    cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(ws);
    free(hA); free(hB); free(hC); free(ref);
    printf("gpu ok\n");
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && strcmp(argv[1], "gpu") == 0) return gpu_checks();
    return cpu_checks();
}
