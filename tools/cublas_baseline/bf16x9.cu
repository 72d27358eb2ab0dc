// Same-box baseline (context, not product): cuBLAS 12.9 SGEMM, its BF16x9 FP32 emulation
// (CUBLAS_COMPUTE_32F_EMULATED_16BFX9) and TF32, on N x N uniform[-1,1] inputs.  Built against the
// toolkit's libcublas (torch bundles 12.8, which lacks the emulated compute type), so it runs as a
// separate process.  Prints one JSON line per variant: sustained TFLOP/s (2N^3/t over ~secs
// seconds) and the error vs an fp64 dot product on sampled outputs (E64rel over the sample).
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

__host__ __device__ inline float uni(uint64_t seed, uint64_t i) {   // splitmix64 -> [-1, 1)
    uint64_t z = seed + 0x9E3779B97F4A7C15ull * (i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (float)((double)(z >> 40) * (1.0 / 16777216.0) * 2.0 - 1.0);
}
__global__ void fill(float* x, int64_t n, uint64_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        x[i] = uni(seed, i);
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 16384;
    const double secs = argc > 2 ? atof(argv[2]) : 3.0;
    const int64_t nn = (int64_t)n * n;
    float *A, *B, *C;
    cudaMalloc(&A, nn * 4); cudaMalloc(&B, nn * 4); cudaMalloc(&C, nn * 4);
    fill<<<4096, 256>>>(A, nn, 1); fill<<<4096, 256>>>(B, nn, 2);
    cublasHandle_t h;
    cublasCreate(&h);
    struct V { const char* name; cublasComputeType_t ct; } vs[] = {
        {"cuBLAS BF16x9 emulated FP32 (CUBLAS_COMPUTE_32F_EMULATED_16BFX9)", CUBLAS_COMPUTE_32F_EMULATED_16BFX9},
        {"cuBLAS SGEMM (CUBLAS_COMPUTE_32F)", CUBLAS_COMPUTE_32F},
        {"cuBLAS TF32 (CUBLAS_COMPUTE_32F_FAST_TF32)", CUBLAS_COMPUTE_32F_FAST_TF32}};
    const float one = 1.f, zero = 0.f;
    // row-major C = A B  <=>  column-major C^T = B^T A^T
    for (auto& v : vs) {
        auto run = [&]() {
            return cublasGemmEx(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, B, CUDA_R_32F, n, A, CUDA_R_32F, n, &zero, C,
                                CUDA_R_32F, n, v.ct, CUBLAS_GEMM_DEFAULT);
        };
        cublasStatus_t st = run();
        cudaDeviceSynchronize();
        if (st != CUBLAS_STATUS_SUCCESS) { printf("{\"impl\": \"%s\", \"error\": %d}\n", v.name, (int)st); continue; }
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0); run(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float one_ms; cudaEventElapsedTime(&one_ms, e0, e1);
        int reps = (int)(secs * 1000.0 / one_ms); if (reps < 3) reps = 3;
        cudaEventRecord(e0);
        for (int r = 0; r < reps; r++) run();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= reps;
        // accuracy on 48 x 48 sampled outputs vs fp64 dot products
        const int R = 48;
        std::vector<float> row(n), col(n), out((size_t)n);
        double num = 0, den = 0;
        std::vector<float> hA((size_t)n), hB((size_t)n * R);
        for (int a = 0; a < R; a++) {
            int i = (int)((int64_t)a * 7919 % n);
            cudaMemcpy(out.data(), C + (int64_t)i * n, (size_t)n * 4, cudaMemcpyDeviceToHost);
            for (int k = 0; k < n; k++) row[k] = uni(1, (int64_t)i * n + k);
            for (int b = 0; b < R; b++) {
                int j = (int)((int64_t)b * 104729 % n);
                double ref = 0;
                for (int k = 0; k < n; k++) ref += (double)row[k] * (double)uni(2, (int64_t)k * n + j);
                num += (out[j] - ref) * (out[j] - ref);
                den += ref * ref;
            }
        }
        printf("{\"impl\": \"%s\", \"n\": %d, \"ms\": %.4f, \"tflops\": %.2f, \"reps\": %d, \"E64rel_sampled\": %.3e}\n",
               v.name, n, ms, 2.0 * n * (double)n * n / (ms / 1e3) / 1e12, reps, sqrt(num / den));
        fflush(stdout);
    }
    cublasDestroy(h);
    return 0;
}
