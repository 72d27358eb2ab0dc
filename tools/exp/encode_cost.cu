// time cuTensorMapEncodeTiled and an empty cudaLaunchKernelEx on the host (experiment only)
#include <cuda.h>
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
__global__ void empty_k(int) {}
int main() {
    void* p; cudaMalloc(&p, 1 << 24);
    cudaStream_t st; cudaStreamCreate(&st);
    CUtensorMap m;
    cuuint64_t dims[2] = {4096, 4096}; cuuint64_t strides[1] = {8192}; cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
    const int R = 20000;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < R; i++)
        cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    auto t1 = std::chrono::steady_clock::now();
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(148); cfg.blockDim = dim3(256); cfg.stream = st;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization; at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    for (int i = 0; i < 100; i++) cudaLaunchKernelEx(&cfg, empty_k, i);
    cudaStreamSynchronize(st);
    auto t2 = std::chrono::steady_clock::now();
    for (int i = 0; i < R; i++) { cudaLaunchKernelEx(&cfg, empty_k, i); if ((i & 1023) == 0) cudaStreamSynchronize(st); }
    auto t3 = std::chrono::steady_clock::now();
    cudaStreamCaptureStatus cs;
    for (int i = 0; i < R; i++) cudaStreamIsCapturing(st, &cs);
    auto t4 = std::chrono::steady_clock::now();
    int d; for (int i = 0; i < R; i++) cudaGetDevice(&d);
    auto t5 = std::chrono::steady_clock::now();
    auto us = [&](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count() / R; };
    printf("encode %.3f us, launchEx(PDL) %.3f us, isCapturing %.3f us, getDevice %.3f us\n", us(t0, t1), us(t2, t3), us(t3, t4), us(t4, t5));
    return 0;
}
