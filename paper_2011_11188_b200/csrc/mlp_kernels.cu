// mlp_kernels.cu — the non-GEMM steps of a dense-network training step.
//
// PAPER.md:301 (§3.2 closing): "the form of operations in DNN are theoretically able to well
// approximate operations of fp32 using mixed-precision operations in fp16".  The GEMMs of the
// step run through split3_sgemm_ex (3 FP16 products); everything here stays FP32 (SPEC.md's
// ledger: bias, activations and softmax/cross-entropy never in fp16).  All kernels are
// HBM-bound elementwise / row / column passes; results are deterministic (fixed reduction
// orders, no floating-point atomics except the fp64 loss sum, which is reduced per block first
// and then added in block order by a second pass).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"

namespace split3 {
namespace {

// H = act(Z + b), b broadcast over rows.  act: 0 identity, 1 ReLU.  Work item = (row, 1024-column
// segment): one 64-bit division per 1024 elements; float4 when Z, H, b allow it.
__global__ void __launch_bounds__(256) bias_act_kernel(int64_t M, int64_t N, const float* __restrict__ Z,
                                                       int64_t ldz, const float* __restrict__ b,
                                                       float* __restrict__ H, int64_t ldh, int relu) {
    const int64_t nseg = (N + 1023) / 1024, items = M * nseg;
    const bool vec = (N % 4 == 0) && (ldz % 4 == 0) && (ldh % 4 == 0) &&
                     ((reinterpret_cast<uintptr_t>(Z) | reinterpret_cast<uintptr_t>(H) |
                       reinterpret_cast<uintptr_t>(b)) & 15u) == 0;
    auto act = [&](float z, float bb) {
        const float v = __fadd_rn(z, bb);
        return relu ? (v > 0.0f ? v : 0.0f) : v;
    };
    for (int64_t w = blockIdx.x; w < items; w += gridDim.x) {
        const int64_t r = w / nseg, c = (w - r * nseg) * 1024 + 4 * threadIdx.x;
        if (c >= N) continue;
        const float* z = Z + r * ldz + c;
        float* h = H + r * ldh + c;
        if (vec) {
            const float4 zv = *reinterpret_cast<const float4*>(z);
            const float4 bv = b ? *reinterpret_cast<const float4*>(b + c) : make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4*>(h) = make_float4(act(zv.x, bv.x), act(zv.y, bv.y), act(zv.z, bv.z), act(zv.w, bv.w));
        } else {
            for (int j = 0; j < 4 && c + j < N; j++) h[j] = act(z[j], b ? b[c + j] : 0.0f);
        }
    }
}

// dZ = dH * 1[H > 0]   (ReLU backward through its output); float4 when all three are aligned
__global__ void __launch_bounds__(256) relu_bwd_kernel(int64_t M, int64_t N, const float* __restrict__ dH,
                                                       const float* __restrict__ H, float* __restrict__ dZ) {
    const int64_t total = M * N;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool vec = ((reinterpret_cast<uintptr_t>(dH) | reinterpret_cast<uintptr_t>(H) |
                       reinterpret_cast<uintptr_t>(dZ)) & 15u) == 0;
    int64_t done = 0;
    if (vec) {
        const int64_t n4 = total / 4;
        for (int64_t i = t0; i < n4; i += stride) {
            const float4 d = reinterpret_cast<const float4*>(dH)[i], h = reinterpret_cast<const float4*>(H)[i];
            reinterpret_cast<float4*>(dZ)[i] = make_float4(h.x > 0.0f ? d.x : 0.0f, h.y > 0.0f ? d.y : 0.0f,
                                                           h.z > 0.0f ? d.z : 0.0f, h.w > 0.0f ? d.w : 0.0f);
        }
        done = n4 * 4;
    }
    for (int64_t i = done + t0; i < total; i += stride) dZ[i] = H[i] > 0.0f ? dH[i] : 0.0f;
}

// Row-wise softmax cross-entropy: one warp per row.  P = softmax(L) (max-subtracted),
// dL = (P - onehot(label)) / M, row_loss[r] = -log P[r, label] in fp64.
__global__ void __launch_bounds__(256) softmax_xent_kernel(int64_t M, int64_t N, const float* __restrict__ L,
                                                           const int32_t* __restrict__ labels,
                                                           float* __restrict__ P, float* __restrict__ dL,
                                                           double* __restrict__ row_loss) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (row >= M) return;
    const float* l = L + row * N;
    float mx = -INFINITY;
    for (int64_t c = lane; c < N; c += 32) mx = fmaxf(mx, l[c]);
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double s = 0.0;
    for (int64_t c = lane; c < N; c += 32) s += (double)expf(l[c] - mx);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const int32_t y = labels ? labels[row] : -1;
    const float inv_m = 1.0f / (float)M;
    for (int64_t c = lane; c < N; c += 32) {
        const float p = (float)((double)expf(l[c] - mx) / s);
        if (P) P[row * N + c] = p;
        if (dL) dL[row * N + c] = (p - (c == y ? 1.0f : 0.0f)) * inv_m;
    }
    if (lane == 0 && row_loss) row_loss[row] = (y >= 0) ? -((double)(l[y] - mx) - log(s)) : 0.0;
}

// db[c] = sum_r dZ[r, c] in a fixed order (deterministic): a block (1024 threads) owns 32 columns;
// warp g sums the rows r = g, g + 32, g + 64, ... in increasing order (lane = column: 128-B
// coalesced loads), then the 32 group sums are added in group order.
__global__ void __launch_bounds__(1024) col_sum_kernel(int64_t M, int64_t N, const float* __restrict__ dZ,
                                                       float* __restrict__ db) {
    __shared__ float part[32][33];
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    for (int64_t c0 = (int64_t)blockIdx.x * 32; c0 < N; c0 += (int64_t)gridDim.x * 32) {
        const int64_t c = c0 + lane;
        float acc = 0.0f;
        if (c < N) {
#pragma unroll 4
            for (int64_t r = g; r < M; r += 32) acc = __fadd_rn(acc, dZ[r * N + c]);
        }
        part[g][lane] = acc;
        __syncthreads();
        if (g == 0 && c < N) {
            float t = part[0][lane];
            for (int k = 1; k < 32; k++) t = __fadd_rn(t, part[k][lane]);
            db[c] = t;
        }
        __syncthreads();
    }
}

// Two-stage form for tall dZ (scratch available): stage 1 — block (column tile x, row chunk y)
// sums rows [y*rows_per, (y+1)*rows_per) of 32 columns as 8 interleaved groups (row order inside a
// group, groups in order) into part[y][c]; stage 2 — db[c] = part[0][c] + part[1][c] + ... in
// chunk order.  Fixed order throughout (deterministic), ~1 load per thread per 8 rows in flight.
__global__ void __launch_bounds__(256) col_sum_part_kernel(int64_t M, int64_t N, const float* __restrict__ dZ,
                                                           int64_t rows_per, float* __restrict__ part) {
    __shared__ float sp[8][33];
    const int lane = threadIdx.x & 31, g = threadIdx.x >> 5;
    const int64_t c = (int64_t)blockIdx.x * 32 + lane;
    const int64_t r0 = (int64_t)blockIdx.y * rows_per;
    const int64_t r1 = r0 + rows_per < M ? r0 + rows_per : M;
    float acc = 0.0f;
    if (c < N) {
#pragma unroll 4
        for (int64_t r = r0 + g; r < r1; r += 8) acc = __fadd_rn(acc, dZ[r * N + c]);
    }
    sp[g][lane] = acc;
    __syncthreads();
    if (g == 0 && c < N) {
        float t = sp[0][lane];
        for (int k = 1; k < 8; k++) t = __fadd_rn(t, sp[k][lane]);
        part[(int64_t)blockIdx.y * N + c] = t;
    }
}
__global__ void __launch_bounds__(256) col_sum_fold_kernel(int64_t N, int chunks, const float* __restrict__ part,
                                                           float* __restrict__ db) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < N; c += (int64_t)gridDim.x * blockDim.x) {
        float t = part[c];
        for (int k = 1; k < chunks; k++) t = __fadd_rn(t, part[(int64_t)k * N + c]);
        db[c] = t;
    }
}

// sum of n doubles in index order (single block, fixed tree): out[0] = sum
__global__ void __launch_bounds__(256) sum_f64_kernel(int64_t n, const double* __restrict__ x, double* out) {
    __shared__ double sh[256];
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += x[i];
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = sh[0];
}

// w -= lr * g
__global__ void __launch_bounds__(256) sgd_kernel(int64_t n, float* __restrict__ w, const float* __restrict__ g,
                                                  float lr) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        w[i] = __fmaf_rn(-lr, g[i], w[i]);
}

inline unsigned grid_for(int64_t work, int num_sms) {
    int64_t g = (work + 255) / 256;
    const int64_t cap = (int64_t)num_sms * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

inline int ok() { return cudaPeekAtLastError() == cudaSuccess ? 1 : -1; }

}  // namespace

int launch_bias_act(cudaStream_t st, int64_t M, int64_t N, const float* Z, int64_t ldz, const float* b, float* H,
                    int64_t ldh, int relu, int num_sms) {
    bias_act_kernel<<<grid_for(M * ((N + 1023) / 1024) * 256, num_sms), 256, 0, st>>>(M, N, Z, ldz, b, H, ldh, relu);
    return ok();
}
int launch_relu_bwd(cudaStream_t st, int64_t M, int64_t N, const float* dH, const float* H, float* dZ, int num_sms) {
    relu_bwd_kernel<<<grid_for((M * N + 3) / 4, num_sms), 256, 0, st>>>(M, N, dH, H, dZ);
    return ok();
}
int launch_softmax_xent(cudaStream_t st, int64_t M, int64_t N, const float* L, const int32_t* labels, float* P,
                        float* dL, double* row_loss, double* loss_sum) {
    const unsigned g = (unsigned)((M + 7) / 8);
    softmax_xent_kernel<<<g, 256, 0, st>>>(M, N, L, labels, P, dL, row_loss);
    if (ok() < 0) return -1;
    if (row_loss && loss_sum) {
        sum_f64_kernel<<<1, 256, 0, st>>>(M, row_loss, loss_sum);
        if (ok() < 0) return -1;
        return 2;
    }
    return 1;
}
int launch_col_sum(cudaStream_t st, int64_t M, int64_t N, const float* dZ, float* db, int num_sms, float* scratch,
                   size_t scratch_bytes) {
    // chunk count from M only (never from the device), so the summation order is fixed
    const int64_t ctiles = (N + 31) / 32;
    int chunks = (int)((M + 255) / 256);   // 256-row chunks, at most 64
    if (chunks > 64) chunks = 64;
    if (chunks >= 2 && ctiles <= 65535 * 64 && scratch && (size_t)chunks * (size_t)N * 4 <= scratch_bytes) {
        const int64_t rows_per = (M + chunks - 1) / chunks;
        col_sum_part_kernel<<<dim3((unsigned)ctiles, (unsigned)chunks), 256, 0, st>>>(M, N, dZ, rows_per, scratch);
        col_sum_fold_kernel<<<grid_for(N, num_sms), 256, 0, st>>>(N, chunks, scratch, db);
        return ok() < 0 ? -1 : 2;
    }
    const int64_t tiles = (N + 31) / 32, cap = (int64_t)num_sms * 8;
    col_sum_kernel<<<(unsigned)(tiles < cap ? tiles : cap), 1024, 0, st>>>(M, N, dZ, db);
    return ok();
}
int launch_sgd(cudaStream_t st, int64_t n, float* w, const float* g, float lr, int num_sms) {
    sgd_kernel<<<grid_for(n, num_sms), 256, 0, st>>>(n, w, g, lr);
    return ok();
}

}  // namespace split3
