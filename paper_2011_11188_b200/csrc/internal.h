// internal.h — declarations shared by the CUDA translation units of libsplit3.so.
// Not part of the public ABI (that is include/split3.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace split3 {

// ---- programmatic dependent launch ------------------------------------------------------
// Every kernel of the split3_sgemm path is launched with programmatic stream serialization:
// it may be scheduled while its predecessor in the stream drains, runs its prologue, and waits
// in griddepcontrol.wait (full completion + memory flush of the predecessor) before its first
// global-memory access.  Hides the launch gap between the 4-5 kernels of a call.
#ifndef SPLIT3_PDL
#define SPLIT3_PDL 1
#endif
__device__ __forceinline__ void pdl_wait() {
#if SPLIT3_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger() {
#if SPLIT3_PDL
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
// wait for the predecessor, then let the successor be scheduled (small kernels)
__device__ __forceinline__ void pdl_enter() {
    pdl_wait();
    pdl_trigger();
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = SPLIT3_PDL ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...);
}
// cooperative (all blocks co-resident: the kernel has a grid-wide barrier) + programmatic
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k_coop(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                 Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = SPLIT3_PDL ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...);
}

// Padded plane leading dimension: a multiple of 8 elements (16 bytes, the TMA stride unit).
inline int64_t plane_ld(int64_t k) { return ((k + 7) / 8) * 8; }

// ---- split_kernels.cu ------------------------------------------------------------------
// Each launcher returns the number of kernels it launched (>= 0) or -1 on a launch error.
// One-launch front end for small problems (both operands fp32, plain splits): max-abs of both,
// a grid-wide barrier (cooperative launch), then both non-transposing splits.  `sync` points to
// 2 zeroed words (arrival count, sense flag) left reusable; partials holds >= 2 * grid words.
struct PrepOperand {
    const float* X;
    int64_t rows, cols, ld;     // the STORED matrix
    uint16_t *hi, *lo;
    int64_t ldp;
    float* d_max;
    int32_t* d_sexp;
};
constexpr int64_t kPrepMaxElems = 4 << 20;   // both operands together; larger: separate kernels
int launch_prep2(cudaStream_t s, const PrepOperand& a, const PrepOperand& b, unsigned* partials,
                 unsigned* sync, int num_sms);

int launch_maxabs(cudaStream_t s, int64_t rows, int64_t cols, const float* X, int64_t ld,
                  float* d_max, long long* d_bad, int num_sms);
// max-abs of two matrices in one launch (no bad-index tracking): block partials (<= max_parts
// per matrix) + the last block's reduction write *d_max0 / *d_max1 directly (no reset needed;
// `ticket` must be 0 before the first use and is left 0).  Strided or misaligned operands fall
// back to two atomic launches after resetting *d_max0 / *d_max1.
int launch_maxabs2(cudaStream_t s, int64_t rows0, int64_t cols0, const float* X0, int64_t ld0, float* d_max0,
                   int64_t rows1, int64_t cols1, const float* X1, int64_t ld1, float* d_max1, int num_sms,
                   float* partials, int max_parts, unsigned* ticket);
// host-buffer pipeline: max |x| and min nonzero |x| (uint bits) of a contiguous chunk,
// and the per-matrix scale check over the row blocks (see split_kernels.cu)
int launch_maxmin(cudaStream_t s, int64_t n, const float* X, unsigned* d_max, unsigned* d_min, int num_sms);
int launch_maxmin2d(cudaStream_t s, int64_t rows, int64_t cols, const float* X, int64_t ld, unsigned* d_max,
                    unsigned* d_min, int num_sms);   // strided region (ld >= cols)
int launch_host_scale_check(cudaStream_t s, const unsigned* maxblk, const unsigned* minblk, const int32_t* sblk,
                            int nblk, float* d_max, int32_t* d_sexp, int32_t* flags);
int launch_split(cudaStream_t s, int64_t rows, int64_t cols, const float* X, int64_t ld,
                 const float* d_max, uint16_t* hi, uint16_t* lo, int64_t ldp, int32_t* d_sexp,
                 int num_sms);
// bf16 x 3 planes (no scale); transpose as for launch_split_t
int launch_split_bf16x3(cudaStream_t s, int64_t rows, int64_t cols, const float* X, int64_t ld, uint16_t* p1,
                        uint16_t* p2, uint16_t* p3, int64_t ldp, int transpose, int num_sms);
int launch_split_t(cudaStream_t s, int64_t rows, int64_t cols, const float* X, int64_t ld,
                   const float* d_max, uint16_t* hi, uint16_t* lo, int64_t ldp, int32_t* d_sexp,
                   int num_sms);

// ---- gemm3.cu --------------------------------------------------------------------------
// D_hi promotion period in 64-wide k-blocks (4 MMAs each) when the handle sets none
// (DESIGN.md §3 R9: measured truncating accumulation, promote every 8 MMAs).
constexpr int kDefaultPromoKb = 2;

// GEMM scheduling knobs (results never depend on them).
constexpr int kDefaultGroupM = 8;     // raster group, in pair m-blocks
struct GemmTuneIn {
    int group_m = 0;                  // 0 = default
    int pol_a = 0, pol_b = 0;         // L2 policy for A / B plane loads: 0 normal, 1 evict_first, 2 evict_last
};
struct GemmTune {
    int group_m;
    uint64_t pol_a, pol_b;
};

// Work split of the persistent GEMM: `whole` tiles run over the full K; the last `nsplit` tiles
// (all tiles of a problem with fewer tiles than CTA pairs, else the tail wave) are cut into
// `slices` K slices whose partials are reduced in a fixed order (deterministic).
struct SplitPlan {
    int64_t whole;
    int64_t nsplit;
    int slices;
};
SplitPlan gemm3_split_plan(int64_t M, int64_t N, int64_t K, int terms, int num_sms, int promo_kb, bool fold = false);
// debug build (SPLIT3_DEBUG=1): read / reset the GEMM's check record, inject a fault; release
// builds return 0 (not available), -1 on a CUDA error, 1 on success
int gemm3_debug_init();   // map the host record (handle creation)
int gemm3_debug_read(unsigned long long* out8, int reset);
int gemm3_debug_fault(int fault);
int64_t gemm3_partial_elems(const SplitPlan& p, int terms, bool fold = false);
bool gemm3_fold_chosen(int64_t M, int64_t N, int64_t K, int terms, int fold);   // the handle's fold mode   // floats of partial workspace

// terms: 1, 3, 4, or 6 (= bf16 x 3: planes A1..A3, B1t..B3t, 6 products, no scale).
// mn bit 0: the B planes are MN-major, K x N row-major with leading dimension ldpb >= N (the
// plain split of a row-major K x N B), else K-major N x K with ldpb >= K; bit 1: the A planes
// are MN-major, K x M with ldpa >= M (the plain split of a stored K x M A^T), else M x K.  `partial` (may be NULL: no split-K) holds partial_elems floats.
// Fused B (terms == 3 only): Bf != NULL is the fp32 B itself (mn bit 0: K x N
// row-major, else stored N x K; ldb % 4 == 0, 16-B aligned) and d_maxB its max-abs; the GEMM splits
// it in shared memory (B1t/B2t are ignored) and writes the scale exponent to d_sB.
// c_trans != 0: C (ldc) is the caller's N x M matrix and receives the TRANSPOSE of this M x N
// product (the fused-A form C_caller = (B^T A^T)^T); C must be 16-B aligned with ldc % 4 == 0.
// Returns kernels launched (1, or 2 with the split-K reduction) or -1 (*err set to a status).
int launch_gemm3(cudaStream_t s, int64_t M, int64_t N, int64_t K,
                 const uint16_t* A1, const uint16_t* A2, int64_t ldpa, const int32_t* d_sA,
                 const uint16_t* B1t, const uint16_t* B2t, int64_t ldpb, const int32_t* d_sB,
                 float* C, int64_t ldc, int terms, int num_sms, int promo_kb,
                 unsigned* wave_counter, const GemmTuneIn& tune, float* partial, int64_t partial_elems,
                 int* err, const uint16_t* A3 = nullptr, const uint16_t* B3t = nullptr, int mn = 0,
                 const float* Bf = nullptr, int64_t ldb = 0, const float* d_maxB = nullptr, int c_trans = 0,
                 int fold = 0);

// ---- mlp_kernels.cu (NEXT #3: the non-GEMM steps of a dense-network training step) --------
int launch_bias_act(cudaStream_t s, int64_t M, int64_t N, const float* Z, int64_t ldz, const float* b, float* H,
                    int64_t ldh, int relu, int num_sms);
int launch_relu_bwd(cudaStream_t s, int64_t M, int64_t N, const float* dH, const float* H, float* dZ, int num_sms);
int launch_softmax_xent(cudaStream_t s, int64_t M, int64_t N, const float* L, const int32_t* labels, float* P,
                        float* dL, double* row_loss, double* loss_sum);
// scratch (may be NULL): chunks * N floats for the two-stage fixed-order form
int launch_col_sum(cudaStream_t s, int64_t M, int64_t N, const float* dZ, float* db, int num_sms,
                   float* scratch = nullptr, size_t scratch_bytes = 0);
int launch_sgd(cudaStream_t s, int64_t n, float* w, const float* g, float lr, int num_sms);

}  // namespace split3
