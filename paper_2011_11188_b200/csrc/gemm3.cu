// gemm3.cu — steps a3 (FP16 tensor-core products) and a4 (fused rescaling epilogue).
//
// Eq. A_2 with the dropped term:
//     D_hi  = A1 * B1                    (coefficient a1b1)
//     D_mid = A1 * B2 + A2 * B1          (both carry a1b2 = a2b1 = 2^-11 a1b1, one accumulator)
//     D_lo  = A2 * B2                    (2^-22 a1b1; only with SPLIT3_FOUR_TERM)
//     C     = (D_hi + 2^-11 D_mid [+ 2^-22 D_lo]) * 2^(sA+sB)      (DESIGN.md §3 R7)
// FP16 inputs, FP32 accumulation -> tcgen05.mma kind::f16, D in TMEM.
//
// sm_100a design:
//  * persistent, one CTA per SM, static tile schedule with grouped rasterisation;
//  * warp 0 = TMA producer (one lane): A1/A2 (128 x 64) and B1t/B2t (128 x 64) boxes per
//    stage, 128-byte swizzle, into a STAGES-deep shared-memory ring guarded by mbarriers;
//  * warp 1 = MMA issuer (one lane): per 16-wide k step, 3 tcgen05.mma (4 with D_lo) of
//    M=128, N=128, K=16 into TMEM; tcgen05.commit releases the smem stage / signals the
//    epilogue; it also owns the TMEM allocation;
//  * warps 2..5 = epilogue: tcgen05.ld 32 columns of D_hi/D_mid(/D_lo) per step, one fma,
//    the exact power-of-two rescale, masked float4 stores.  The accumulators are double
//    buffered in TMEM (2 x 256 of 512 columns) so the epilogue of tile i overlaps the
//    mainloop of tile i+1 (3-term and 1-term; 4-term uses a single 384-column buffer).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace split3 {
namespace {

constexpr int BM = 128;
constexpr int BN = 128;
constexpr int BK = 64;                              // 64 fp16 = 128 B = one swizzle row
constexpr int STAGES = 3;
constexpr int TILE_A_BYTES = BM * BK * 2;           // 16 KB
constexpr int TILE_B_BYTES = BN * BK * 2;           // 16 KB
constexpr int STAGE_BYTES = 2 * TILE_A_BYTES + 2 * TILE_B_BYTES;   // 64 KB
constexpr int NUM_THREADS = 192;                    // 6 warps
constexpr int GROUP_M = 16;                         // rasterisation group (m-blocks)
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align slack*/ + 256 /*barriers*/;

// ------------------------------------------------------------------ PTX wrappers -------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int32_t x, int32_t y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, kind::f16, FP32 accumulation.
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                        uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);   // start address      [0,14)
    d |= (uint64_t)1 << 16;                       // LBO (unused, SW128 K-major) [16,30)
    d |= (uint64_t)(1024 >> 4) << 32;             // SBO = 1024 B       [32,46)
    d |= (uint64_t)1 << 46;                       // descriptor version [46,48) = 1 (sm_100)
    d |= (uint64_t)2 << 61;                       // layout: SWIZZLE_128B
    return d;
}

// Instruction descriptor, kind::f16: A = B = F16, D = F32, both K-major, M x N.
__host__ __device__ constexpr uint32_t make_idesc(int m, int n) {
    return (1u << 4)                              // D format F32
         | (0u << 7) | (0u << 10)                 // A, B format F16
         | (0u << 15) | (0u << 16)                // A, B K-major
         | ((uint32_t)(n >> 3) << 17)             // N >> 3
         | ((uint32_t)(m >> 4) << 24);            // M >> 4
}

__device__ __forceinline__ void tile_coords(int64_t tile, int64_t num_m, int64_t num_n,
                                            int64_t& mb, int64_t& nb) {
    const int64_t per_group = (int64_t)GROUP_M * num_n;
    const int64_t g = tile / per_group;
    const int64_t first_m = g * GROUP_M;
    int64_t gsize = num_m - first_m;
    if (gsize > GROUP_M) gsize = GROUP_M;
    const int64_t r = tile - g * per_group;
    mb = first_m + r % gsize;
    nb = r / gsize;
}

// Exact 2^e scaling with a single rounding (only the result can round: underflow/overflow).
__device__ __forceinline__ float scale_pow2(float v, int e, float f, bool fast) {
    return fast ? v * f : ldexpf(v, e);
}

template <int TERMS>
__global__ void __launch_bounds__(NUM_THREADS, 1)
gemm3_kernel(const __grid_constant__ CUtensorMap mapA1, const __grid_constant__ CUtensorMap mapA2,
             const __grid_constant__ CUtensorMap mapB1, const __grid_constant__ CUtensorMap mapB2,
             int M, int N, int K, const int32_t* __restrict__ d_sA,
             const int32_t* __restrict__ d_sB, float* __restrict__ C, int64_t ldc) {
    constexpr int NACC = TERMS == 1 ? 1 : (TERMS == 3 ? 2 : 3);    // accumulators per tile
    constexpr int ACC_STAGES = (NACC * BN * 2 <= 512) ? 2 : 1;
    constexpr uint32_t TMEM_COLS = 512;
    constexpr bool LOAD_LO = TERMS != 1;
    constexpr uint32_t TX_BYTES = LOAD_LO ? STAGE_BYTES : TILE_A_BYTES + TILE_B_BYTES;
    constexpr uint32_t IDESC = make_idesc(BM, BN);

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* full_bar = bars;                       // [STAGES]
    uint64_t* empty_bar = bars + STAGES;             // [STAGES]
    uint64_t* tfull_bar = bars + 2 * STAGES;         // [ACC_STAGES]
    uint64_t* tempty_bar = bars + 2 * STAGES + 2;    // [ACC_STAGES]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
    const int64_t num_tiles = num_m * num_n;
    const int num_kb = (K + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&mapA1); tma_prefetch(&mapB1);
        if (LOAD_LO) { tma_prefetch(&mapA2); tma_prefetch(&mapB2); }
        for (int i = 0; i < STAGES; i++) {
            mbar_init(smem_u32(&full_bar[i]), 1);
            mbar_init(smem_u32(&empty_bar[i]), 1);
        }
        for (int i = 0; i < ACC_STAGES; i++) {
            mbar_init(smem_u32(&tfull_bar[i]), 1);
            mbar_init(smem_u32(&tempty_bar[i]), 4);      // one arrive per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int64_t mb, nb;
                tile_coords(tile, num_m, num_n, mb, nb);
                const int32_t y_a = (int32_t)(mb * BM), y_b = (int32_t)(nb * BN);
                for (int kb = 0; kb < num_kb; kb++) {
                    mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
                    const uint32_t fb = smem_u32(&full_bar[stage]);
                    mbar_expect_tx(fb, TX_BYTES);
                    uint8_t* st = smem + stage * STAGE_BYTES;
                    const int32_t x = kb * BK;
                    tma_load_2d(smem_u32(st), &mapA1, fb, x, y_a);
                    tma_load_2d(smem_u32(st + 2 * TILE_A_BYTES), &mapB1, fb, x, y_b);
                    if (LOAD_LO) {
                        tma_load_2d(smem_u32(st + TILE_A_BYTES), &mapA2, fb, x, y_a);
                        tma_load_2d(smem_u32(st + 2 * TILE_A_BYTES + TILE_B_BYTES), &mapB2, fb, x, y_b);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int as = 0;
            uint32_t aphase = 0;
            for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                mbar_wait(smem_u32(&tempty_bar[as]), aphase ^ 1);
                tc_fence_after();
                const uint32_t t_hi = tmem_base + (uint32_t)(as * NACC * BN);
                const uint32_t t_mid = t_hi + BN;
                const uint32_t t_lo = t_hi + 2 * BN;
                for (int kb = 0; kb < num_kb; kb++) {
                    mbar_wait(smem_u32(&full_bar[stage]), phase);
                    tc_fence_after();
                    uint8_t* st = smem + stage * STAGE_BYTES;
                    const uint64_t a1 = sdesc_sw128(smem_u32(st));
                    const uint64_t a2 = sdesc_sw128(smem_u32(st + TILE_A_BYTES));
                    const uint64_t b1 = sdesc_sw128(smem_u32(st + 2 * TILE_A_BYTES));
                    const uint64_t b2 = sdesc_sw128(smem_u32(st + 2 * TILE_A_BYTES + TILE_B_BYTES));
#pragma unroll
                    for (int k = 0; k < BK / 16; k++) {
                        const uint64_t dk = (uint64_t)(2 * k);   // +32 B along K per 16 elements
                        const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
                        mma_f16(t_hi, a1 + dk, b1 + dk, IDESC, acc);
                        if (TERMS >= 3) {
                            mma_f16(t_mid, a1 + dk, b2 + dk, IDESC, acc);
                            mma_f16(t_mid, a2 + dk, b1 + dk, IDESC, 1u);
                        }
                        if (TERMS == 4) mma_f16(t_lo, a2 + dk, b2 + dk, IDESC, acc);
                    }
                    mma_commit(smem_u32(&empty_bar[stage]));      // smem stage free when done
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                mma_commit(smem_u32(&tfull_bar[as]));             // accumulators ready
                if (++as == ACC_STAGES) { as = 0; aphase ^= 1; }
            }
        }
    } else {
        // ===================== epilogue (warps 2..5) =====================
        const int quad = warp & 3;                       // TMEM lane quadrant of this warp
        const int sAB = *d_sA + *d_sB;
        const bool fast = sAB >= -126 && sAB <= 127;
        const float fscale = fast ? __uint_as_float((unsigned)(sAB + 127) << 23) : 1.0f;
        const bool vec_ok = (ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(C) & 15u) == 0);
        int as = 0;
        uint32_t aphase = 0;
        for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            int64_t mb, nb;
            tile_coords(tile, num_m, num_n, mb, nb);
            mbar_wait(smem_u32(&tfull_bar[as]), aphase);
            tc_fence_after();
            const int64_t row = mb * BM + quad * 32 + lane;
            const uint32_t t_row = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(as * NACC * BN);
            float* crow = C + row * ldc;
#pragma unroll 1
            for (int c = 0; c < BN / 32; c++) {
                uint32_t hi[32], mid[32], lo[32];
                tmem_ld32(t_row + c * 32, hi);
                if (TERMS >= 3) tmem_ld32(t_row + BN + c * 32, mid);
                if (TERMS == 4) tmem_ld32(t_row + 2 * BN + c * 32, lo);
                tmem_ld_wait();
                float out[32];
#pragma unroll
                for (int j = 0; j < 32; j++) {
                    float v = __uint_as_float(hi[j]);
                    if (TERMS == 3) v = __fmaf_rn(__uint_as_float(mid[j]), 0x1p-11f, v);
                    if (TERMS == 4)
                        v = __fmaf_rn(__fmaf_rn(__uint_as_float(lo[j]), 0x1p-11f, __uint_as_float(mid[j])),
                                      0x1p-11f, v);
                    out[j] = scale_pow2(v, sAB, fscale, fast);
                }
                const int64_t col0 = nb * BN + c * 32;
                if (row < M) {
                    if (vec_ok && col0 + 32 <= N) {
                        float4* dst = reinterpret_cast<float4*>(crow + col0);
#pragma unroll
                        for (int j = 0; j < 8; j++)
                            dst[j] = make_float4(out[4 * j], out[4 * j + 1], out[4 * j + 2], out[4 * j + 3]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; j++)
                            if (col0 + j < N) crow[col0 + j] = out[j];
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&tempty_bar[as]));
            if (++as == ACC_STAGES) { as = 0; aphase ^= 1; }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS)
                     : "memory");
    }
}

// ------------------------------------------------------------------ host side ---------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2-D map over a K-major FP16 plane: rows x K elements, leading dimension ld (elements).
bool make_plane_map(CUtensorMap* map, const void* base, int64_t rows, int64_t K, int64_t ld,
                    int box_rows) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
    cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int TERMS>
int launch_t(cudaStream_t st, int64_t M, int64_t N, int64_t K, const CUtensorMap& a1,
             const CUtensorMap& a2, const CUtensorMap& b1, const CUtensorMap& b2,
             const int32_t* d_sA, const int32_t* d_sB, float* C, int64_t ldc, int num_sms) {
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(gemm3_kernel<TERMS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_BYTES) != cudaSuccess)
            return -1;
        attr_set = true;
    }
    const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
    const int grid = (int)(tiles < num_sms ? tiles : num_sms);
    gemm3_kernel<TERMS><<<grid, NUM_THREADS, SMEM_BYTES, st>>>(a1, a2, b1, b2, (int)M, (int)N, (int)K,
                                                               d_sA, d_sB, C, ldc);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace

int launch_gemm3(cudaStream_t st, int64_t M, int64_t N, int64_t K, const uint16_t* A1,
                 const uint16_t* A2, int64_t ldpa, const int32_t* d_sA, const uint16_t* B1t,
                 const uint16_t* B2t, int64_t ldpb, const int32_t* d_sB, float* C, int64_t ldc,
                 int terms, int num_sms, int* err) {
    CUtensorMap ma1, ma2, mb1, mb2;
    const uint16_t* A2e = terms == 1 ? A1 : A2;
    const uint16_t* B2e = terms == 1 ? B1t : B2t;
    if (!make_plane_map(&ma1, A1, M, K, ldpa, BM) || !make_plane_map(&ma2, A2e, M, K, ldpa, BM) ||
        !make_plane_map(&mb1, B1t, N, K, ldpb, BN) || !make_plane_map(&mb2, B2e, N, K, ldpb, BN)) {
        *err = 4;   // SPLIT3_ERR_CUDA
        return -1;
    }
    int r;
    if (terms == 1) r = launch_t<1>(st, M, N, K, ma1, ma2, mb1, mb2, d_sA, d_sB, C, ldc, num_sms);
    else if (terms == 4) r = launch_t<4>(st, M, N, K, ma1, ma2, mb1, mb2, d_sA, d_sB, C, ldc, num_sms);
    else r = launch_t<3>(st, M, N, K, ma1, ma2, mb1, mb2, d_sA, d_sB, C, ldc, num_sms);
    if (r < 0) *err = 4;
    return r;
}

}  // namespace split3
