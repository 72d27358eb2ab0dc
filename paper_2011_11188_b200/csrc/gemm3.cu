// gemm3.cu — steps a3 (FP16 tensor-core products) and a4 (fused rescaling epilogue).
//
// Eq. A_2 with the dropped term:
//     D_hi  = A1 * B1                    (coefficient a1b1)
//     D_mid = A1 * B2 + A2 * B1          (both carry a1b2 = a2b1 = 2^-11 a1b1, one accumulator)
//     D_lo  = A2 * B2                    (2^-22 a1b1; only with SPLIT3_FOUR_TERM)
//     C     = (D_hi + 2^-11 D_mid [+ 2^-22 D_lo]) * 2^(sA+sB)      (DESIGN.md §3 R7)
// FP16 inputs, FP32 accumulation -> tcgen05.mma kind::f16, D in TMEM.
//
// FP32 accumulation on sm_100 tcgen05 TRUNCATES (measured: tests/test_gpu_parity.py
// ::test_tc_accumulation_probe, DESIGN.md §3 R9).  D_hi therefore accumulates in TMEM for at
// most `promo_kb` k-blocks (4*promo_kb MMAs), after which the epilogue warps add the chunk,
// with one round-to-nearest FP32 add, into a master copy held in registers ("promotion").
// D_mid (weight 2^-11) and D_lo (2^-22) accumulate over the whole K in TMEM.
//
// sm_100a design:
//  * CTA pairs (cluster of 2, tcgen05 cta_group::2): one 256 x 128 C tile per pair; CTA r of
//    the pair loads A rows [m0 + 128 r, +128) and B^T rows [n0 + 64 r, +64); the leader's
//    single thread issues M=256, N=128, K=16 MMAs that read both CTAs' shared memory, and
//    each CTA's TMEM holds its 128 rows of the accumulators;
//  * persistent: gridDim.x/2 pairs walk the tiles with a static, grouped raster;
//  * warp 0 = TMA producer, warp 1 = MMA issuer (leader CTA) + TMEM owner, warps 2..5 =
//    epilogue (promotion + final combine + masked stores);
//  * TMEM (512 columns per CTA): D_hi ping-pong chunk buffers [0,128) and [128,256);
//    D_mid double-buffered across tiles at [256,384) and [384,512) (3-term).  4-term: one
//    D_mid buffer at 256 and D_lo at 384.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace split3 {
namespace {

constexpr int BM = 128;                             // rows per CTA (pair: 256)
constexpr int BN = 128;                             // columns per pair tile
constexpr int BNH = BN / 2;                         // B^T rows loaded per CTA
constexpr int BK = 64;                              // 64 fp16 = 128 B = one swizzle row
constexpr int STAGES = 4;
constexpr int TILE_A_BYTES = BM * BK * 2;           // 16 KB
constexpr int TILE_B_BYTES = BNH * BK * 2;          // 8 KB
constexpr int STAGE_BYTES = 2 * TILE_A_BYTES + 2 * TILE_B_BYTES;   // 48 KB
constexpr int NUM_THREADS = 192;                    // 6 warps
constexpr int GROUP_M = 8;                          // rasterisation group (pair m-blocks)
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align slack*/ + 256 /*barriers*/;
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;         // shared::cluster address of the leader CTA

// ------------------------------------------------------------------ PTX wrappers -------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// one lane of a converged warp (returns true on exactly one lane)
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "elect.sync _|p, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
}
// arrive on the barrier at this offset in the LEADER CTA (own CTA when called by the leader)
__device__ __forceinline__ void mbar_arrive_leader(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar & PEER_MASK) : "memory");
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
// 2-SM TMA: data lands in this CTA's smem, the transaction bytes on the leader's barrier.
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                 int32_t x, int32_t y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & PEER_MASK), "r"(x), "r"(y)
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
// D[tmem] (+)= A[smem] * B[smem]^T over the CTA pair, kind::f16, FP32 accumulation.
__device__ __forceinline__ void mma_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// arrive (once) on the barrier at this offset in BOTH CTAs of the pair when the MMAs complete
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
        "h"((uint16_t)3)
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

// Add 32 TMEM columns (one row per thread) into master[off .. off+32).
template <int OFF>
__device__ __forceinline__ void promote32(uint32_t taddr, float (&master)[BN]) {
    uint32_t v[32];
    tmem_ld32(taddr + OFF, v);
    tmem_ld_wait();
#pragma unroll
    for (int j = 0; j < 32; j++) master[OFF + j] = __fadd_rn(master[OFF + j], __uint_as_float(v[j]));
}

template <int TERMS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
gemm3_kernel(const __grid_constant__ CUtensorMap mapA1, const __grid_constant__ CUtensorMap mapA2,
             const __grid_constant__ CUtensorMap mapB1, const __grid_constant__ CUtensorMap mapB2,
             int M, int N, int K, int promo_kb, const int32_t* __restrict__ d_sA,
             const int32_t* __restrict__ d_sB, float* __restrict__ C, int64_t ldc) {
    constexpr bool LOAD_LO = TERMS != 1;
    constexpr int MID_BUFS = TERMS == 3 ? 2 : 1;      // D_mid buffers (cross-tile overlap)
    constexpr uint32_t TX_BYTES = 2u * (LOAD_LO ? STAGE_BYTES : TILE_A_BYTES + TILE_B_BYTES);
    constexpr uint32_t IDESC = make_idesc(2 * BM, BN);
    constexpr uint32_t COL_HI = 0;                    // + 128 * hb
    constexpr uint32_t COL_MID = 256;                 // + 128 * mb (3-term)
    constexpr uint32_t COL_LO = 384;                  // 4-term

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* full_bar = bars;                        // [STAGES]   leader: TMA bytes landed
    uint64_t* empty_bar = bars + STAGES;              // [STAGES]   both: stage consumed
    uint64_t* hfull_bar = bars + 2 * STAGES;          // [2]        both: D_hi chunk ready
    uint64_t* hempty_bar = bars + 2 * STAGES + 2;     // [2]        leader: D_hi chunk drained
    uint64_t* mfull_bar = bars + 2 * STAGES + 4;      // [2]        both: D_mid (D_lo) ready
    uint64_t* mempty_bar = bars + 2 * STAGES + 6;     // [2]        leader: D_mid drained
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 8);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t crank = cluster_rank();
    const bool leader = crank == 0;
    const int64_t num_m = (M + 2 * BM - 1) / (2 * BM), num_n = (N + BN - 1) / BN;
    const int64_t num_tiles = num_m * num_n;
    const int num_kb = (K + BK - 1) / BK;
    const int64_t pair = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&mapA1); tma_prefetch(&mapB1);
        if (LOAD_LO) { tma_prefetch(&mapA2); tma_prefetch(&mapB2); }
        for (int i = 0; i < STAGES; i++) {
            mbar_init(smem_u32(&full_bar[i]), 1);
            mbar_init(smem_u32(&empty_bar[i]), 1);
        }
        for (int i = 0; i < 2; i++) {
            mbar_init(smem_u32(&hfull_bar[i]), 1);
            mbar_init(smem_u32(&hempty_bar[i]), 8);      // 4 epilogue warps x 2 CTAs
            mbar_init(smem_u32(&mfull_bar[i]), 1);
            mbar_init(smem_u32(&mempty_bar[i]), 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer (both CTAs; warp-uniform, one elected lane) =====
        {
            int stage = 0;
            uint32_t phase = 0;
            for (int64_t tile = pair; tile < num_tiles; tile += num_pairs) {
                int64_t mb, nb;
                tile_coords(tile, num_m, num_n, mb, nb);
                const int32_t y_a = (int32_t)(mb * 2 * BM + crank * BM);
                const int32_t y_b = (int32_t)(nb * BN + crank * BNH);
                for (int kb = 0; kb < num_kb; kb++) {
                    mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
                    const uint32_t fb = smem_u32(&full_bar[stage]);
                    uint8_t* st = smem + stage * STAGE_BYTES;
                    const int32_t x = kb * BK;
                    if (elect_one()) {
                        if (leader) mbar_expect_tx(fb, TX_BYTES);
                        tma_load_2d_pair(smem_u32(st), &mapA1, fb, x, y_a);
                        tma_load_2d_pair(smem_u32(st + 2 * TILE_A_BYTES), &mapB1, fb, x, y_b);
                        if (LOAD_LO) {
                            tma_load_2d_pair(smem_u32(st + TILE_A_BYTES), &mapA2, fb, x, y_a);
                            tma_load_2d_pair(smem_u32(st + 2 * TILE_A_BYTES + TILE_B_BYTES), &mapB2, fb, x, y_b);
                        }
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA; warp-uniform, one elected lane) ======
        if (leader) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t cc = 0;       // global D_hi chunk counter
            uint32_t tc = 0;       // tile counter
            for (int64_t tile = pair; tile < num_tiles; tile += num_pairs, tc++) {
                const uint32_t mbuf = MID_BUFS == 2 ? (tc & 1) : 0;
                const uint32_t mphase = MID_BUFS == 2 ? ((tc >> 1) & 1) : (tc & 1);
                if (TERMS != 1) {
                    mbar_wait(smem_u32(&mempty_bar[mbuf]), mphase ^ 1);
                    tc_fence_after();
                }
                const uint32_t t_mid = tmem_base + COL_MID + (TERMS == 3 ? 128 * mbuf : 0);
                const uint32_t t_lo = tmem_base + COL_LO;
                for (int kb0 = 0; kb0 < num_kb; kb0 += promo_kb, cc++) {
                    const uint32_t hb = cc & 1, hphase = (cc >> 1) & 1;
                    mbar_wait(smem_u32(&hempty_bar[hb]), hphase ^ 1);
                    tc_fence_after();
                    const uint32_t t_hi = tmem_base + COL_HI + 128 * hb;
                    const int kb1 = kb0 + promo_kb < num_kb ? kb0 + promo_kb : num_kb;
                    for (int kb = kb0; kb < kb1; kb++) {
                        mbar_wait(smem_u32(&full_bar[stage]), phase);
                        tc_fence_after();
                        uint8_t* st = smem + stage * STAGE_BYTES;
                        const uint64_t a1 = sdesc_sw128(smem_u32(st));
                        const uint64_t a2 = sdesc_sw128(smem_u32(st + TILE_A_BYTES));
                        const uint64_t b1 = sdesc_sw128(smem_u32(st + 2 * TILE_A_BYTES));
                        const uint64_t b2 = sdesc_sw128(smem_u32(st + 2 * TILE_A_BYTES + TILE_B_BYTES));
                        if (elect_one()) {
#pragma unroll
                            for (int k = 0; k < BK / 16; k++) {
                                const uint64_t dk = (uint64_t)(2 * k);   // +32 B along K per 16 elements
                                const uint32_t acc_hi = (kb > kb0 || k > 0) ? 1u : 0u;
                                const uint32_t acc_md = (kb > 0 || k > 0) ? 1u : 0u;
                                mma_pair(t_hi, a1 + dk, b1 + dk, IDESC, acc_hi);
                                if (TERMS >= 3) {
                                    mma_pair(t_mid, a1 + dk, b2 + dk, IDESC, acc_md);
                                    mma_pair(t_mid, a2 + dk, b1 + dk, IDESC, 1u);
                                }
                                if (TERMS == 4) mma_pair(t_lo, a2 + dk, b2 + dk, IDESC, acc_md);
                            }
                            mma_commit_pair(smem_u32(&empty_bar[stage]));   // stage free in both CTAs
                        }
                        __syncwarp();
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                    if (elect_one()) mma_commit_pair(smem_u32(&hfull_bar[hb]));   // D_hi chunk ready
                    __syncwarp();
                }
                if (TERMS != 1) {
                    if (elect_one()) mma_commit_pair(smem_u32(&mfull_bar[mbuf]));   // D_mid ready
                    __syncwarp();
                }
            }
        }
    } else {
        // ===================== epilogue (warps 2..5, both CTAs) =====================
        const int quad = warp & 3;                       // TMEM lane quadrant of this warp
        const int sAB = *d_sA + *d_sB;
        const bool fast = sAB >= -126 && sAB <= 127;
        const float fscale = fast ? __uint_as_float((unsigned)(sAB + 127) << 23) : 1.0f;
        const bool vec_ok = (ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(C) & 15u) == 0);
        const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16);
        uint32_t cc = 0, tc = 0;
        for (int64_t tile = pair; tile < num_tiles; tile += num_pairs, tc++) {
            int64_t mb, nb;
            tile_coords(tile, num_m, num_n, mb, nb);
            float master[BN];
#pragma unroll
            for (int j = 0; j < BN; j++) master[j] = 0.0f;
            for (int kb0 = 0; kb0 < num_kb; kb0 += promo_kb, cc++) {
                const uint32_t hb = cc & 1, hphase = (cc >> 1) & 1;
                mbar_wait(smem_u32(&hfull_bar[hb]), hphase);
                tc_fence_after();
                const uint32_t t_hi = lane_base + COL_HI + 128 * hb;
                promote32<0>(t_hi, master);
                promote32<32>(t_hi, master);
                promote32<64>(t_hi, master);
                promote32<96>(t_hi, master);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_leader(smem_u32(&hempty_bar[hb]));
            }
            const uint32_t mbuf = MID_BUFS == 2 ? (tc & 1) : 0;
            const uint32_t mphase = MID_BUFS == 2 ? ((tc >> 1) & 1) : (tc & 1);
            if (TERMS != 1) {
                mbar_wait(smem_u32(&mfull_bar[mbuf]), mphase);
                tc_fence_after();
            }
            const int64_t row = mb * 2 * BM + crank * BM + quad * 32 + lane;
            float* crow = C + row * ldc;
            const uint32_t t_mid = lane_base + COL_MID + (TERMS == 3 ? 128 * mbuf : 0);
            const uint32_t t_lo = lane_base + COL_LO;
#pragma unroll
            for (int c = 0; c < BN / 32; c++) {
                float out[32];
                if (TERMS == 1) {
#pragma unroll
                    for (int j = 0; j < 32; j++) out[j] = master[c * 32 + j];
                } else {
                    uint32_t mid[32];
                    tmem_ld32(t_mid + c * 32, mid);
                    if (TERMS == 4) {
                        uint32_t lo[32];
                        tmem_ld32(t_lo + c * 32, lo);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; j++)
                            out[j] = __fmaf_rn(__fmaf_rn(__uint_as_float(lo[j]), 0x1p-11f, __uint_as_float(mid[j])),
                                               0x1p-11f, master[c * 32 + j]);
                    } else {
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 32; j++)
                            out[j] = __fmaf_rn(__uint_as_float(mid[j]), 0x1p-11f, master[c * 32 + j]);
                    }
                }
#pragma unroll
                for (int j = 0; j < 32; j++) out[j] = fast ? out[j] * fscale : ldexpf(out[j], sAB);
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
            if (TERMS != 1) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_leader(smem_u32(&mempty_bar[mbuf]));
            }
        }
    }

    tc_fence_before();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
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
             const int32_t* d_sA, const int32_t* d_sB, float* C, int64_t ldc, int num_sms,
             int promo_kb) {
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(gemm3_kernel<TERMS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_BYTES) != cudaSuccess)
            return -1;
        attr_set = true;
    }
    const int64_t tiles = ((M + 2 * BM - 1) / (2 * BM)) * ((N + BN - 1) / BN);
    const int64_t pairs = num_sms / 2;
    const int grid = 2 * (int)(tiles < pairs ? tiles : pairs);
    gemm3_kernel<TERMS><<<grid, NUM_THREADS, SMEM_BYTES, st>>>(a1, a2, b1, b2, (int)M, (int)N, (int)K,
                                                               promo_kb, d_sA, d_sB, C, ldc);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace

int launch_gemm3(cudaStream_t st, int64_t M, int64_t N, int64_t K, const uint16_t* A1,
                 const uint16_t* A2, int64_t ldpa, const int32_t* d_sA, const uint16_t* B1t,
                 const uint16_t* B2t, int64_t ldpb, const int32_t* d_sB, float* C, int64_t ldc,
                 int terms, int num_sms, int promo_kb, int* err) {
    CUtensorMap ma1, ma2, mb1, mb2;
    const uint16_t* A2e = terms == 1 ? A1 : A2;
    const uint16_t* B2e = terms == 1 ? B1t : B2t;
    if (!make_plane_map(&ma1, A1, M, K, ldpa, BM) || !make_plane_map(&ma2, A2e, M, K, ldpa, BM) ||
        !make_plane_map(&mb1, B1t, N, K, ldpb, BNH) || !make_plane_map(&mb2, B2e, N, K, ldpb, BNH)) {
        *err = 4;   // SPLIT3_ERR_CUDA
        return -1;
    }
    const int promo = promo_kb > 0 ? promo_kb : kDefaultPromoKb;
    int r;
    if (terms == 1) r = launch_t<1>(st, M, N, K, ma1, ma2, mb1, mb2, d_sA, d_sB, C, ldc, num_sms, promo);
    else if (terms == 4) r = launch_t<4>(st, M, N, K, ma1, ma2, mb1, mb2, d_sA, d_sB, C, ldc, num_sms, promo);
    else r = launch_t<3>(st, M, N, K, ma1, ma2, mb1, mb2, d_sA, d_sB, C, ldc, num_sms, promo);
    if (r < 0) *err = 4;
    return r;
}

}  // namespace split3
