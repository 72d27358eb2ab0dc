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
// sm_100a design, v3:
//  * CTA pairs (cluster of 2, tcgen05 cta_group::2): one 256 x 256 C tile per pair (4-term:
//    256 x 128); CTA r of the pair TMA-loads A rows [m0 + 128 r, +128) and B rows
//    [n0 + 128 r, +128) of each 64-wide k-block (128-B swizzle; B K-major or MN-major), and the
//    leader's single elected thread issues the M = 256, K = 16 MMAs that read both CTAs' shared
//    memory; each CTA's TMEM holds its 128 rows of the accumulators;
//  * persistent: gridDim.x / 2 pairs walk the work units (whole tiles, then the split-K slices of
//    the tail wave) with a grouped raster; a bounded wave lockstep keeps the concurrent tiles in
//    the same K window of L2;
//  * warp 0 = TMA producer, warp 1 = MMA issuer (leader CTA) + TMEM owner, warps 2..9 = 8
//    epilogue warps (two per TMEM lane quadrant, 128 columns each: D_hi promotion into an FP32
//    master in registers, the final fma with D_mid, the exact 2^(sA+sB) rescale and TMA stores);
//    fused-B builds add warps 10..11, converters that split B's fp32 tiles in shared memory;
//  * TMEM (512 columns per CTA): 3-term D_hi [0,256) + D_mid [256,512) (one D_hi buffer: the MMA
//    warp issues a k-block's D_mid MMAs before waiting for the drained D_hi); unfolded 4-term
//    (BN = 128) D_hi ping-pong [0,256) + D_mid [256,384) + D_lo [384,512); 1-term D_hi ping-pong;
//  * folded accumulator (LAY bit 3, the 4-term default): per k-block ONE accumulator T takes
//    A2*B2, then A1*B2 + A2*B1 entered with tcgen05 scale-input-d 11 (T <- P + 2^-11 T), then
//    A1*B1 likewise; T ping-pongs in [0,256) / [256,512) and is promoted every k-block — no D_mid
//    or D_lo accumulator, so 4-term keeps 256-wide tiles.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string.h>

#include "internal.h"
#include "split_math.h"

namespace split3 {
namespace {

constexpr int BM = 128;                             // rows per CTA (pair: 256)
constexpr int BK = 64;                              // 64 fp16 = 128 B = one swizzle row
constexpr int TILE_A_BYTES = BM * BK * 2;           // 16 KB
constexpr int NUM_EPI_WARPS = 8;                    // 2 per TMEM lane quadrant
constexpr int NUM_THREADS = 64 + 32 * NUM_EPI_WARPS;   // TMA warp, MMA warp, epilogue warps
constexpr int NUM_CONV_WARPS = 2;                   // fused-B variant: fp32 -> plane converter warps
constexpr int LAY_FB = 4;                           // LAY bit 2: B arrives as fp32, split in SMEM
constexpr int LAY_FOLD = 8;                         // LAY bit 3: one accumulator per k-block (scale-input-d fold)
template <int LAY>
struct NThr { static constexpr int v = NUM_THREADS + ((LAY & LAY_FB) ? 32 * NUM_CONV_WARPS : 0); };
constexpr uint32_t TMEM_COLS = 512;
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;         // shared::cluster address of the leader CTA

// L2 cache-policy encodings for the .L2::cache_hint operand (as CUTLASS's CacheHintSm90).
constexpr uint64_t kPolicyNormal = 0x1000000000000000ull;
constexpr uint64_t kPolicyFirst = 0x12F0000000000000ull;
constexpr uint64_t kPolicyLast = 0x14F0000000000000ull;

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
__device__ __forceinline__ uint64_t globaltimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// Wave lockstep (L2 locality): every CTA's producer announces that it starts its
// i-th tile, then waits — at most kWaveWaitNs — until all CTAs that have an i-th tile did.  A
// performance hint only: the bounded wait can never deadlock (e.g. if not all CTAs are resident).
constexpr uint64_t kWaveWaitNs = 200000;
// The counter starts every launch at 0: the last CTA to exit zeroes it (see the kernel's end).
__device__ __forceinline__ void wave_sync(unsigned* counter, unsigned target) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(counter) : "memory");
    const uint64_t t0 = globaltimer_ns();
    unsigned v;
    do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        if ((int)(v - target) >= 0) break;
        __nanosleep(64);
    } while (globaltimer_ns() - t0 < kWaveWaitNs);
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
// ---- debug build (SPLIT3_DEBUG=1: libsplit3_debug.so) ----------------------
// What compute-sanitizer would check in this kernel's synchronisation, built in.  Every mbarrier
// wait has a watchdog (kDbgWatchdogNs of globaltimer): on expiry the failure is written to
// host-mapped pinned memory (readable even after the context is lost) and the kernel traps, so a
// broken pipeline ends with a report and a launch error instead of a hung GPU.  The other checks
// record and continue.  Record: [0] first failure code, [1] detail, [2] CTA, [3] warp, [4] number
// of failures.  Codes: 1 mbarrier watchdog (detail = barrier smem address << 32 | parity), 2 TMEM
// base not column 0, 3 tile coordinates out of range, 4 shared-memory carve-out beyond the dynamic
// allocation, 5 empty k-block range, 6 D_hi chunks committed != chunks drained, 7 wave counter not
// 2 x (units - busy pairs).  g_dbg_fault (split3_debug_fault) injects a missing TMA load (1).
#ifndef SPLIT3_DEBUG
#define SPLIT3_DEBUG 0
#endif
#if SPLIT3_DEBUG
constexpr uint64_t kDbgWatchdogNs = 2000000000ull;
__device__ unsigned long long* g_dbg;   // host-mapped record (gemm3_debug_init)
__device__ int g_dbg_fault;
__device__ __noinline__ void dbg_report(unsigned code, unsigned long long detail) {
    if (!g_dbg) return;
    if (atomicCAS_system(&g_dbg[0], 0ull, (unsigned long long)code) == 0ull) {
        g_dbg[1] = detail;
        g_dbg[2] = blockIdx.x;
        g_dbg[3] = threadIdx.x >> 5;
    }
    atomicAdd_system(&g_dbg[4], 1ull);
    __threadfence_system();
}
#define DBG_CHECK(cond, code, detail) \
    do {                               \
        if (!(cond)) dbg_report((code), (unsigned long long)(detail)); \
    } while (0)
#else
#define DBG_CHECK(cond, code, detail) \
    do {                               \
    } while (0)
#endif

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t done;
#if SPLIT3_DEBUG
    const uint64_t t0 = globaltimer_ns();
    uint32_t spins = 0;
#endif
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
#if SPLIT3_DEBUG
        if (!done && (++spins & 255u) == 0 && globaltimer_ns() - t0 > kDbgWatchdogNs) {
            dbg_report(1, ((unsigned long long)bar << 32) | parity);
            __trap();
        }
#endif
    } while (!done);
}
// 2-SM TMA: data lands in this CTA's smem, the transaction bytes on the leader's barrier.
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                 int32_t x, int32_t y, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & PEER_MASK), "r"(x), "r"(y), "l"(policy)
        : "memory");
}
// 1-SM TMA into this CTA's smem, transaction bytes on this CTA's barrier (fused-B fp32 tiles).
__device__ __forceinline__ void tma_load_2d_cta(uint32_t dst, const CUtensorMap* map, uint32_t bar, int32_t x,
                                                int32_t y, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y), "l"(policy)
        : "memory");
}
// TMA store of a shared-memory box to global (bulk async group of the issuing thread)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int32_t x, int32_t y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void st_shared_f32(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ float ld_shared_f32(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, float a, float b, float c, float d) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
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
// The same with the A operand kept in the tensor core's collector buffer (A_KEEP: read from shared
// memory and keep) or taken from it (A_REUSE: no shared-memory read of A); for two consecutive
// MMAs that multiply the same A tile (A1 * B1 into D_hi, then A1 * B2 into D_mid).
__device__ __forceinline__ void mma_pair_keep_a(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16.collector::a::fill [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void mma_pair_reuse_a(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                 uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// D = A * B + 2^-11 * D (tcgen05 scale-input-d = 11): the folded accumulator's step from a
// lower-weight group of products to the next one up (LAY_FOLD)
__device__ __forceinline__ void mma_pair_fold11(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, 1, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p, 11;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc)
        : "memory");
}
// arrive (once) on the barrier at this offset in BOTH CTAs of the pair when the MMAs complete
__device__ __forceinline__ void mma_commit_pair(uint32_t bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
        "h"((uint16_t)3)
        : "memory");
}
// 32 lanes x 16 consecutive 32-bit columns -> 16 registers per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
// 32 lanes x 8 consecutive 32-bit columns -> 8 registers per thread.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() {
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart.
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t sbo = 1024) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);   // start address      [0,14)
    d |= (uint64_t)1 << 16;                       // LBO (unused, SW128 K-major) [16,30)
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;  // SBO (1024 B: dense 8-row groups) [32,46)
    d |= (uint64_t)1 << 46;                       // descriptor version [46,48) = 1 (sm_100)
    d |= (uint64_t)2 << 61;                       // layout: SWIZZLE_128B
    return d;
}

// Smem descriptor of an MN-major (N-contiguous) SW128 operand: 64-element (128-B) rows along N,
// 8 k-rows per 1024-B swizzle atom; SBO = 1024 B between 8-k groups, LBO = `lbo` bytes between
// 64-wide N atoms (here: consecutive 64 x 64 TMA boxes).  One K = 16 MMA step = +2048 B.
__device__ __forceinline__ uint64_t sdesc_mn_sw128(uint32_t saddr, uint32_t lbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);   // start address      [0,14)
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;  // LBO                [16,30)
    d |= (uint64_t)(1024 >> 4) << 32;             // SBO = 1024 B       [32,46)
    d |= (uint64_t)1 << 46;                       // descriptor version [46,48) = 1 (sm_100)
    d |= (uint64_t)2 << 61;                       // layout: SWIZZLE_128B
    return d;
}

// Instruction descriptor, kind::f16: A = B = F16, D = F32, both K-major, M x N.
__host__ __device__ constexpr uint32_t make_idesc(int m, int n, bool bf16 = false) {
    return (1u << 4)                              // D format F32
         | ((bf16 ? 1u : 0u) << 7) | ((bf16 ? 1u : 0u) << 10)   // A, B format F16 (0) / BF16 (1)
         | (0u << 15) | (0u << 16)                // A, B K-major
         | ((uint32_t)(n >> 3) << 17)             // N >> 3
         | ((uint32_t)(m >> 4) << 24);            // M >> 4
}

// Unit and tile indices are 32-bit on the device (the host rejects > 2^31 - 1 work units): fewer
// live registers in the epilogue, whose 128-float FP32 master leaves little room.
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int group_m, int& mb, int& nb) {
    const int per_group = group_m * num_n;
    const int g = tile / per_group;
    const int first_m = g * group_m;
    int gsize = num_m - first_m;
    if (gsize > group_m) gsize = group_m;
    const int r = tile - g * per_group;
    mb = first_m + r % gsize;
    nb = r / gsize;
}

// Device copy of the host's SplitPlan in 32-bit fields.
struct UnitPlan {
    int whole, nsplit, slices;
};

__device__ __forceinline__ void decode_unit(int u, const UnitPlan& p, int num_kb, int kps, int& tile, int& kb_begin,
                                            int& kb_end, int& slot) {
    if (u < p.whole) {
        tile = u;
        kb_begin = 0;
        kb_end = num_kb;
        slot = -1;
        return;
    }
    const int v = u - p.whole;
    const int t = v % p.nsplit;
    const int s = v / p.nsplit;
    tile = p.whole + t;
    kb_begin = s * kps;
    kb_end = kb_begin + kps < num_kb ? kb_begin + kps : num_kb;
    slot = v;   // = s * nsplit + t
}

// Tile geometry per instantiation: BN_ = 256 (3-term, 1-term, bf16x3) or 128 (4-term: D_lo
// needs TMEM); PL = planes per operand (2, or 3 for bf16x3).
template <int BN_, int PL = 2>
struct Geo {
    static constexpr int BNH = BN_ / 2;                               // B^T rows loaded per CTA
    static constexpr int TILE_B_BYTES = BNH * BK * 2;
    static constexpr int STAGE_BYTES = PL * TILE_A_BYTES + PL * TILE_B_BYTES;
    static constexpr int STAGES = (220 * 1024) / STAGE_BYTES > 6 ? 6 : (220 * 1024) / STAGE_BYTES;
    static constexpr int STAGING = 8 * 4096;   // epilogue: 4 KB (32 rows x 32 fp32) per warp
    static constexpr int SMEM = STAGES * STAGE_BYTES + STAGING + 1024 + 256;
};

// Add this thread's row of NCOL TMEM columns into master[], 16 columns per tcgen05.ld.
template <int NCOL>
__device__ __forceinline__ void promote_all(uint32_t taddr, float (&master)[NCOL]) {
#pragma unroll
    for (int c = 0; c < NCOL / 16; c++) {
        uint32_t v[16];
        tmem_ld16(taddr + c * 16, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; j++) master[c * 16 + j] = __fadd_rn(master[c * 16 + j], __uint_as_float(v[j]));
    }
}

// LAY bit 0 (BMN): the B planes are MN-major (K x N row-major, as split from a row-major K x N fp32
// B without a transpose), else K-major (N x K); bit 1 (AMN): likewise A (K x M planes of a stored
// K x M fp32 A = op(A)^T), else K-major (M x K).
// Fused-B stage layout: the fp32 B tile of a k-block (64 k-rows x 128 N, 512-B
// rows, no swizzle) is TMA-loaded into the stage's 32 KB B region and split IN PLACE, one K = 16
// MMA step (16 k-rows = 8 KB) at a time: the step's planes take exactly its own 8 KB,
//     hi: N atom 0 at +0, N atom 1 at +2 KB;  lo: +4 KB, +6 KB   (MN-major SW128, SBO 1 KB),
// so the MMA reads B1 at B_OFF + 8 KB * k with LBO 2 KB, B2 at +4 KB.
constexpr int FB_STEP_BYTES = 8192;
constexpr int FB_LBO = 2048;
constexpr int FB_LO_OFF = 4096;
// K-major (B given as B^T, stored N x K): the tile is 128 n-rows x 64 K (256-B rows); each 8-row
// group (2 KB) is split in place into its hi atom (+0, 8 rows x 128 B, SW128) and lo atom (+1 KB),
// so the MMA reads B1 with SBO 2 KB and B2 at +1 KB; a K = 16 step is +32 B as usual.
constexpr int FBK_GROUP_BYTES = 2048;
constexpr int FBK_LO_OFF = 1024;

// Split one K step in place (one converter warp): each of the 16 LDS.128 reads one fp32 k-row
// (lane L: N values 4L..4L+3, conflict-free), all reads precede all writes (__syncwarp), then every
// lane stores two 8-B pieces (hi, lo) of 16-B SW128 chunks: lanes 0-15 -> N atom 0, 16-31 -> atom 1.
__device__ __forceinline__ void convert_step(uint8_t* step, int lane, float f) {
    float4 v[16];
#pragma unroll
    for (int r = 0; r < 16; r++) v[r] = *reinterpret_cast<const float4*>(step + r * 512 + lane * 16);
    __syncwarp();
    const int l16 = lane & 15;
    uint8_t* base = step + (lane >> 4) * FB_LBO + ((l16 & 1) << 3);
#pragma unroll
    for (int r = 0; r < 16; r++) {
        uint2 hi, lo;
        split4(v[r], f, hi, lo);
        uint8_t* a = base + (r >> 3) * 1024 + (r & 7) * 128 + (((l16 >> 1) ^ (r & 7)) << 4);
        *reinterpret_cast<uint2*>(a) = hi;
        *reinterpret_cast<uint2*>(a + FB_LO_OFF) = lo;
    }
}

// Split NG 8-row groups (at grp + j * stride) of a K-major fp32 tile in place (one converter
// warp): per group 4 LDS.128 (lane L: row 2i + L/16, K values 4(L%16)..+3, conflict-free); all
// groups' reads precede the writes (__syncwarp; each group's region is this warp's alone); each
// lane then stores 8-B hi / lo pieces of its rows' 16-B SW128 chunks (lanes 0-15 and 16-31 each
// fill one 128-B row per store).  NG groups keep 4 * NG independent rows in flight.
template <int NG>
__device__ __forceinline__ void convert_kgroups(uint8_t* grp, int stride, int lane, float f) {
    float4 v[NG][4];
#pragma unroll
    for (int j = 0; j < NG; j++)
#pragma unroll
        for (int i = 0; i < 4; i++) v[j][i] = *reinterpret_cast<const float4*>(grp + j * stride + i * 512 + lane * 16);
    __syncwarp();
    const int c4 = lane & 15;
#pragma unroll
    for (int j = 0; j < NG; j++)
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const int r = 2 * i + (lane >> 4);    // row within the group (= row & 7 of the atom)
            uint2 hi, lo;
            split4(v[j][i], f, hi, lo);
            uint8_t* a = grp + j * stride + r * 128 + (((c4 >> 1) ^ r) << 4) + ((c4 & 1) << 3);
            *reinterpret_cast<uint2*>(a) = hi;
            *reinterpret_cast<uint2*>(a + FBK_LO_OFF) = lo;
        }
}

// LAY bit 2 (FB, fused B; 3-term): mapB1 is a map
// over the fp32 B (row-major K x N when BMN, else B^T stored N x K), TMA-loaded per k-block into
// the stage's B region; converter warps 10..11 apply Eq. A_1 in place (split4, the split kernels'
// arithmetic) and write the B1/B2 planes in the layouts above.  The scale exponent comes from *fb_maxB; CTA 0 stores it to *fb_sB (read by the
// split-K reduction).
template <int TERMS, int BN_, int LAY>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NThr<LAY>::v, 1)
gemm3_kernel(const __grid_constant__ CUtensorMap mapA1, const __grid_constant__ CUtensorMap mapA2,
             const __grid_constant__ CUtensorMap mapB1, const __grid_constant__ CUtensorMap mapB2,
             const __grid_constant__ CUtensorMap mapA3, const __grid_constant__ CUtensorMap mapB3,
             const __grid_constant__ CUtensorMap mapC, int tma_store,
             int M, int N, int K, int promo_kb, const int32_t* __restrict__ d_sA,
             const int32_t* __restrict__ d_sB, float* __restrict__ C, int64_t ldc,
             unsigned* __restrict__ wave_counter, const GemmTune tune,
             const SplitPlan plan, float* __restrict__ partial, const float* __restrict__ fb_maxB,
             int32_t* __restrict__ fb_sB) {
    constexpr bool BF3 = TERMS == 6;                 // bf16 x 3 split (NEXT #4): 3 planes, 6 products
    constexpr int PL = BF3 ? 3 : 2;
    constexpr bool FB = (LAY & LAY_FB) != 0;
    static_assert(!FB || TERMS == 3, "fused B: 3-term only");
    // Folded accumulator (LAY_FOLD): per k-block ONE TMEM accumulator T takes, in order,
    // [A2*B2 (4-term)], then A1*B2 + A2*B1 entered with scale-input-d 11 (T <- products + 2^-11 T),
    // then A1*B1 entered likewise, so T = D_hi + 2^-11 D_mid [+ 2^-22 D_lo] of that k-block; the
    // epilogue adds T into the FP32 master with RN every k-block (promotion period 1).  No D_mid /
    // D_lo accumulators: two 256-column T buffers ping-pong, 4-term keeps 256-wide tiles.
    constexpr bool FOLD = (LAY & LAY_FOLD) != 0;
    static_assert(!FOLD || ((TERMS == 3 || TERMS == 4) && BN_ == 256), "fold: 3-/4-term, 256-wide tiles");
    using G = Geo<BN_, PL>;
    constexpr int F32_BYTES = G::BNH * BK * 4;   // fused B: one fp32 tile = the stage's B region
    static_assert(!FB || F32_BYTES == 2 * G::TILE_B_BYTES, "fused B: in-place split");
    constexpr int STAGES = G::STAGES;
    constexpr int STAGE_BYTES = G::STAGE_BYTES;
    constexpr int TILE_B_BYTES = G::TILE_B_BYTES;
    constexpr int BNH = G::BNH;
    constexpr bool LOAD_LO = TERMS != 1;
    constexpr bool HAS_MID = TERMS != 1 && !FOLD;
    // TMEM columns per CTA: 512.  D_hi chunk buffers (HB of them), then D_mid (+ D_lo).
    constexpr int HB = (TERMS == 1 || BN_ == 128 || FOLD) ? 2 : 1;
    constexpr uint32_t COL_MID = HB * BN_;
    constexpr uint32_t COL_LO = COL_MID + BN_;
    static_assert(HB * BN_ + (HAS_MID ? BN_ : 0) + (TERMS == 4 && !FOLD ? BN_ : 0) <= 512, "TMEM budget");
    constexpr uint32_t TX_BYTES =
        FB ? 2u * (2 * TILE_A_BYTES) : 2u * (LOAD_LO ? STAGE_BYTES : TILE_A_BYTES + TILE_B_BYTES);
    constexpr bool BMN = (LAY & 1) != 0, AMN = (LAY & 2) != 0;
    constexpr uint32_t IDESC = make_idesc(2 * BM, BN_, BF3) | (AMN ? (1u << 15) : 0u) | (BMN ? (1u << 16) : 0u);
    constexpr uint64_t DKB = (FB && BMN) ? (FB_STEP_BYTES >> 4) : BMN ? (2048 >> 4) : (32 >> 4);   // B step per K = 16
    constexpr uint64_t DKA = AMN ? (2048 >> 4) : (32 >> 4);   // A descriptor step per K = 16
    constexpr int MN_BOX_BYTES = 64 * BK * 2;                 // one 64 (N) x 64 (K) box
    constexpr int B_OFF = PL * TILE_A_BYTES;         // B planes follow the A planes in a stage
    constexpr int NCOL = BN_ / 2;                    // columns per epilogue warp (2 warps per quadrant)
    constexpr uint32_t EPI_ARRIVALS = 2 * NUM_EPI_WARPS;

    extern __shared__ uint8_t smem_raw[];
    // 1024-B aligned (SW128 atoms); offsetting smem_raw keeps the pointer in the shared space
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* staging = smem + STAGES * STAGE_BYTES;   // 1024-aligned (128-B swizzle atoms)
    uint64_t* bars = reinterpret_cast<uint64_t*>(staging + G::STAGING);
    uint64_t* full_bar = bars;                        // [STAGES]   leader: TMA bytes landed
    uint64_t* empty_bar = bars + STAGES;              // [STAGES]   both: stage consumed
    uint64_t* hfull_bar = bars + 2 * STAGES;          // [2]        both: D_hi chunk ready
    uint64_t* hempty_bar = bars + 2 * STAGES + 2;     // [2]        leader: D_hi chunk drained
    uint64_t* mfull_bar = bars + 2 * STAGES + 4;      // [1]        both: D_mid (D_lo) ready
    uint64_t* mempty_bar = bars + 2 * STAGES + 5;     // [1]        leader: D_mid drained
    uint64_t* ffull_bar = bars + 2 * STAGES + 6;      // [STAGES]   own CTA: fused B fp32 tile landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * STAGES + 6);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t crank = cluster_rank();
    const bool leader = crank == 0;
    const int num_m = (M + 2 * BM - 1) / (2 * BM), num_n = (N + BN_ - 1) / BN_;
    const int num_kb = (K + BK - 1) / BK;
    // Work units (SplitPlan, host-chosen): units [0, whole) are whole tiles 0..whole-1; the
    // remaining `nsplit` tiles (the tail wave, or all tiles of a small problem) are cut into
    // `slices` K slices of kps k-blocks: unit whole + s*nsplit + t = slice s of tile whole + t.
    const UnitPlan up{(int)plan.whole, (int)plan.nsplit, plan.slices};
    const int kps = (num_kb + up.slices - 1) / up.slices;
    const int num_units = up.whole + up.nsplit * up.slices;
    const int pair = blockIdx.x >> 1, num_pairs = gridDim.x >> 1;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&mapA1); tma_prefetch(&mapB1);
        if (LOAD_LO) { tma_prefetch(&mapA2); tma_prefetch(&mapB2); }
        if (BF3) { tma_prefetch(&mapA3); tma_prefetch(&mapB3); }
        for (int i = 0; i < STAGES; i++) {
            // fused B: the leader's full barrier also collects one arrival per converter warp of both CTAs
            mbar_init(smem_u32(&full_bar[i]), FB ? 1 + 2 * NUM_CONV_WARPS : 1);
            mbar_init(smem_u32(&empty_bar[i]), 1);
        }
        if (FB)
            for (int i = 0; i < STAGES; i++) mbar_init(smem_u32(&ffull_bar[i]), 1);
        for (int i = 0; i < 2; i++) {
            mbar_init(smem_u32(&hfull_bar[i]), 1);
            mbar_init(smem_u32(&hempty_bar[i]), EPI_ARRIVALS);
        }
        mbar_init(smem_u32(&mfull_bar[0]), 1);
        mbar_init(smem_u32(&mempty_bar[0]), EPI_ARRIVALS);
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
    pdl_wait();   // prologue above overlaps the predecessor's tail; no global access before here
#if SPLIT3_DEBUG
    if (threadIdx.x == 0) {
        DBG_CHECK(tmem_base == 0, 2, tmem_base);   // all 512 columns allocated: base lane 0, column 0
        uint32_t dyn;
        asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
        const uint32_t used = (uint32_t)(reinterpret_cast<uint8_t*>(tmem_slot + 1) - smem_raw);
        DBG_CHECK(used <= dyn, 4, ((unsigned long long)used << 32) | dyn);
    }
    __shared__ uint32_t dbg_chunks;                   // D_hi chunks the MMA warp committed (leader)
#endif

    if (warp == 0) {
        // ===================== TMA producer (both CTAs; warp-uniform, one elected lane) =====
        int stage = 0;
        uint32_t phase = 0;
        unsigned wave_target = 0;   // cumulative arrivals expected up to this unit index (counter starts at 0)
        int idx = 0;
        for (int unit = pair; unit < num_units; unit += num_pairs, idx++) {
            int tile;
            int kb_begin, kb_end, slot;
            decode_unit(unit, up, num_kb, kps, tile, kb_begin, kb_end, slot);
            if (wave_counter && idx > 0) {
                int active = num_units - idx * num_pairs;   // pairs with an idx-th unit
                if (active > num_pairs) active = num_pairs;
                wave_target += 2u * (unsigned)active;
                if (elect_one()) wave_sync(wave_counter, wave_target);
                __syncwarp();
            }
            int mb, nb;
            tile_coords(tile, num_m, num_n, tune.group_m, mb, nb);
            DBG_CHECK(mb >= 0 && mb < num_m && nb >= 0 && nb < num_n, 3, ((unsigned long long)mb << 32) | (unsigned)nb);
            DBG_CHECK(kb_begin < kb_end && kb_end <= num_kb, 5, ((unsigned long long)kb_begin << 32) | (unsigned)kb_end);
            const int32_t y_a = (int32_t)(mb * 2 * BM + crank * BM);
            const int32_t y_b = (int32_t)(nb * BN_ + crank * BNH);
            for (int kb = kb_begin; kb < kb_end; kb++) {
                mbar_wait(smem_u32(&empty_bar[stage]), phase ^ 1);
                const uint32_t fb = smem_u32(&full_bar[stage]);
                uint8_t* st = smem + stage * STAGE_BYTES;
                const int32_t x = kb * BK;
                if (elect_one()) {
                    // K-major B: one 64 (K) x BNH (N) box; MN-major B: BNH/64 boxes of 64 (N) x 64 (K)
                    auto load_b = [&](int off, const CUtensorMap* map) {
                        if (BMN) {
#pragma unroll
                            for (int h = 0; h < BNH / 64; h++)
                                tma_load_2d_pair(smem_u32(st + off + h * MN_BOX_BYTES), map, fb, y_b + 64 * h, x,
                                                 tune.pol_b);
                        } else {
                            tma_load_2d_pair(smem_u32(st + off), map, fb, x, y_b, tune.pol_b);
                        }
                    };
                    auto load_a = [&](int off, const CUtensorMap* map) {
                        if (AMN) {
#pragma unroll
                            for (int h = 0; h < BM / 64; h++)
                                tma_load_2d_pair(smem_u32(st + off + h * MN_BOX_BYTES), map, fb, y_a + 64 * h, x,
                                                 tune.pol_a);
                        } else {
                            tma_load_2d_pair(smem_u32(st + off), map, fb, x, y_a, tune.pol_a);
                        }
                    };
                    if (leader) mbar_expect_tx(fb, TX_BYTES);
                    if (FB) {   // fp32 B tile into the stage's B region (own CTA, own barrier)
                        const uint32_t ffb = smem_u32(&ffull_bar[stage]);
                        mbar_expect_tx(ffb, F32_BYTES);
                        if (BMN) tma_load_2d_cta(smem_u32(st + B_OFF), &mapB1, ffb, y_b, x, tune.pol_b);   // 128 N x 64 K
                        else tma_load_2d_cta(smem_u32(st + B_OFF), &mapB1, ffb, x, y_b, tune.pol_b);       // 64 K x 128 N
                    }
#if SPLIT3_DEBUG
                    // injected fault (tests): the first unit's second k-block loses its A1 load, so
                    // the full barrier's transaction count is never reached
                    if (!(g_dbg_fault == 1 && idx == 0 && kb == kb_begin + 1))
#endif
                    load_a(0, &mapA1);
                    if (!FB) load_b(B_OFF, &mapB1);
                    if (LOAD_LO) {
                        load_a(TILE_A_BYTES, &mapA2);
                        if (!FB) load_b(B_OFF + TILE_B_BYTES, &mapB2);
                    }
                    if (BF3) {
                        load_a(2 * TILE_A_BYTES, &mapA3);
                        load_b(B_OFF + 2 * TILE_B_BYTES, &mapB3);
                    }
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA; warp-uniform, one elected lane) ======
        // Per k-block the D_mid (and D_lo) MMAs are issued BEFORE waiting for the D_hi buffer, so
        // a promotion drain overlaps ~8 queued MMAs; at a tile start D_hi goes first (the
        // epilogue drains D_hi before D_mid).
        if (leader) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t cc = 0;       // global D_hi chunk counter
            uint32_t tc = 0;       // tile counter
            for (int unit = pair; unit < num_units; unit += num_pairs, tc++) {
                int tile_unused;
                int kb_begin, kb_end, slot;
                decode_unit(unit, up, num_kb, kps, tile_unused, kb_begin, kb_end, slot);
                const uint32_t t_mid = tmem_base + COL_MID;
                const uint32_t t_lo = tmem_base + COL_LO;
                bool mid_ready = false;
                int cpos = 0;      // k-block position inside the current D_hi chunk (no % on this path)
                for (int kb = kb_begin; kb < kb_end; kb++) {
                    const bool chunk_start = cpos == 0;
                    const bool chunk_end = cpos + 1 == promo_kb || kb + 1 == kb_end;
                    cpos = cpos + 1 == promo_kb ? 0 : cpos + 1;
                    if (chunk_start && kb > kb_begin) cc++;
                    const uint32_t hb = HB == 2 ? (cc & 1) : 0;
                    const uint32_t hphase = HB == 2 ? ((cc >> 1) & 1) : (cc & 1);
                    const uint32_t t_hi = tmem_base + hb * BN_;
                    mbar_wait(smem_u32(&full_bar[stage]), phase);
                    tc_fence_after();
                    uint8_t* st = smem + stage * STAGE_BYTES;
                    auto adesc = [&](int off) {
                        return AMN ? sdesc_mn_sw128(smem_u32(st + off), MN_BOX_BYTES) : sdesc_sw128(smem_u32(st + off));
                    };
                    const uint64_t a1 = adesc(0);
                    const uint64_t a2 = adesc(TILE_A_BYTES);
                    const uint64_t a3 = adesc(2 * TILE_A_BYTES);
                    auto bdesc = [&](int off) {
                        return FB ? (BMN ? sdesc_mn_sw128(smem_u32(st + off), FB_LBO)
                                         : sdesc_sw128(smem_u32(st + off), FBK_GROUP_BYTES))
                                  : BMN ? sdesc_mn_sw128(smem_u32(st + off), MN_BOX_BYTES) : sdesc_sw128(smem_u32(st + off));
                    };
                    const uint64_t b1 = bdesc(B_OFF);
                    const uint64_t b2 = bdesc(B_OFF + (FB ? (BMN ? FB_LO_OFF : FBK_LO_OFF) : TILE_B_BYTES));
                    const uint64_t b3 = bdesc(B_OFF + 2 * TILE_B_BYTES);
                    // D_hi first at both ends of a unit: at the start the epilogue frees D_hi before
                    // D_mid; at the end the last D_hi drain overlaps the last D_mid MMAs
                    const bool hi_first = kb == kb_begin || kb + 1 == kb_end;
                    auto issue_mid = [&]() {
                        if (!HAS_MID) return;
                        if (!mid_ready) {
                            mbar_wait(smem_u32(&mempty_bar[0]), (tc & 1) ^ 1);
                            tc_fence_after();
                            mid_ready = true;
                        }
                        if (elect_one()) {
#pragma unroll
                            for (int k = 0; k < BK / 16; k++) {
                                const uint64_t dk = DKA * k, dkb = DKB * k;
                                const uint32_t acc = (kb > kb_begin || k > 0) ? 1u : 0u;
                                mma_pair(t_mid, a1 + dk, b2 + dkb, IDESC, acc);
                                mma_pair(t_mid, a2 + dk, b1 + dkb, IDESC, 1u);
                                if (TERMS == 4) mma_pair(t_lo, a2 + dk, b2 + dkb, IDESC, acc);
                                if (BF3) {          // the 2^-16-weighted products share D_mid
                                    mma_pair(t_mid, a1 + dk, b3 + dkb, IDESC, 1u);
                                    mma_pair(t_mid, a2 + dk, b2 + dkb, IDESC, 1u);
                                    mma_pair(t_mid, a3 + dk, b1 + dkb, IDESC, 1u);
                                }
                            }
                        }
                        __syncwarp();
                    };
                    auto issue_hi = [&]() {
                        if (chunk_start) {
                            mbar_wait(smem_u32(&hempty_bar[hb]), hphase ^ 1);
                            tc_fence_after();
                        }
                        if (elect_one()) {
#pragma unroll
                            for (int k = 0; k < BK / 16; k++) {
                                const uint64_t dk = DKA * k, dkb = DKB * k;
                                mma_pair(t_hi, a1 + dk, b1 + dkb, IDESC, (!chunk_start || k > 0) ? 1u : 0u);
                            }
                            // D_hi chunk ready: the commit covers only MMAs issued so far, so with
                            // D_hi first the drain starts while this k-block's D_mid MMAs run
                            if (chunk_end) mma_commit_pair(smem_u32(&hfull_bar[hb]));
                        }
                        __syncwarp();
                    };
                    // Interleaved (3-term, inside a D_hi chunk, not a unit's last k-block: D_hi needs no
                    // wait and D_mid is already owned): per K = 16 step A1*B1 -> D_hi keeps A1 in the
                    // collector and A1*B2 -> D_mid reuses it, so A1 is read from shared memory once
                    // instead of twice.  Same accumulators, same per-accumulator order: same bits.
                    const bool interleave = TERMS == 3 && !BF3 && !FOLD && !chunk_start && kb + 1 != kb_end && mid_ready;
                    if (FOLD) {
                        // one k-block per chunk: T[hb] = [A2B2], then + A1B2 + A2B1 entered with
                        // T <- P + 2^-11 T, then + A1B1 likewise (every K = 16 step of a group
                        // before the next group: the 2^-11 applies to the whole lower group)
                        mbar_wait(smem_u32(&hempty_bar[hb]), hphase ^ 1);
                        tc_fence_after();
                        if (elect_one()) {
                            if (TERMS == 4) {
#pragma unroll
                                for (int k = 0; k < BK / 16; k++)
                                    mma_pair(t_hi, a2 + DKA * k, b2 + DKB * k, IDESC, k > 0 ? 1u : 0u);
                            }
#pragma unroll
                            for (int k = 0; k < BK / 16; k++) {
                                const uint64_t dk = DKA * k, dkb = DKB * k;
                                if (TERMS == 4 && k == 0) mma_pair_fold11(t_hi, a1 + dk, b2 + dkb, IDESC);
                                else mma_pair(t_hi, a1 + dk, b2 + dkb, IDESC, (TERMS == 4 || k > 0) ? 1u : 0u);
                                mma_pair(t_hi, a2 + dk, b1 + dkb, IDESC, 1u);
                            }
#pragma unroll
                            for (int k = 0; k < BK / 16; k++) {
                                if (k == 0) mma_pair_fold11(t_hi, a1, b1, IDESC);
                                else mma_pair(t_hi, a1 + DKA * k, b1 + DKB * k, IDESC, 1u);
                            }
                            mma_commit_pair(smem_u32(&hfull_bar[hb]));
                        }
                        __syncwarp();
                    } else if (interleave) {
                        if (elect_one()) {
#pragma unroll
                            for (int k = 0; k < BK / 16; k++) {
                                const uint64_t dk = DKA * k, dkb = DKB * k;
                                mma_pair_keep_a(t_hi, a1 + dk, b1 + dkb, IDESC, 1u);
                                mma_pair_reuse_a(t_mid, a1 + dk, b2 + dkb, IDESC, 1u);
                                mma_pair(t_mid, a2 + dk, b1 + dkb, IDESC, 1u);
                            }
                            if (chunk_end) mma_commit_pair(smem_u32(&hfull_bar[hb]));
                        }
                        __syncwarp();
                    } else if (hi_first) { issue_hi(); issue_mid(); } else { issue_mid(); issue_hi(); }
                    if (elect_one()) {
                        mma_commit_pair(smem_u32(&empty_bar[stage]));        // stage free in both CTAs
                        if (HAS_MID && kb + 1 == kb_end) mma_commit_pair(smem_u32(&mfull_bar[0]));
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                cc++;
                }
#if SPLIT3_DEBUG
            if (elect_one()) dbg_chunks = cc;
            __syncwarp();
#endif
        }
    } else if (FB && warp >= 2 + NUM_EPI_WARPS) {
        // ===================== fused-B converters (warps 10..11, both CTAs) ================
        // Per k-block: wait for the fp32 tile in the stage, split K steps cw and cw + 2 in place,
        // make the plane stores visible to the async proxy, arrive on the leader's full barrier.
        const int cw = warp - (2 + NUM_EPI_WARPS);
        const int sB = scale_exp_dev(*fb_maxB);
        const float f = pow2_neg(sB);
        if (fb_sB && blockIdx.x == 0 && cw == 0 && lane == 0) *fb_sB = sB;
        static_assert(NUM_CONV_WARPS == 2 && BK / 16 == 4, "two K steps per converter warp");
        int stage = 0;
        uint32_t phase = 0;
        for (int unit = pair; unit < num_units; unit += num_pairs) {
            int tile_unused;
            int kb_begin, kb_end, slot;
            decode_unit(unit, up, num_kb, kps, tile_unused, kb_begin, kb_end, slot);
            for (int kb = kb_begin; kb < kb_end; kb++) {
                mbar_wait(smem_u32(&ffull_bar[stage]), phase);
                uint8_t* breg = smem + stage * STAGE_BYTES + B_OFF;
                if (BMN) {
                    convert_step(breg + cw * FB_STEP_BYTES, lane, f);
                    convert_step(breg + (cw + 2) * FB_STEP_BYTES, lane, f);
                } else {
                    // groups cw, cw + 2, ... (8 per warp) in two passes of 4
                    static_assert(!FB || BNH / 8 == 8 * NUM_CONV_WARPS, "8 groups per converter warp");
                    convert_kgroups<4>(breg + cw * FBK_GROUP_BYTES, NUM_CONV_WARPS * FBK_GROUP_BYTES, lane, f);
                    convert_kgroups<4>(breg + (cw + 4 * NUM_CONV_WARPS) * FBK_GROUP_BYTES, NUM_CONV_WARPS * FBK_GROUP_BYTES,
                                       lane, f);
                }
                fence_async_smem();   // generic-proxy plane stores -> visible to the MMA (async proxy)
                __syncwarp();
                if (lane == 0) mbar_arrive_leader(smem_u32(&full_bar[stage]));
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else {
        // ===================== epilogue (warps 2..9, both CTAs) =====================
        // warp w reads TMEM lane quadrant (w % 4) and columns [NCOL * half, + NCOL).
        const int quad = warp & 3;
        const int half = (warp - 2) >> 2;
        const int sAB = *d_sA + (FB ? scale_exp_dev(*fb_maxB) : *d_sB);
        const bool fast = sAB >= -126 && sAB <= 127;
        const float fscale = fast ? __uint_as_float((unsigned)(sAB + 127) << 23) : 1.0f;
        // C = master * 2^sAB, exact unless the result is subnormal (one rounding); 2^sAB outside
        // the fp32 normal range goes through fp64 (exact factor, then one rounding to fp32).  Applied
        // as each value is stored, so no separate pass holds the whole master.
        auto scl = [&](float x) {
            return fast ? x * fscale
                        : __double2float_rn(__dmul_rn((double)x, __longlong_as_double((long long)(sAB + 1023) << 52)));
        };
        const uint32_t lane_base = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(half * NCOL);
        uint32_t cc = 0, tc = 0;
        for (int unit = pair; unit < num_units; unit += num_pairs, tc++) {
            int tile;
            int kb_begin, kb_end, slot;
            decode_unit(unit, up, num_kb, kps, tile, kb_begin, kb_end, slot);
            int mb, nb;
            tile_coords(tile, num_m, num_n, tune.group_m, mb, nb);
            float master[NCOL];
#pragma unroll
            for (int j = 0; j < NCOL; j++) master[j] = 0.0f;
            for (int kb0 = kb_begin; kb0 < kb_end; kb0 += promo_kb, cc++) {
                const uint32_t hb = HB == 2 ? (cc & 1) : 0;
                const uint32_t hphase = HB == 2 ? ((cc >> 1) & 1) : (cc & 1);
                mbar_wait(smem_u32(&hfull_bar[hb]), hphase);
                tc_fence_after();
                promote_all<NCOL>(lane_base + hb * BN_, master);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_leader(smem_u32(&hempty_bar[hb]));
            }
            if (HAS_MID) {
                mbar_wait(smem_u32(&mfull_bar[0]), tc & 1);
                tc_fence_after();
                if (TERMS == 4) {
#pragma unroll
                    for (int c = 0; c < NCOL / 16; c++) {
                        uint32_t mid[16], lo[16];
                        tmem_ld16(lane_base + COL_MID + c * 16, mid);
                        tmem_ld16(lane_base + COL_LO + c * 16, lo);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 16; j++)
                            master[c * 16 + j] = __fmaf_rn(
                                __fmaf_rn(__uint_as_float(lo[j]), 0x1p-11f, __uint_as_float(mid[j])), 0x1p-11f,
                                master[c * 16 + j]);
                    }
                } else {
                    // 8 columns per load: the 128-float master leaves few registers
#pragma unroll
                    for (int c = 0; c < NCOL / 8; c++) {
                        uint32_t mid[8];
                        tmem_ld8(lane_base + COL_MID + c * 8, mid);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 8; j++)
                            master[c * 8 + j] = BF3 ? __fadd_rn(master[c * 8 + j], __uint_as_float(mid[j]))   // bf16: C = D_hi + D_mid
                                                    : __fmaf_rn(__uint_as_float(mid[j]), 0x1p-11f, master[c * 8 + j]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_leader(smem_u32(&mempty_bar[0]));   // D_mid free early
            }
            if (slot >= 0) {                              // split tile: raw partial, reduced later
                // tile-local partial block (2*BM x BN_) of slot `slot`
                const int lr = crank * BM + quad * 32 + lane;
                float* prow = partial + ((int64_t)slot * (2 * BM) + lr) * BN_ + half * NCOL;
#pragma unroll
                for (int j = 0; j < NCOL / 4; j++)
                    reinterpret_cast<float4*>(prow)[j] =
                        make_float4(master[4 * j], master[4 * j + 1], master[4 * j + 2], master[4 * j + 3]);
                continue;
            }
            const int col0 = nb * BN_ + half * NCOL;
            if (tma_store) {
                // stage 32 rows x 32 columns per step (row = lane, 16-B chunks XOR-swizzled by
                // row % 8 as the map's SWIZZLE_128B expects: 4 wavefronts per warp store), then one
                // lane stores the box with TMA (clipped at M, N); the buffer is reused once the
                // previous store has read it.  tma_store == 2 (transposed C, the fused-A form
                // C^T = B^T A^T): the box is staged transposed — lane L writes its 32 values down
                // column L (one conflict-free wavefront per row) — and stored at (row, column)
                // swapped into the map of the caller's C.
                const uint32_t stg = smem_u32(staging + (warp - 2) * 4096);
                const int32_t r0 = (int32_t)(mb * 2 * BM + crank * BM + quad * 32);
#pragma unroll
                for (int c = 0; c < NCOL / 32; c++) {
                    if (lane == 0) bulk_wait_read0();
                    __syncwarp();
                    if (tma_store == 2) {
#pragma unroll
                        for (int j = 0; j < 32; j++)
                            st_shared_f32(stg + j * 128 + ((((lane >> 2) ^ (j & 7)) * 16) | ((lane & 3) * 4)),
                                          scl(master[c * 32 + j]));
                    } else {
#pragma unroll
                        for (int q = 0; q < 8; q++)
                            st_shared_v4(stg + lane * 128 + ((q ^ (lane & 7)) * 16), scl(master[c * 32 + 4 * q]),
                                         scl(master[c * 32 + 4 * q + 1]), scl(master[c * 32 + 4 * q + 2]),
                                         scl(master[c * 32 + 4 * q + 3]));
                    }
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (tma_store == 2) tma_store_2d(&mapC, stg, r0, (int32_t)(col0 + c * 32));
                        else tma_store_2d(&mapC, stg, (int32_t)(col0 + c * 32), r0);
                        bulk_commit();
                    }
                }
                continue;
            }
            // no TMA store (C not 16-B aligned, ldc % 4 != 0): the same 32 x 32 staging, then
            // each lane stores one column of the staged rows (coalesced rows, clipped at M, N)
            const uint32_t stg = smem_u32(staging + (warp - 2) * 4096);
            const int row0 = mb * 2 * BM + crank * BM + quad * 32;
#pragma unroll
            for (int c = 0; c < NCOL / 32; c++) {
#pragma unroll
                for (int q = 0; q < 8; q++)
                    st_shared_v4(stg + lane * 128 + ((q ^ (lane & 7)) * 16), scl(master[c * 32 + 4 * q]),
                                 scl(master[c * 32 + 4 * q + 1]), scl(master[c * 32 + 4 * q + 2]),
                                 scl(master[c * 32 + 4 * q + 3]));
                __syncwarp();
                const int col = col0 + c * 32 + lane;
                for (int r = 0; r < 32; r++) {
                    const float v = ld_shared_f32(stg + r * 128 + ((((lane >> 2) ^ (r & 7)) * 16) | ((lane & 3) * 4)));
                    if (row0 + r < M && col < N) C[(int64_t)(row0 + r) * ldc + col] = v;
                }
                __syncwarp();
            }
        }
    }

    if (warp >= 2 && warp < 2 + NUM_EPI_WARPS && tma_store && lane == 0) bulk_wait0();   // C stores done
#if SPLIT3_DEBUG
    uint32_t dbg_epi_chunks = 0;     // warp 2's drained D_hi chunk count (recomputed: same loop shape)
    if (warp == 2 && leader) {
        for (int unit = pair; unit < num_units; unit += num_pairs) {
            int tile_unused;
            int kb_begin, kb_end, slot;
            decode_unit(unit, up, num_kb, kps, tile_unused, kb_begin, kb_end, slot);
            dbg_epi_chunks += (uint32_t)((kb_end - kb_begin + promo_kb - 1) / promo_kb);
        }
    }
#endif
    tc_fence_before();
    cluster_sync();
#if SPLIT3_DEBUG
    if (warp == 2 && leader && lane == 0 && pair < num_units)
        DBG_CHECK(dbg_chunks == dbg_epi_chunks, 6, ((unsigned long long)dbg_chunks << 32) | dbg_epi_chunks);
#endif
    // Wave-lockstep counter reset: the last CTA to get here (exit ticket, word 3) zeroes the
    // counter, so every launch — eager or a CUDA-graph replay — starts from 0 with no memset.
    if (wave_counter && threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(wave_counter + 3, 1u) == gridDim.x - 1) {
#if SPLIT3_DEBUG
            // every producer announced each of its units but the first: 2 CTAs x (units - 1) per pair
            const int busy = num_units < num_pairs ? num_units : num_pairs;
            const unsigned expect = (unsigned)(2 * (num_units - busy));
            const unsigned got = atomicAdd(wave_counter, 0u);
            DBG_CHECK(got == expect, 7, ((unsigned long long)got << 32) | expect);
#endif
            atomicExch(wave_counter, 0u);
            atomicExch(wave_counter + 3, 0u);
        }
    }
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS)
                     : "memory");
    }
}

// Split-tile reduction: for each split tile t and element (r, c) of its 256 x BN block,
// C = 2^(sA+sB) * sum_{s=0}^{S-1} P[s*nsplit + t][r][c]  (fixed slice order -> deterministic).
// Launch: grid (2*BM / kReduceRows, nsplit), 256 threads; block (x, t) handles rows
// [x*kReduceRows, +kReduceRows) of split tile t, one float4 column group per thread per row.
constexpr int kReduceRows = 16;
__global__ void __launch_bounds__(256) ksplit_reduce_kernel(const float* __restrict__ P, SplitPlan plan, int bn,
                                                            int64_t M, int64_t N, int group_m,
                                                            float* __restrict__ C, int64_t ldc,
                                                            const int32_t* __restrict__ d_sA,
                                                            const int32_t* __restrict__ d_sB, int trans) {
    // trans (the fused-A form C^T = B^T A^T): the kernel's (row, col) is C's (col, row); the block's
    // kReduceRows x bn results go through shared memory so C's rows are written 64 B at a time
    __shared__ float tT[kReduceRows][256 + 1];
    pdl_enter();
    const int sAB = *d_sA + *d_sB;
    const bool fast = sAB >= -126 && sAB <= 127;
    const float f = fast ? __uint_as_float((unsigned)(sAB + 127) << 23) : 1.0f;
    const double fd = __longlong_as_double((long long)(sAB + 1023) << 52);
    auto scale = [&](float a) { return fast ? a * f : __double2float_rn(__dmul_rn((double)a, fd)); };
    const int64_t blk = (int64_t)(2 * BM) * bn;
    const int64_t t = blockIdx.y;
    const int64_t num_m = (M + 2 * BM - 1) / (2 * BM), num_n = (N + bn - 1) / bn;
    int mb, nb;
    tile_coords((int)(plan.whole + t), (int)num_m, (int)num_n, group_m, mb, nb);
    const int groups = bn / 4;                       // float4 column groups per row
    const int rows_per_pass = 256 / groups;
    const int g = threadIdx.x % groups;
    const int64_t col = (int64_t)nb * bn + 4 * g;
    const bool vec = (ldc % 4) == 0 && (reinterpret_cast<uintptr_t>(C) & 15u) == 0 && col + 4 <= N;
    for (int r = blockIdx.x * kReduceRows + threadIdx.x / groups; r < (int)(blockIdx.x + 1) * kReduceRows;
         r += rows_per_pass) {
        const int64_t row = (int64_t)mb * 2 * BM + r;
        if (row >= M || col >= N) continue;
        const int64_t e = (int64_t)r * bn + 4 * g;
        float4 acc = *reinterpret_cast<const float4*>(P + t * blk + e);
        for (int sl = 1; sl < plan.slices; sl++) {     // fixed slice order -> deterministic
            const float4 v = *reinterpret_cast<const float4*>(P + ((int64_t)sl * plan.nsplit + t) * blk + e);
            acc.x = __fadd_rn(acc.x, v.x); acc.y = __fadd_rn(acc.y, v.y);
            acc.z = __fadd_rn(acc.z, v.z); acc.w = __fadd_rn(acc.w, v.w);
        }
        if (trans) {
            const int rr = r - (int)blockIdx.x * kReduceRows;
            tT[rr][4 * g] = scale(acc.x); tT[rr][4 * g + 1] = scale(acc.y);
            tT[rr][4 * g + 2] = scale(acc.z); tT[rr][4 * g + 3] = scale(acc.w);
            continue;
        }
        float* dst = C + row * ldc + col;
        if (vec) {
            *reinterpret_cast<float4*>(dst) = make_float4(scale(acc.x), scale(acc.y), scale(acc.z), scale(acc.w));
        } else {
            const float a[4] = {acc.x, acc.y, acc.z, acc.w};
            for (int j = 0; j < 4 && col + j < N; j++) dst[j] = scale(a[j]);
        }
    }
    if (!trans) return;
    __syncthreads();
    const int rr = threadIdx.x % kReduceRows;
    const int64_t krow = (int64_t)mb * 2 * BM + blockIdx.x * kReduceRows + rr;   // C's column
    for (int cc = threadIdx.x / kReduceRows; cc < bn; cc += 256 / kReduceRows) {
        const int64_t kcol = (int64_t)nb * bn + cc;                            // C's row
        if (krow < M && kcol < N) C[kcol * ldc + krow] = tT[rr][cc];
    }
}

// ------------------------------------------------------------------ host side ---------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
    static const EncodeTiledFn fn = [] {   // thread-safe one-time lookup of the driver entry point
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<EncodeTiledFn>(p);
        return static_cast<EncodeTiledFn>(nullptr);
    }();
    return fn;
}

// 2-D map over C (fp32 row-major, M x N, ldc): 32 x 32 boxes, 128-B swizzle (the epilogue's
// staging layout).  Requires C 16-byte aligned and ldc % 4 == 0.
bool make_c_map(CUtensorMap* map, float* C, int64_t M, int64_t N, int64_t ldc) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)(ldc * 4)};
    cuuint32_t box[2] = {32, 32};
    const CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B;
    cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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

// 2-D map over an fp32 matrix (rows x cols, leading dimension ld elements), box box_cols x
// box_rows, no swizzle (the fused-B staging tile; the converters read it row by row).
bool make_f32_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols, int64_t ld, int box_cols,
                  int box_rows) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int TERMS, int BN_, int LAY>
int launch_t(cudaStream_t st, int64_t M, int64_t N, int64_t K, const CUtensorMap& a1,
             const CUtensorMap& a2, const CUtensorMap& b1, const CUtensorMap& b2, const CUtensorMap& a3,
             const CUtensorMap& b3, const CUtensorMap& mc, int tma_store,
             const int32_t* d_sA, const int32_t* d_sB, float* C, int64_t ldc, int num_sms,
             int promo_kb, unsigned* wave_counter, const GemmTune& tune, const SplitPlan& plan,
             float* partial, const float* fb_maxB, int32_t* fb_sB) {
    constexpr int SMEM_BYTES = Geo<BN_, TERMS == 6 ? 3 : 2>::SMEM;
    // the dynamic-smem opt-in is per device: remember it per device ordinal
    static std::atomic<uint64_t> attr_set{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_set.load() & bit)) {
        if (cudaFuncSetAttribute(gemm3_kernel<TERMS, BN_, LAY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 SMEM_BYTES) != cudaSuccess)
            return -1;
        attr_set.fetch_or(bit);
    }
    const int64_t tiles = plan.whole + plan.nsplit * plan.slices;   // work units
    const int64_t pairs = num_sms / 2;
    const int grid = 2 * (int)(tiles < pairs ? tiles : pairs);
    if (launch_k(gemm3_kernel<TERMS, BN_, LAY>, dim3((unsigned)grid), dim3(NThr<LAY>::v), SMEM_BYTES, st, a1, a2, b1,
                 b2, a3, b3, mc, tma_store, (int)M, (int)N, (int)K, promo_kb, d_sA, d_sB, C, ldc, wave_counter,
                 tune, plan, partial, fb_maxB, fb_sB) != cudaSuccess)
        return -1;
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

using LaunchFn = int (*)(cudaStream_t, int64_t, int64_t, int64_t, const CUtensorMap&, const CUtensorMap&,
                         const CUtensorMap&, const CUtensorMap&, const CUtensorMap&, const CUtensorMap&,
                         const CUtensorMap&, int, const int32_t*, const int32_t*, float*, int64_t, int, int,
                         unsigned*, const GemmTune&, const SplitPlan&, float*, const float*, int32_t*);

// the four operand layouts (mn bit 0: B MN-major, bit 1: A MN-major) of one kernel family
template <int TERMS, int BN_, int FB>
LaunchFn pick(int mn) {
    static constexpr LaunchFn table[4] = {launch_t<TERMS, BN_, FB | 0>, launch_t<TERMS, BN_, FB | 1>,
                                          launch_t<TERMS, BN_, FB | 2>, launch_t<TERMS, BN_, FB | 3>};
    return table[mn & 3];
}

}  // namespace

#if SPLIT3_DEBUG
namespace {
unsigned long long* g_dbg_host = nullptr;   // the mapped record (host view)
}
#endif

int gemm3_debug_init() {
#if SPLIT3_DEBUG
    if (g_dbg_host) return 1;
    void* p = nullptr;
    if (cudaHostAlloc(&p, 64, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) return -1;
    memset(p, 0, 64);
    void* d = nullptr;
    if (cudaHostGetDevicePointer(&d, p, 0) != cudaSuccess) return -1;
    if (cudaMemcpyToSymbol(g_dbg, &d, sizeof(d)) != cudaSuccess) return -1;
    g_dbg_host = static_cast<unsigned long long*>(p);
    return 1;
#else
    return 0;
#endif
}

int gemm3_debug_read(unsigned long long* out8, int reset) {
#if SPLIT3_DEBUG
    if (!g_dbg_host) {
        memset(out8, 0, 64);
        return 1;
    }
    volatile unsigned long long* r = g_dbg_host;   // host memory: readable after a device fault
    for (int i = 0; i < 8; i++) out8[i] = r[i];
    if (reset)
        for (int i = 0; i < 8; i++) r[i] = 0;
    return 1;
#else
    (void)out8; (void)reset;
    return 0;
#endif
}

int gemm3_debug_fault(int fault) {
#if SPLIT3_DEBUG
    return cudaMemcpyToSymbol(g_dbg_fault, &fault, sizeof(fault)) == cudaSuccess ? 1 : -1;
#else
    (void)fault;
    return 0;
#endif
}

SplitPlan gemm3_split_plan(int64_t M, int64_t N, int64_t K, int terms, int num_sms, int promo_kb, bool fold) {
    const int bn = (terms == 4 && !fold) ? 128 : 256;
    const int64_t tiles = ((M + 255) / 256) * ((N + bn - 1) / bn);
    const int64_t pairs = num_sms / 2;
    const int64_t num_kb = (K + 63) / 64;
    SplitPlan p;
    p.whole = tiles;
    p.nsplit = 0;
    p.slices = 1;
    if (tiles == 0 || pairs < 1) return p;
    const int promo = promo_kb > 0 ? promo_kb : kDefaultPromoKb;
    const int64_t max_by_k = num_kb / (promo > 4 ? promo : 4);   // >= 4 k-blocks per slice
    // tiles split along K: all of them when there is less than one wave, else the tail wave
    const int64_t rem = tiles < pairs ? tiles : tiles % pairs;
    if (rem == 0) return p;
    int64_t S = pairs / rem;
    if (S > max_by_k) S = max_by_k;
    if (S > 16) S = 16;
    if (S < 2) return p;
    const int64_t kps = (num_kb + S - 1) / S;
    S = (num_kb + kps - 1) / kps;              // every slice non-empty
    if (S < 2) return p;
    p.whole = tiles - rem;
    p.nsplit = rem;
    p.slices = (int)S;
    return p;
}

// Folded accumulator (LAY_FOLD): fold 1 = 4-term calls of at least 8192^3 multiply-adds (the
// power-capped regime: N = 16384 sustained +5.4 %; single 4096^3 .. 4096 x 8192^2 calls at
// higher clocks -2 .. -6 %, 8192^3 +1 %: profiles/fold_ab_*_r02.json, fold_bench_r02.json),
// 2 = every 3- and 4-term call (3-term: -1.6 % sustained).
bool gemm3_fold_chosen(int64_t M, int64_t N, int64_t K, int terms, int fold) {
    const bool big = (double)M * (double)N * (double)K >= 549755813888.0;   // 2^39 = 8192^3
    return (terms == 4 && (fold >= 2 || (fold == 1 && big))) || (terms == 3 && fold >= 2);
}

int64_t gemm3_partial_elems(const SplitPlan& p, int terms, bool fold) {
    const int bn = (terms == 4 && !fold) ? 128 : 256;
    return p.slices > 1 ? (int64_t)p.slices * p.nsplit * 256 * bn : 0;
}

int launch_gemm3(cudaStream_t st, int64_t M, int64_t N, int64_t K, const uint16_t* A1,
                 const uint16_t* A2, int64_t ldpa, const int32_t* d_sA, const uint16_t* B1t,
                 const uint16_t* B2t, int64_t ldpb, const int32_t* d_sB, float* C, int64_t ldc,
                 int terms, int num_sms, int promo_kb, unsigned* wave_counter, const GemmTuneIn& tin,
                 float* partial, int64_t partial_elems, int* err, const uint16_t* A3, const uint16_t* B3t,
                 int mn, const float* Bf, int64_t ldb, const float* d_maxB, int c_trans, int fold) {
    const bool fd = gemm3_fold_chosen(M, N, K, terms, fold);   // folded accumulator (LAY_FOLD)
    const int bn_t = (terms == 4 && !fd) ? 128 : 256;         // tile width
    const bool b_mn = (mn & 1) != 0, a_mn = (mn & 2) != 0;
    CUtensorMap ma1, ma2, mb1, mb2, ma3, mb3;
    if (Bf) {   // fused B (3-term): fp32 B map in place of the B plane maps
        if (terms != 3 || !d_maxB || (ldb % 4) != 0 || (reinterpret_cast<uintptr_t>(Bf) & 15u) != 0) {
            *err = 1;   // SPLIT3_ERR_INVALID_VALUE
            return -1;
        }
        B1t = B2t = nullptr;
    }
    const uint16_t* A2e = terms == 1 ? A1 : A2;
    const uint16_t* B2e = terms == 1 ? B1t : B2t;
    const int bnh = bn_t / 2;
    // B planes: K-major N x K (box 64 K x bnh N), or MN-major K x N (box 64 N x 64 K, bnh/64 per plane)
    auto map_b = [&](CUtensorMap* m, const uint16_t* p) {
        return b_mn ? make_plane_map(m, p, K, N, ldpb, BK) : make_plane_map(m, p, N, K, ldpb, bnh);
    };
    auto map_a = [&](CUtensorMap* m, const uint16_t* p) {
        return a_mn ? make_plane_map(m, p, K, M, ldpa, BK) : make_plane_map(m, p, M, K, ldpa, BM);
    };
    // fused B: row-major K x N fp32, box 128 N x 64 K
    const bool bmaps = Bf ? (b_mn ? make_f32_map(&mb1, Bf, K, N, ldb, bnh, BK) : make_f32_map(&mb1, Bf, N, K, ldb, BK, bnh))
                          : (map_b(&mb1, B1t) && map_b(&mb2, B2e));
    if (Bf) mb2 = mb1;
    if (!map_a(&ma1, A1) || !map_a(&ma2, A2e) || !bmaps) {
        *err = 4;   // SPLIT3_ERR_CUDA
        return -1;
    }
    if (terms == 6 && (!A3 || !B3t || !map_a(&ma3, A3) || !map_b(&mb3, B3t))) {
        *err = 4;
        return -1;
    }
    if (terms != 6) { ma3 = ma1; mb3 = mb1; }
    // TMA-store epilogue when C allows it (else per-thread float4 / scalar stores)
    CUtensorMap mc = ma1;
    int tma_store = 0;
    const bool c_tma_ok = (ldc % 4) == 0 && (reinterpret_cast<uintptr_t>(C) & 15u) == 0;
    if (c_trans) {   // the caller's C is N x M (this GEMM computes its transpose): TMA stores only
        if (!c_tma_ok) {
            *err = 1;   // SPLIT3_ERR_INVALID_VALUE
            return -1;
        }
        if (!make_c_map(&mc, C, N, M, ldc)) {
            *err = 4;
            return -1;
        }
        tma_store = 2;
    } else if (c_tma_ok && make_c_map(&mc, C, M, N, ldc)) {
        tma_store = 1;
    }
    const int promo = fd ? 1 : (promo_kb > 0 ? promo_kb : kDefaultPromoKb);   // fold: every k-block
    GemmTune tune;
    tune.group_m = tin.group_m > 0 ? tin.group_m : kDefaultGroupM;
    auto pol = [](int p) { return p == 1 ? kPolicyFirst : (p == 2 ? kPolicyLast : kPolicyNormal); };
    tune.pol_a = pol(tin.pol_a);
    tune.pol_b = pol(tin.pol_b);
    SplitPlan plan = gemm3_split_plan(M, N, K, terms, num_sms, promo, fd);
    // the kernel indexes work units and tiles in 32 bits (far above any matrix that fits in HBM)
    if (plan.whole + plan.nsplit * plan.slices > INT32_MAX || M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) {
        *err = 1;   // SPLIT3_ERR_INVALID_VALUE
        return -1;
    }
    if (plan.slices > 1 && (!partial || gemm3_partial_elems(plan, terms, fd) > partial_elems)) {
        plan.whole += plan.nsplit;   // no room for partials: whole tiles only
        plan.nsplit = 0;
        plan.slices = 1;
    }
    // instantiation table: TERMS x tile width x operand layout (LAY bits: B MN-major, A MN-major,
    // fused B)
    LaunchFn fn;
    if (terms == 1) fn = pick<1, 256, 0>(mn);
    else if (terms == 4) fn = fd ? pick<4, 256, LAY_FOLD>(mn) : pick<4, 128, 0>(mn);
    else if (terms == 6) fn = pick<6, 256, 0>(mn);
    else if (Bf) fn = fd ? pick<3, 256, LAY_FB | LAY_FOLD>(mn) : pick<3, 256, LAY_FB>(mn);
    else fn = fd ? pick<3, 256, LAY_FOLD>(mn) : pick<3, 256, 0>(mn);
    int r = fn(st, M, N, K, ma1, ma2, mb1, mb2, ma3, mb3, mc, tma_store, d_sA, d_sB, C, ldc, num_sms, promo,
               wave_counter, tune, plan, partial, Bf ? d_maxB : nullptr, Bf ? const_cast<int32_t*>(d_sB) : nullptr);
    if (r < 0) { *err = 4; return -1; }
    if (plan.slices > 1) {
        const int bn = bn_t;
        const dim3 grid((unsigned)(2 * BM / kReduceRows), (unsigned)plan.nsplit);
        launch_k(ksplit_reduce_kernel, grid, dim3(256), 0, st, partial, plan, bn, M, N, tune.group_m, C, ldc, d_sA, d_sB,
                 c_trans ? 1 : 0);
        if (cudaPeekAtLastError() != cudaSuccess) { *err = 4; return -1; }
        r += 1;
    }
    return r;
}

}  // namespace split3

