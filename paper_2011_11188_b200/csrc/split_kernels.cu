// split_kernels.cu — steps a1 (scale: max-abs) and a2 (split/encode) of the hot path.
//
// a1: m = max |x| over finite entries (the scale keeps A1/A2 "within the
//     limited dynamic range of fp16"; reading R1/R8 in DESIGN.md §3).  Order-independent and
//     exact: an atomicMax on the bit pattern of |x| (non-negative floats order like uints).
// a2: Eq. A_1: x' = x*2^-s (exact), A1 = RN16(x'), r = x' - A1 (exact in
//     fp32, DESIGN.md §3 R5), A2 = RN16(2^11 r)  (a2 = 2^-11 a1).
//     RN16 is cvt.rn.f16.f32 (round-to-nearest-even, subnormals kept: no FTZ in this TU).
//
// Both are HBM-bound streaming kernels: 4 B/el read for a1; 4 B/el read + 2x2 B/el written
// for a2.  float4 loads, grids sized in multiples of the SM count, grid-stride loops.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <climits>
#include <stdint.h>

#include "internal.h"
#include "split_math.h"

namespace split3 {
namespace {

constexpr unsigned kFiniteLimit = 0x7F800000u;   // |x| bits >= this: Inf or NaN

// Block-level reduction of the per-thread max (bits) and min bad index, one atomic each.
__device__ __forceinline__ void block_fold(unsigned m, long long bad, float* d_max, long long* d_bad) {
    __shared__ unsigned sm[32];
    __shared__ long long sb[32];
    for (int o = 16; o > 0; o >>= 1) {
        m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        bad = min(bad, (long long)__shfl_xor_sync(0xffffffffu, bad, o));
    }
    int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { sm[w] = m; sb[w] = bad; }
    __syncthreads();
    if (w == 0) {
        int nw = blockDim.x >> 5;
        m = l < nw ? sm[l] : 0u;
        bad = l < nw ? sb[l] : LLONG_MAX;
        for (int o = 16; o > 0; o >>= 1) {
            m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
            bad = min(bad, (long long)__shfl_xor_sync(0xffffffffu, bad, o));
        }
        if (l == 0) {
            if (m) atomicMax(reinterpret_cast<unsigned*>(d_max), m);
            if (d_bad && bad != LLONG_MAX) atomicMin(d_bad, bad);
        }
    }
}

__device__ __forceinline__ void fold_finite(float x, unsigned& m) {
    const unsigned u = __float_as_uint(x) & 0x7FFFFFFFu;
    if (u < kFiniteLimit) m = max(m, u);
}

__device__ __forceinline__ void fold1(float x, long long idx, unsigned& m, long long& bad) {
    unsigned u = __float_as_uint(x) & 0x7FFFFFFFu;
    if (u < kFiniteLimit) m = max(m, u);
    else bad = min(bad, idx);
}

// Contiguous (ld == cols) matrix viewed as n floats; VEC: 16-byte aligned base.
template <bool VEC>
__global__ void __launch_bounds__(256) maxabs_1d_kernel(const float* __restrict__ X, int64_t n,
                                                        float* d_max, long long* d_bad) {
    pdl_enter();
    unsigned m = 0;
    long long bad = LLONG_MAX;
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t done = 0;
    if (VEC) {
        const int64_t n4 = n / 4;
        const float4* X4 = reinterpret_cast<const float4*>(X);
        int64_t i = tid;
        for (; i + 3 * nthr < n4; i += 4 * nthr) {          // 4 independent 16-B loads in flight
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; u++) v[u] = __ldcs(X4 + i + u * nthr);
#pragma unroll
            for (int u = 0; u < 4; u++) {
                int64_t b = 4 * (i + u * nthr);
                fold1(v[u].x, b, m, bad); fold1(v[u].y, b + 1, m, bad);
                fold1(v[u].z, b + 2, m, bad); fold1(v[u].w, b + 3, m, bad);
            }
        }
        for (; i < n4; i += nthr) {
            float4 v = __ldcs(X4 + i);
            int64_t b = 4 * i;
            fold1(v.x, b, m, bad); fold1(v.y, b + 1, m, bad);
            fold1(v.z, b + 2, m, bad); fold1(v.w, b + 3, m, bad);
        }
        done = n4 * 4;
    }
    for (int64_t i = done + tid; i < n; i += nthr) fold1(__ldcs(X + i), i, m, bad);
    block_fold(m, bad, d_max, d_bad);
}

// Two contiguous matrices in one launch: blocks [0, gx) reduce X0, the rest X1.  Each block
// writes its max (bits of |x|) to partials[blockIdx.x]; the last block to finish (ticket) folds
// the partials into *d_max0 / *d_max1 and resets the ticket (threadfence-reduction pattern).
__global__ void __launch_bounds__(256) maxabs2_1d_kernel(const float* __restrict__ X0, int64_t n0, float* d_max0,
                                                         const float* __restrict__ X1, int64_t n1, float* d_max1,
                                                         int gx, unsigned* partials, unsigned* ticket) {
    pdl_enter();
    const bool first = (int)blockIdx.x < gx;
    const float* X = first ? X0 : X1;
    const int64_t n = first ? n0 : n1;
    const int64_t b = first ? blockIdx.x : blockIdx.x - gx;
    const int64_t nb = first ? gx : gridDim.x - gx;
    unsigned m = 0;
    long long bad = LLONG_MAX;
    const int64_t tid = b * blockDim.x + threadIdx.x;
    const int64_t nthr = nb * blockDim.x;
    const int64_t n4 = n / 4;
    const float4* X4 = reinterpret_cast<const float4*>(X);
    int64_t i = tid;
    for (; i + 3 * nthr < n4; i += 4 * nthr) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; u++) v[u] = __ldcs(X4 + i + u * nthr);
#pragma unroll
        for (int u = 0; u < 4; u++) {
            fold1(v[u].x, 0, m, bad); fold1(v[u].y, 0, m, bad);
            fold1(v[u].z, 0, m, bad); fold1(v[u].w, 0, m, bad);
        }
    }
    for (; i < n4; i += nthr) {
        float4 v = __ldcs(X4 + i);
        fold1(v.x, 0, m, bad); fold1(v.y, 0, m, bad); fold1(v.z, 0, m, bad); fold1(v.w, 0, m, bad);
    }
    for (int64_t j = n4 * 4 + tid; j < n; j += nthr) fold1(__ldcs(X + j), 0, m, bad);
    // block max -> partial
    __shared__ unsigned sm[32];
    __shared__ bool last;
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) sm[w] = m;
    __syncthreads();
    if (w == 0) {
        m = l < (int)(blockDim.x >> 5) ? sm[l] : 0u;
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (l == 0) {
            partials[blockIdx.x] = m;
            __threadfence();
            last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        }
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    unsigned m0 = 0, m1 = 0;
    for (int k = threadIdx.x; k < (int)gridDim.x; k += blockDim.x) {
        const unsigned v = __ldcg(partials + k);
        if (k < gx) m0 = max(m0, v);
        else m1 = max(m1, v);
    }
    for (int o = 16; o > 0; o >>= 1) {
        m0 = max(m0, __shfl_xor_sync(0xffffffffu, m0, o));
        m1 = max(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    }
    __shared__ unsigned s0[32], s1[32];
    if (l == 0) { s0[w] = m0; s1[w] = m1; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < (int)(blockDim.x >> 5); k++) { m0 = max(m0, s0[k]); m1 = max(m1, s1[k]); }
        m0 = max(m0, s0[0]);
        m1 = max(m1, s1[0]);
        *reinterpret_cast<unsigned*>(d_max0) = m0;
        *reinterpret_cast<unsigned*>(d_max1) = m1;
        *ticket = 0u;
    }
}

// Strided matrix: grid-stride over rows, threads over columns.
__global__ void __launch_bounds__(256) maxabs_2d_kernel(const float* __restrict__ X, int64_t rows,
                                                        int64_t cols, int64_t ld, float* d_max,
                                                        long long* d_bad) {
    pdl_enter();
    unsigned m = 0;
    long long bad = LLONG_MAX;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
        for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols;
             c += (int64_t)gridDim.x * blockDim.x)
            fold1(X[r * ld + c], r * cols + c, m, bad);
    block_fold(m, bad, d_max, d_bad);
}

// scale_exp_dev, pow2_neg, split1: split_math.h (shared with the fused-B GEMM converter)

// Host-buffer pipeline (split3_sgemm_host): max |x| and min nonzero |x| over the
// finite entries of a contiguous chunk, as uint bits (non-negative floats order like uints);
// *d_max must start at 0, *d_min at 0xFFFFFFFF (= no nonzero entry).
template <bool VEC>
__global__ void __launch_bounds__(256) maxmin_1d_kernel(const float* __restrict__ X, int64_t n, unsigned* d_max,
                                                        unsigned* d_min) {
    pdl_enter();
    unsigned mx = 0, mn = 0xFFFFFFFFu;
    auto fold = [&](float x) {
        const unsigned u = __float_as_uint(x) & 0x7FFFFFFFu;
        if (u < kFiniteLimit) {
            mx = max(mx, u);
            if (u) mn = min(mn, u);
        }
    };
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    int64_t done = 0;
    if (VEC) {
        const int64_t n4 = n / 4;
        const float4* X4 = reinterpret_cast<const float4*>(X);
        for (int64_t i = tid; i < n4; i += nthr) {
            const float4 v = __ldcs(X4 + i);
            fold(v.x); fold(v.y); fold(v.z); fold(v.w);
        }
        done = n4 * 4;
    }
    for (int64_t i = done + tid; i < n; i += nthr) fold(__ldcs(X + i));
    __shared__ unsigned sx[32], sn[32];
    for (int o = 16; o > 0; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { sx[w] = mx; sn[w] = mn; }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        mx = l < nw ? sx[l] : 0u;
        mn = l < nw ? sn[l] : 0xFFFFFFFFu;
        for (int o = 16; o > 0; o >>= 1) {
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (l == 0) {
            if (mx) atomicMax(d_max, mx);
            if (mn != 0xFFFFFFFFu) atomicMin(d_min, mn);
        }
    }
}

// Same for a strided rows x cols region (a column panel of a row-major matrix, ld >= cols).
template <bool VEC>
__global__ void __launch_bounds__(256) maxmin_2d_kernel(const float* __restrict__ X, int64_t rows, int64_t cols,
                                                        int64_t ld, unsigned* d_max, unsigned* d_min) {
    pdl_enter();
    unsigned mx = 0, mn = 0xFFFFFFFFu;
    auto fold = [&](float x) {
        const unsigned u = __float_as_uint(x) & 0x7FFFFFFFu;
        if (u < kFiniteLimit) {
            mx = max(mx, u);
            if (u) mn = min(mn, u);
        }
    };
    const int64_t units = VEC ? cols / 4 : cols;
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
        for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < units; c += (int64_t)gridDim.x * blockDim.x) {
            if (VEC) {
                const float4 v = __ldcs(reinterpret_cast<const float4*>(X + r * ld) + c);
                fold(v.x); fold(v.y); fold(v.z); fold(v.w);
            } else {
                fold(__ldcs(X + r * ld + c));
            }
        }
    __shared__ unsigned sx[32], sn[32];
    for (int o = 16; o > 0; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { sx[w] = mx; sn[w] = mn; }
    __syncthreads();
    if (w == 0) {
        const int nw = blockDim.x >> 5;
        mx = l < nw ? sx[l] : 0u;
        mn = l < nw ? sn[l] : 0xFFFFFFFFu;
        for (int o = 16; o > 0; o >>= 1) {
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (l == 0) {
            if (mx) atomicMax(d_max, mx);
            if (mn != 0xFFFFFFFFu) atomicMin(d_min, mn);
        }
    }
}

// After all row blocks: the per-matrix max (reading R1) and scale exponent sA from the block maxima;
// flags[b] = 1 iff block b was split with an exponent below sA AND holds a nonzero |x| < 2^(sA-12):
// only such an entry can round differently (fp16-subnormal A1 or A2), every other
// entry's planes, products and C are the global-scale ones times an exact power of two.
__global__ void host_scale_check_kernel(const unsigned* maxblk, const unsigned* minblk, const int32_t* sblk, int nblk,
                                        float* d_max, int32_t* d_sexp, int32_t* flags) {
    pdl_enter();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    unsigned g = 0;
    for (int b = 0; b < nblk; b++) g = max(g, maxblk[b]);
    const int s = scale_exp_dev(__uint_as_float(g));
    *d_max = __uint_as_float(g);
    *d_sexp = s;
    const int e = s - 12;                                   // in [-139, 101]
    const unsigned thr = e >= -126 ? (unsigned)(e + 127) << 23 : 1u << (e + 149);   // bits of 2^e
    for (int b = 0; b < nblk; b++) flags[b] = (sblk[b] != s && minblk[b] < thr) ? 1 : 0;
}


// Non-transposed split: planes rows x cols (ldp).  VEC: cols % 4 == 0, ld % 4 == 0, aligned.
template <bool VEC>
__global__ void __launch_bounds__(256) split_kernel(const float* __restrict__ X, int64_t rows,
                                                    int64_t cols, int64_t ld,
                                                    const float* __restrict__ d_max,
                                                    uint16_t* __restrict__ hi,
                                                    uint16_t* __restrict__ lo, int64_t ldp,
                                                    int32_t* d_sexp) {
    pdl_enter();
    const int s = scale_exp_dev(*d_max);
    const float f = pow2_neg(s);
    if (d_sexp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *d_sexp = s;
    if (VEC) {
        // U rows per iteration: U independent 16-B loads in flight per thread before any store
        constexpr int U = 4;
        const int64_t c4n = cols / 4;
        const int64_t gy = gridDim.y;
        for (int64_t r0 = blockIdx.y; r0 < rows; r0 += U * gy) {
            for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < c4n;
                 c += (int64_t)gridDim.x * blockDim.x) {
                float4 v[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int64_t r = r0 + u * gy;
                    if (r < rows) v[u] = __ldcs(reinterpret_cast<const float4*>(X + r * ld) + c);
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int64_t r = r0 + u * gy;
                    if (r < rows) {
                        unsigned short a[4], b[4];
                        split1(v[u].x, f, a[0], b[0]); split1(v[u].y, f, a[1], b[1]);
                        split1(v[u].z, f, a[2], b[2]); split1(v[u].w, f, a[3], b[3]);
                        __stcs(reinterpret_cast<uint2*>(hi + r * ldp) + c,
                               make_uint2(a[0] | ((unsigned)a[1] << 16), a[2] | ((unsigned)a[3] << 16)));
                        __stcs(reinterpret_cast<uint2*>(lo + r * ldp) + c,
                               make_uint2(b[0] | ((unsigned)b[1] << 16), b[2] | ((unsigned)b[3] << 16)));
                    }
                }
            }
        }
    } else {
        for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
            for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols;
                 c += (int64_t)gridDim.x * blockDim.x) {
                unsigned short a, b;
                split1(X[r * ld + c], f, a, b);
                hi[r * ldp + c] = a;
                lo[r * ldp + c] = b;
            }
    }
}

// Transposed split: X is rows x cols (row-major), planes are cols x rows (ldp >= rows), i.e.
// the K-major layout of B^T the GEMM reads.  64 x 64 tiles through shared memory (measured:
// 32 x 64 ties, 128 x 64 and N-fastest tile orders are slower): 256-B reads along X's rows,
// full 128-B lines written along the planes' rows; the next tile's loads are in flight while the
// current tile is stored.
template <bool VEC>
__global__ void __launch_bounds__(256) split_t_kernel(const float* __restrict__ X, int64_t rows,
                                                      int64_t cols, int64_t ld,
                                                      const float* __restrict__ d_max,
                                                      uint16_t* __restrict__ hi,
                                                      uint16_t* __restrict__ lo, int64_t ldp,
                                                      int32_t* d_sexp) {
    pdl_enter();
    constexpr int TK = 64, TN = 64;   // X rows (K) x X columns (N) per tile
    constexpr int TKP = TK + 2;       // halves per smem row (132 B: 4-B aligned, breaks the bank stride)
    __shared__ __align__(16) unsigned short s1[TN][TKP];
    __shared__ __align__(16) unsigned short s2[TN][TKP];
    const int s = scale_exp_dev(*d_max);
    const float f = pow2_neg(s);
    if (d_sexp && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *d_sexp = s;
    const int t = threadIdx.x;
    const int64_t ntr = (rows + TK - 1) / TK, ntc = (cols + TN - 1) / TN;
    const int64_t ntiles = ntr * ntc;
    // thread t covers the adjacent X rows rr, rr + 1 with rr = 2 (t/16) + 32 i (i < 2) and the
    // columns cc .. cc+3, cc = 4 (t%16): its two rows of a column pack into one 32-bit smem store.
    const int cc = 4 * (t % 16);
    float v[4][4];   // [2 i + row parity][column]
    auto load_tile = [&](int64_t tile) {
        const int64_t r0 = (tile % ntr) * TK, c0 = (tile / ntr) * TN;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int64_t r = r0 + 2 * (t / 16) + 32 * (q >> 1) + (q & 1), c = c0 + cc;
            v[q][0] = v[q][1] = v[q][2] = v[q][3] = 0.f;
            if (r < rows) {
                if (VEC && c + 3 < cols) {
                    float4 w = __ldcs(reinterpret_cast<const float4*>(X + r * ld + c));
                    v[q][0] = w.x; v[q][1] = w.y; v[q][2] = w.z; v[q][3] = w.w;
                } else {
#pragma unroll
                    for (int j = 0; j < 4; j++)
                        if (c + j < cols) v[q][j] = X[r * ld + c + j];
                }
            }
        }
    };
    int64_t tile = blockIdx.x;
    if (tile < ntiles) load_tile(tile);
    for (; tile < ntiles; tile += gridDim.x) {
        const int64_t r0 = (tile % ntr) * TK;   // consecutive blocks walk down X's rows (K)
        const int64_t c0 = (tile / ntr) * TN;
#pragma unroll
        for (int i = 0; i < 2; i++) {
            const int rr = 2 * (t / 16) + 32 * i;
#pragma unroll
            for (int j = 0; j < 4; j++) {
                unsigned short a0, b0, a1, b1;
                split1(v[2 * i][j], f, a0, b0);
                split1(v[2 * i + 1][j], f, a1, b1);
                *reinterpret_cast<unsigned*>(&s1[cc + j][rr]) = a0 | ((unsigned)a1 << 16);
                *reinterpret_cast<unsigned*>(&s2[cc + j][rr]) = b0 | ((unsigned)b1 << 16);
            }
        }
        __syncthreads();
        if (tile + gridDim.x < ntiles) load_tile(tile + gridDim.x);   // in flight during the stores
        // store: plane row n = c0 + t/4 gets K entries r0 + 16 (t%4) .. +15 (two 16-B chunks)
        {
            const int nn = t / 4, kk = 16 * (t % 4);
            const int64_t n = c0 + nn;
            if (n < cols) {
                const unsigned* p1 = reinterpret_cast<const unsigned*>(&s1[nn][kk]);
                const unsigned* p2 = reinterpret_cast<const unsigned*>(&s2[nn][kk]);
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int64_t k = r0 + kk + 8 * h;
                    if (k < ldp) {   // chunk lies inside the padded row (ldp % 8 == 0)
                        uint4 w1 = make_uint4(p1[4 * h], p1[4 * h + 1], p1[4 * h + 2], p1[4 * h + 3]);
                        uint4 w2 = make_uint4(p2[4 * h], p2[4 * h + 1], p2[4 * h + 2], p2[4 * h + 3]);
                        __stcs(reinterpret_cast<uint4*>(hi + n * ldp + k), w1);
                        __stcs(reinterpret_cast<uint4*>(lo + n * ldp + k), w2);
                    }
                }
            }
        }
        __syncthreads();
    }
}

// ---- one-launch front end for small problems (launch_prep2) -------------------------------
// Work item w of an operand = (row w / nseg, 1024-column segment w % nseg): 256 threads x float4.
__device__ __forceinline__ void prep_max(const PrepOperand& p, int64_t w0, int64_t wstep, unsigned& m) {
    const int64_t nseg = (p.cols + 1023) / 1024, items = p.rows * nseg;
    const bool vec = (p.cols % 4 == 0) && (p.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(p.X) & 15u) == 0);
    for (int64_t w = w0; w < items; w += wstep) {
        const int64_t r = w / nseg, c = (w - r * nseg) * 1024 + 4 * threadIdx.x;
        const float* row = p.X + r * p.ld;
        if (vec && c + 3 < p.cols) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(row + c));
            fold_finite(v.x, m); fold_finite(v.y, m); fold_finite(v.z, m); fold_finite(v.w, m);
        } else {
            for (int j = 0; j < 4 && c + j < p.cols; j++) fold_finite(row[c + j], m);
        }
    }
}
__device__ __forceinline__ void prep_split(const PrepOperand& p, float f, int64_t w0, int64_t wstep) {
    const int64_t nseg = (p.cols + 1023) / 1024, items = p.rows * nseg;
    const bool vec = (p.cols % 4 == 0) && (p.ld % 4 == 0) && ((reinterpret_cast<uintptr_t>(p.X) & 15u) == 0);
    for (int64_t w = w0; w < items; w += wstep) {
        const int64_t r = w / nseg, c = (w - r * nseg) * 1024 + 4 * threadIdx.x;
        const float* row = p.X + r * p.ld;
        if (vec && c + 3 < p.cols) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(row + c));
            unsigned short a[4], b[4];
            split1(v.x, f, a[0], b[0]); split1(v.y, f, a[1], b[1]);
            split1(v.z, f, a[2], b[2]); split1(v.w, f, a[3], b[3]);
            *reinterpret_cast<uint2*>(p.hi + r * p.ldp + c) = make_uint2(a[0] | ((unsigned)a[1] << 16), a[2] | ((unsigned)a[3] << 16));
            *reinterpret_cast<uint2*>(p.lo + r * p.ldp + c) = make_uint2(b[0] | ((unsigned)b[1] << 16), b[2] | ((unsigned)b[3] << 16));
        } else {
            for (int j = 0; j < 4 && c + j < p.cols; j++) {
                unsigned short a, b;
                split1(row[c + j], f, a, b);
                p.hi[r * p.ldp + c + j] = a;
                p.lo[r * p.ldp + c + j] = b;
            }
        }
    }
}

__global__ void __launch_bounds__(256) prep2_kernel(const PrepOperand pa, const PrepOperand pb,
                                                    unsigned* partials, unsigned* sync) {
    pdl_wait();
    __shared__ unsigned sm0[8], sm1[8];
    __shared__ bool last;
    unsigned* count = sync;
    unsigned* sense = sync + 1;
    unsigned my_sense = 0;
    if (threadIdx.x == 0) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(my_sense) : "l"(sense) : "memory");
    // phase 1 (a1): max-abs of both operands
    unsigned m0 = 0, m1 = 0;
    prep_max(pa, blockIdx.x, gridDim.x, m0);
    prep_max(pb, blockIdx.x, gridDim.x, m1);
    for (int o = 16; o > 0; o >>= 1) {
        m0 = max(m0, __shfl_xor_sync(0xffffffffu, m0, o));
        m1 = max(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    }
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) { sm0[w] = m0; sm1[w] = m1; }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < 8; k++) { m0 = max(m0, sm0[k]); m1 = max(m1, sm1[k]); }
        partials[2 * blockIdx.x] = m0;
        partials[2 * blockIdx.x + 1] = m1;
        __threadfence();
        last = atomicAdd(count, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {   // fold the partials, publish max and scale of both, release the barrier
        __threadfence();
        unsigned t0 = 0, t1 = 0;
        for (unsigned k = threadIdx.x; k < gridDim.x; k += blockDim.x) {
            t0 = max(t0, __ldcg(partials + 2 * k));
            t1 = max(t1, __ldcg(partials + 2 * k + 1));
        }
        for (int o = 16; o > 0; o >>= 1) {
            t0 = max(t0, __shfl_xor_sync(0xffffffffu, t0, o));
            t1 = max(t1, __shfl_xor_sync(0xffffffffu, t1, o));
        }
        __syncthreads();
        if (l == 0) { sm0[w] = t0; sm1[w] = t1; }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 0; k < 8; k++) { t0 = max(t0, sm0[k]); t1 = max(t1, sm1[k]); }
            *reinterpret_cast<unsigned*>(pa.d_max) = t0;
            *reinterpret_cast<unsigned*>(pb.d_max) = t1;
            *pa.d_sexp = scale_exp_dev(__uint_as_float(t0));
            *pb.d_sexp = scale_exp_dev(__uint_as_float(t1));
            *count = 0u;
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(sense), "r"(my_sense ^ 1u) : "memory");
        }
    } else if (threadIdx.x == 0) {   // grid-wide barrier (all blocks co-resident: cooperative launch)
        unsigned v;
        do {
            __nanosleep(32);
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sense) : "memory");
        } while (v == my_sense);
    }
    __syncthreads();
    pdl_trigger();
    // phase 2 (a2): both splits with the exact scales
    const float fa = pow2_neg(scale_exp_dev(__ldcg(pa.d_max)));
    const float fb = pow2_neg(scale_exp_dev(__ldcg(pb.d_max)));
    prep_split(pa, fa, blockIdx.x, gridDim.x);
    prep_split(pb, fb, blockIdx.x, gridDim.x);
}

// ---- bf16 x 3 split: x = X1 + X2 + X3, X_i = RN_bf16 of the running
// residual (exact in fp32); no scale (bfloat16 has the range of fp32).
__device__ __forceinline__ void split_bf3(float x, unsigned short& h1, unsigned short& h2, unsigned short& h3) {
    __nv_bfloat16 a = __float2bfloat16_rn(x);
    float r1 = __fsub_rn(x, __bfloat162float(a));
    __nv_bfloat16 b = __float2bfloat16_rn(r1);
    float r2 = __fsub_rn(r1, __bfloat162float(b));
    __nv_bfloat16 c = __float2bfloat16_rn(r2);
    h1 = __bfloat16_as_ushort(a);
    h2 = __bfloat16_as_ushort(b);
    h3 = __bfloat16_as_ushort(c);
}

// planes rows x cols (ldp), grid-stride over elements (row-major)
__global__ void __launch_bounds__(256) split_bf3_kernel(const float* __restrict__ X, int64_t rows, int64_t cols,
                                                        int64_t ld, uint16_t* __restrict__ p1,
                                                        uint16_t* __restrict__ p2, uint16_t* __restrict__ p3,
                                                        int64_t ldp) {
    pdl_enter();
    for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
        for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x) {
            unsigned short a, b, d;
            split_bf3(__ldcs(X + r * ld + c), a, b, d);
            p1[r * ldp + c] = a;
            p2[r * ldp + c] = b;
            p3[r * ldp + c] = d;
        }
}

// planes cols x rows (transposed, ldp >= rows) through 64 x 64 shared-memory tiles
__global__ void __launch_bounds__(256) split_bf3_t_kernel(const float* __restrict__ X, int64_t rows, int64_t cols,
                                                          int64_t ld, uint16_t* __restrict__ p1,
                                                          uint16_t* __restrict__ p2, uint16_t* __restrict__ p3,
                                                          int64_t ldp) {
    pdl_enter();
    __shared__ __align__(16) unsigned short sm[3][64][66];
    const int t = threadIdx.x;
    const int64_t ntr = (rows + 63) / 64, ntc = (cols + 63) / 64;
    for (int64_t tile = blockIdx.x; tile < ntr * ntc; tile += gridDim.x) {
        const int64_t r0 = (tile % ntr) * 64, c0 = (tile / ntr) * 64;
#pragma unroll
        for (int i = 0; i < 16; i++) {          // 64 x 64 elements, 16 per thread, coalesced along X's rows
            const int rr = (t / 64) + 4 * i, cc = t % 64;
            const int64_t r = r0 + rr, c = c0 + cc;
            const float x = (r < rows && c < cols) ? X[r * ld + c] : 0.0f;
            unsigned short a, b, d;
            split_bf3(x, a, b, d);
            sm[0][cc][rr] = a;
            sm[1][cc][rr] = b;
            sm[2][cc][rr] = d;
        }
        __syncthreads();
        const int nn = t / 4, kk = 16 * (t % 4);
        const int64_t n = c0 + nn;
        if (n < cols) {
#pragma unroll
            for (int p = 0; p < 3; p++) {
                uint16_t* dst = p == 0 ? p1 : (p == 1 ? p2 : p3);
                const unsigned* src = reinterpret_cast<const unsigned*>(&sm[p][nn][kk]);
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int64_t k = r0 + kk + 8 * h;
                    if (k < ldp)
                        __stcs(reinterpret_cast<uint4*>(dst + n * ldp + k),
                               make_uint4(src[4 * h], src[4 * h + 1], src[4 * h + 2], src[4 * h + 3]));
                }
            }
        }
        __syncthreads();
    }
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

inline int grid_rows(int64_t rows, int num_sms, int64_t blocks_x) {
    int64_t want = (int64_t)num_sms * 8 / (blocks_x > 0 ? blocks_x : 1);
    if (want < 1) want = 1;
    if (want > rows) want = rows;
    if (want > 65535) want = 65535;
    return (int)want;
}

}  // namespace

int launch_prep2(cudaStream_t st, const PrepOperand& a, const PrepOperand& b, unsigned* partials,
                 unsigned* sync, int num_sms) {
    auto items = [](const PrepOperand& p) { return p.rows * ((p.cols + 1023) / 1024); };
    int64_t g = items(a) > items(b) ? items(a) : items(b);
    const int64_t cap = (int64_t)num_sms * 2;   // far below the co-residency limit (8 blocks / SM)
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    const cudaError_t e = launch_k_coop(prep2_kernel, dim3((unsigned)g), dim3(256), 0, st, a, b, partials, sync);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();   // launch-configuration error (not sticky): caller falls back
        return -2;
    }
    return 1;
}

int launch_maxabs(cudaStream_t st, int64_t rows, int64_t cols, const float* X, int64_t ld,
                  float* d_max, long long* d_bad, int num_sms) {
    if (rows <= 0 || cols <= 0) return 0;
    if (ld == cols) {
        int64_t n = rows * cols;
        int64_t blocks = (n / 4 + 255) / 256;
        int64_t cap = (int64_t)num_sms * 8;
        int g = (int)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
        if (aligned16(X)) launch_k(maxabs_1d_kernel<true>, dim3(g), dim3(256), 0, st, X, n, d_max, d_bad);
        else launch_k(maxabs_1d_kernel<false>, dim3(g), dim3(256), 0, st, X, n, d_max, d_bad);
    } else {
        int64_t bx = (cols + 255) / 256;
        if (bx > 64) bx = 64;
        dim3 grid((unsigned)bx, (unsigned)grid_rows(rows, num_sms, bx));
        launch_k(maxabs_2d_kernel, grid, dim3(256), 0, st, X, rows, cols, ld, d_max, d_bad);
    }
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_maxmin(cudaStream_t st, int64_t n, const float* X, unsigned* d_max, unsigned* d_min, int num_sms) {
    if (n <= 0) return 0;
    int64_t blocks = (n / 4 + 255) / 256;
    const int64_t cap = (int64_t)num_sms * 8;
    const int g = (int)(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
    if (aligned16(X)) launch_k(maxmin_1d_kernel<true>, dim3(g), dim3(256), 0, st, X, n, d_max, d_min);
    else launch_k(maxmin_1d_kernel<false>, dim3(g), dim3(256), 0, st, X, n, d_max, d_min);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_maxmin2d(cudaStream_t st, int64_t rows, int64_t cols, const float* X, int64_t ld, unsigned* d_max,
                    unsigned* d_min, int num_sms) {
    if (rows <= 0 || cols <= 0) return 0;
    if (ld == cols) return launch_maxmin(st, rows * cols, X, d_max, d_min, num_sms);
    const bool vec = (cols % 4 == 0) && (ld % 4 == 0) && aligned16(X);
    const int64_t units = vec ? cols / 4 : cols;
    int64_t bx = (units + 255) / 256;
    if (bx > 64) bx = 64;
    dim3 grid((unsigned)bx, (unsigned)grid_rows(rows, num_sms, bx));
    if (vec) launch_k(maxmin_2d_kernel<true>, grid, dim3(256), 0, st, X, rows, cols, ld, d_max, d_min);
    else launch_k(maxmin_2d_kernel<false>, grid, dim3(256), 0, st, X, rows, cols, ld, d_max, d_min);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_host_scale_check(cudaStream_t st, const unsigned* maxblk, const unsigned* minblk, const int32_t* sblk,
                            int nblk, float* d_max, int32_t* d_sexp, int32_t* flags) {
    launch_k(host_scale_check_kernel, dim3(1), dim3(32), 0, st, maxblk, minblk, sblk, nblk, d_max, d_sexp, flags);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_maxabs2(cudaStream_t st, int64_t rows0, int64_t cols0, const float* X0, int64_t ld0, float* d_max0,
                   int64_t rows1, int64_t cols1, const float* X1, int64_t ld1, float* d_max1, int num_sms,
                   float* partials, int max_parts, unsigned* ticket) {
    const bool ok = ld0 == cols0 && ld1 == cols1 && aligned16(X0) && aligned16(X1) && rows0 > 0 && cols0 > 0 &&
                    rows1 > 0 && cols1 > 0 && partials && ticket;
    if (!ok) {
        if (cudaMemsetAsync(d_max0, 0, 4, st) != cudaSuccess || cudaMemsetAsync(d_max1, 0, 4, st) != cudaSuccess)
            return -1;
        int a = launch_maxabs(st, rows0, cols0, X0, ld0, d_max0, nullptr, num_sms);
        if (a < 0) return -1;
        int b = launch_maxabs(st, rows1, cols1, X1, ld1, d_max1, nullptr, num_sms);
        return b < 0 ? -1 : a + b;
    }
    const int64_t n0 = rows0 * cols0, n1 = rows1 * cols1;
    int64_t total_blocks = (int64_t)num_sms * 8;
    if (total_blocks > max_parts) total_blocks = max_parts;
    int64_t g0 = (int64_t)((double)total_blocks * (double)n0 / (double)(n0 + n1));
    int64_t need0 = (n0 / 4 + 255) / 256, need1 = (n1 / 4 + 255) / 256;
    if (g0 > need0) g0 = need0;
    if (g0 < 1) g0 = 1;
    int64_t g1 = total_blocks - g0;
    if (g1 > need1) g1 = need1;
    if (g1 < 1) g1 = 1;
    launch_k(maxabs2_1d_kernel, dim3((unsigned)(g0 + g1)), dim3(256), 0, st, X0, n0, d_max0, X1, n1, d_max1, (int)g0,
             reinterpret_cast<unsigned*>(partials), ticket);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_split(cudaStream_t st, int64_t rows, int64_t cols, const float* X, int64_t ld,
                 const float* d_max, uint16_t* hi, uint16_t* lo, int64_t ldp, int32_t* d_sexp,
                 int num_sms) {
    if (rows <= 0 || cols <= 0) return 0;
    const bool vec = (cols % 4 == 0) && (ld % 4 == 0) && aligned16(X);
    const int64_t units = vec ? cols / 4 : cols;
    int64_t bx = (units + 255) / 256;
    if (bx > 64) bx = 64;
    dim3 grid((unsigned)bx, (unsigned)grid_rows(rows, num_sms, bx));
    if (vec) launch_k(split_kernel<true>, grid, dim3(256), 0, st, X, rows, cols, ld, d_max, hi, lo, ldp, d_sexp);
    else launch_k(split_kernel<false>, grid, dim3(256), 0, st, X, rows, cols, ld, d_max, hi, lo, ldp, d_sexp);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_split_bf16x3(cudaStream_t st, int64_t rows, int64_t cols, const float* X, int64_t ld, uint16_t* p1,
                        uint16_t* p2, uint16_t* p3, int64_t ldp, int transpose, int num_sms) {
    if (rows <= 0 || cols <= 0) return 0;
    if (transpose) {
        int64_t tiles = ((rows + 63) / 64) * ((cols + 63) / 64);
        int64_t cap = (int64_t)num_sms * 8;
        launch_k(split_bf3_t_kernel, dim3((unsigned)(tiles < cap ? tiles : cap)), dim3(256), 0, st, X, rows, cols, ld, p1, p2, p3, ldp);
    } else {
        int64_t bx = (cols + 255) / 256;
        if (bx > 64) bx = 64;
        dim3 grid((unsigned)bx, (unsigned)grid_rows(rows, num_sms, bx));
        launch_k(split_bf3_kernel, grid, dim3(256), 0, st, X, rows, cols, ld, p1, p2, p3, ldp);
    }
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_split_t(cudaStream_t st, int64_t rows, int64_t cols, const float* X, int64_t ld,
                   const float* d_max, uint16_t* hi, uint16_t* lo, int64_t ldp, int32_t* d_sexp,
                   int num_sms) {
    if (rows <= 0 || cols <= 0) return 0;
    const bool vec = (ld % 4 == 0) && aligned16(X);
    int64_t tiles = ((rows + 63) / 64) * ((cols + 63) / 64);
    int64_t cap = (int64_t)num_sms * 8;
    int g = (int)(tiles < cap ? tiles : cap);
    if (vec) launch_k(split_t_kernel<true>, dim3(g), dim3(256), 0, st, X, rows, cols, ld, d_max, hi, lo, ldp, d_sexp);
    else launch_k(split_t_kernel<false>, dim3(g), dim3(256), 0, st, X, rows, cols, ld, d_max, hi, lo, ldp, d_sexp);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace split3
