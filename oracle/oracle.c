/*
 * oracle.c — CPU oracle for the split-FP16 SGEMM of arXiv 2011.11188, Appendix A.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2011_11188_b200/, include/).
 *
 * Plain, slow, obviously-correct C.  All floating-point arithmetic of the method is
 * done in fp64 (binary64).  Each function cites the passage of the paper it follows
 * ("PAPER.md:L" = line L of /root/reference/PAPER.md) and the DESIGN.md reading used
 * where the paper is silent (R1..R9 in DESIGN.md §3).
 *
 * Layout conventions: matrices are row-major with a leading dimension (elements).
 * FP16 values are carried as uint16_t bit patterns (IEEE binary16).
 *
 * Parity pins for every function live in tests/test_oracle_*.py (marker "not gpu").
 */
#include <stdint.h>
#include <string.h>
#include <math.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ------------------------------------------------------------------------------
 * binary16 encode, bit by bit, round-to-nearest-ties-to-even (reading R4).
 * Input is an fp64 value, so the encoder is a single rounding from the exact
 * input (no double rounding for any fp32 or fp64 input).
 * PAPER.md:4-8 (Eq. A_1: "A1_16", "A2_16" are FP16 matrices)
 * ("16-bit IEEE half-precision format (fp16)").  Subnormals are kept; overflow
 * goes to +-inf; NaN -> 0x7E00 (canonical quiet NaN, reading R4).
 * ---------------------------------------------------------------------------- */
uint16_t orc_enc16(double x)
{
    uint64_t b;
    memcpy(&b, &x, sizeof b);
    uint16_t sign = (uint16_t)((b >> 63) << 15);
    int e = (int)((b >> 52) & 0x7FF);
    uint64_t mant = b & ((1ULL << 52) - 1);

    if (e == 0x7FF)                     /* inf or NaN */
        return mant ? (uint16_t)0x7E00 : (uint16_t)(sign | 0x7C00);
    if (e == 0)                         /* zero or fp64-subnormal: |x| < 2^-1022 << 2^-25 */
        return sign;

    int E = e - 1023;                   /* unbiased exponent: |x| = sig * 2^(E-52) */
    uint64_t sig = (1ULL << 52) | mant; /* 53-bit significand */

    if (E > 15)                         /* |x| >= 2^16 > 65520: overflow */
        return (uint16_t)(sign | 0x7C00);

    if (E >= -14) {
        /* normal binary16 range: keep 11 significant bits (1 hidden + 10) */
        int shift = 52 - 10;
        uint64_t q = sig >> shift;
        uint64_t rem = sig & ((1ULL << shift) - 1);
        uint64_t half = 1ULL << (shift - 1);
        if (rem > half || (rem == half && (q & 1)))
            q++;
        if (q == 2048) {                /* mantissa carry into the exponent */
            q = 1024;
            E++;
        }
        if (E > 15)
            return (uint16_t)(sign | 0x7C00);
        return (uint16_t)(sign | (uint16_t)((E + 15) << 10) | (uint16_t)(q & 0x3FF));
    }

    /* subnormal binary16: integer multiple q of 2^-24;  q = sig * 2^(E-52+24) */
    int shift = 28 - E;                 /* >= 43 */
    if (shift > 54)                     /* |x| < 2^-25: rounds to zero (no tie possible) */
        return sign;
    uint64_t q = sig >> shift;
    uint64_t rem = sig & ((1ULL << shift) - 1);
    uint64_t half = 1ULL << (shift - 1);
    if (rem > half || (rem == half && (q & 1)))
        q++;
    /* q == 1024 is exactly the smallest normal 0x0400: the encoding is continuous */
    return (uint16_t)(sign | (uint16_t)q);
}

/* binary16 decode: exact value as fp64.  PAPER.md:278-280. */
double orc_dec16(uint16_t h)
{
    int sign = (h >> 15) & 1;
    int e = (h >> 10) & 0x1F;
    int m = h & 0x3FF;
    double v;
    if (e == 0)
        v = ldexp((double)m, -24);
    else if (e == 31)
        v = m ? NAN : INFINITY;
    else
        v = ldexp((double)(1024 + m), e - 25);
    return sign ? -v : v;
}

void orc_enc16_array(int64_t n, const double *x, uint16_t *h)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        h[i] = orc_enc16(x[i]);
}

void orc_enc16_f32_array(int64_t n, const float *x, uint16_t *h)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        h[i] = orc_enc16((double)x[i]);
}

void orc_dec16_array(int64_t n, const uint16_t *h, double *x)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        x[i] = orc_dec16(h[i]);
}

/* ------------------------------------------------------------------------------
 * Scale (reading R1).  The paper states the purpose only: "Scaling by a1_32
 * (a2_32) ensures A1_16 (A2_16) is within the limited dynamic range of fp16"
 * and "If A_32 is already well scaled, then one can expect
 * a1_32 = 1 and a2_32 = 2^-11 * a1_32".  Reading R1:
 *     m = max |x| over finite entries,
 *     s = 0 if m == 0 else max(E(m) - 14, -127),  E(m) = floor(log2 m),
 *     a1 = 2^s, a2 = 2^(s-11)  (a2 = 2^-11 a1).
 * ---------------------------------------------------------------------------- */
int orc_scale_exp(double m)
{
    if (m == 0.0)
        return 0;
    int e;
    frexp(m, &e);                       /* m = f * 2^e, f in [0.5, 1) -> E(m) = e - 1 */
    int s = (e - 1) - 14;
    return s < -127 ? -127 : s;
}

/* max |x| over finite entries (exact; order-free).  Returns the first non-finite
 * linear index (row*cols + col) or -1 if all entries are finite. */
int64_t orc_maxabs(int64_t rows, int64_t cols, const float *X, int64_t ld, double *out)
{
    double m = 0.0;
    int64_t bad = -1;
    for (int64_t i = 0; i < rows; i++) {
        for (int64_t j = 0; j < cols; j++) {
            double v = fabs((double)X[i * ld + j]);
            if (isfinite(v)) {
                if (v > m)
                    m = v;
            } else if (bad < 0) {
                bad = i * cols + j;
            }
        }
    }
    *out = m;
    return bad;
}

/* ------------------------------------------------------------------------------
 * Two-term split, Eq. A_1 / Eq. (1):
 *     x' = x * 2^-s                 (exact)
 *     A1 = RN16(x')                 (A1 holds the leading digits)
 *     r  = x' - dec(A1)             (exact in fp64)
 *     A2 = RN16(2^11 * r)           (a2 = 2^-11 a1)
 * so that x ~= a1*A1 + a2*A2 with a1 = 2^s, a2 = 2^(s-11).
 * hi/lo are row-major with leading dimension ldp.
 * ---------------------------------------------------------------------------- */
void orc_split(int64_t rows, int64_t cols, const float *X, int64_t ld, int s,
               uint16_t *hi, uint16_t *lo, int64_t ldp)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; i++) {
        for (int64_t j = 0; j < cols; j++) {
            double xs = ldexp((double)X[i * ld + j], -s);
            uint16_t h1 = orc_enc16(xs);
            double r = xs - orc_dec16(h1);
            uint16_t h2 = orc_enc16(ldexp(r, 11));
            hi[i * ldp + j] = h1;
            lo[i * ldp + j] = h2;
        }
    }
}

/* reconstruction a1*A1 + a2*A2 in fp64 (right-hand side of Eq. A_1) */
void orc_reconstruct(int64_t rows, int64_t cols, const uint16_t *hi, const uint16_t *lo,
                     int64_t ldp, int s, double *out, int64_t ldo)
{
    for (int64_t i = 0; i < rows; i++)
        for (int64_t j = 0; j < cols; j++)
            out[i * ldo + j] = ldexp(orc_dec16(hi[i * ldp + j]), s)
                             + ldexp(orc_dec16(lo[i * ldp + j]), s - 11);
}

/* ------------------------------------------------------------------------------
 * FP64 reference GEMM C64 = A*B (no splitting).  fp32*fp32 products are exact in
 * fp64; sums in fp64, naive i-k-j order.  The "C_32 = A_32 * B_32" of PAPER.md:9.
 * ---------------------------------------------------------------------------- */
void orc_gemm64(int64_t M, int64_t N, int64_t K, const float *A, int64_t lda,
                const float *B, int64_t ldb, double *C, int64_t ldc)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < M; i++) {
        double *c = C + i * ldc;
        for (int64_t j = 0; j < N; j++)
            c[j] = 0.0;
        for (int64_t k = 0; k < K; k++) {
            double a = (double)A[i * lda + k];
            const float *b = B + k * ldb;
            for (int64_t j = 0; j < N; j++)
                c[j] += a * (double)b[j];
        }
    }
}

/* ------------------------------------------------------------------------------
 * Split product, Eq. A_2 with the dropped term:
 *     T11 = A1*B1,  Tm = A1*B2 + A2*B1,  T22 = A2*B2      (products exact, fp64 sums)
 *     C   = 2^(sA+sB) * (T11 + 2^-11 * Tm [+ 2^-22 * T22])
 * The coefficients follow from a1b1 = 2^(sA+sB), a1b2 = a2b1 = 2^-11 a1b1 and
 * a2b2 = 2^-22 a1b1.  terms = 1 (A1B1 only: the "naive FP16"
 * control), 3 (default: "3 matrix multiplies in FP16") or 4 (Eq. A_2
 * in full).  A planes are M x K row-major (ldpa), B planes K x N row-major (ldpb).
 * ---------------------------------------------------------------------------- */
void orc_split_gemm(int64_t M, int64_t N, int64_t K,
                    const uint16_t *A1, const uint16_t *A2, int64_t ldpa, int sA,
                    const uint16_t *B1, const uint16_t *B2, int64_t ldpb, int sB,
                    int terms, double *C, int64_t ldc)
{
    #pragma omp parallel
    {
        double *t11 = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
        double *tm  = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
        double *t22 = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
        double *b1  = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
        double *b2  = (double *)malloc(sizeof(double) * (size_t)(N > 0 ? N : 1));
        #pragma omp for schedule(dynamic, 1)
        for (int64_t i = 0; i < M; i++) {
            for (int64_t j = 0; j < N; j++)
                t11[j] = tm[j] = t22[j] = 0.0;
            for (int64_t k = 0; k < K; k++) {
                double a1 = orc_dec16(A1[i * ldpa + k]);
                double a2 = orc_dec16(A2[i * ldpa + k]);
                for (int64_t j = 0; j < N; j++) {
                    b1[j] = orc_dec16(B1[k * ldpb + j]);
                    b2[j] = orc_dec16(B2[k * ldpb + j]);
                }
                for (int64_t j = 0; j < N; j++) {
                    t11[j] += a1 * b1[j];
                    tm[j]  += a1 * b2[j] + a2 * b1[j];
                    t22[j] += a2 * b2[j];
                }
            }
            for (int64_t j = 0; j < N; j++) {
                double v = t11[j];
                if (terms >= 3)
                    v += ldexp(tm[j], -11);
                if (terms >= 4)
                    v += ldexp(t22[j], -22);
                C[i * ldc + j] = ldexp(v, sA + sB);
            }
        }
        free(t11); free(tm); free(t22); free(b1); free(b2);
    }
}

/* The dropped term alone, 2^(sA+sB) * 2^-22 * A2*B2, fp64. */
void orc_dropped_term(int64_t M, int64_t N, int64_t K,
                      const uint16_t *A2, int64_t ldpa, int sA,
                      const uint16_t *B2, int64_t ldpb, int sB, double *C, int64_t ldc)
{
    for (int64_t i = 0; i < M; i++)
        for (int64_t j = 0; j < N; j++) {
            double t = 0.0;
            for (int64_t k = 0; k < K; k++)
                t += orc_dec16(A2[i * ldpa + k]) * orc_dec16(B2[k * ldpb + j]);
            C[i * ldc + j] = ldexp(t, sA + sB - 22);
        }
}

/* ------------------------------------------------------------------------------
 * End-to-end emulation on a sample of the output (the bench's cpu_baseline and the
 * full-size parity tests): the scales come from the WHOLE matrices (R1: per-matrix
 * scale), then only the sampled rows of A and columns of B are split and multiplied.
 * rows[R], cols[Cn] index the sampled outputs; out is R x Cn row-major.
 * Returns the first non-finite index of A (or of B, offset by M*K), or -1.
 * ---------------------------------------------------------------------------- */
int64_t orc_sgemm_sampled(int64_t M, int64_t N, int64_t K,
                          const float *A, int64_t lda, const float *B, int64_t ldb,
                          int64_t R, const int64_t *rows, int64_t Cn, const int64_t *cols,
                          int terms, double *out, int *sA_out, int *sB_out)
{
    double mA, mB;
    int64_t bad = orc_maxabs(M, K, A, lda, &mA);
    if (bad >= 0)
        return bad;
    bad = orc_maxabs(K, N, B, ldb, &mB);
    if (bad >= 0)
        return M * K + bad;
    int sA = orc_scale_exp(mA), sB = orc_scale_exp(mB);
    if (sA_out) *sA_out = sA;
    if (sB_out) *sB_out = sB;

    float *As = (float *)malloc(sizeof(float) * (size_t)(R * K + 1));
    float *Bs = (float *)malloc(sizeof(float) * (size_t)(K * Cn + 1));
    uint16_t *a1 = (uint16_t *)malloc(2 * (size_t)(R * K + 1));
    uint16_t *a2 = (uint16_t *)malloc(2 * (size_t)(R * K + 1));
    uint16_t *b1 = (uint16_t *)malloc(2 * (size_t)(K * Cn + 1));
    uint16_t *b2 = (uint16_t *)malloc(2 * (size_t)(K * Cn + 1));
    for (int64_t r = 0; r < R; r++)
        memcpy(As + r * K, A + rows[r] * lda, sizeof(float) * (size_t)K);
    for (int64_t k = 0; k < K; k++)
        for (int64_t c = 0; c < Cn; c++)
            Bs[k * Cn + c] = B[k * ldb + cols[c]];
    orc_split(R, K, As, K, sA, a1, a2, K);
    orc_split(K, Cn, Bs, Cn, sB, b1, b2, Cn);
    orc_split_gemm(R, Cn, K, a1, a2, K, sA, b1, b2, Cn, sB, terms, out, Cn);
    free(As); free(Bs); free(a1); free(a2); free(b1); free(b2);
    return -1;
}

/* ------------------------------------------------------------------------------
 * bf16 x 3 split ("the 16-bit bfloat16 format ... has the
 * advantage of having the same range as fp32"): no scale.  bfloat16 = binary32 with 8
 * significant bits; RN-even, subnormals kept, overflow -> inf, NaN -> 0x7FC0.
 *     X1 = RNbf(x),  X2 = RNbf(x - X1),  X3 = RNbf(x - X1 - X2)   (residuals exact in fp64)
 * Product (6 of the 9 terms, i + j <= 4):  C = X1Y1 + [X1Y2 + X2Y1 + X1Y3 + X2Y2 + X3Y1].
 * ---------------------------------------------------------------------------- */
uint16_t orc_encbf16(double x)
{
    uint64_t b;
    memcpy(&b, &x, sizeof b);
    uint16_t sign = (uint16_t)((b >> 63) << 15);
    int e = (int)((b >> 52) & 0x7FF);
    uint64_t mant = b & ((1ULL << 52) - 1);
    if (e == 0x7FF)
        return mant ? (uint16_t)0x7FC0 : (uint16_t)(sign | 0x7F80);
    if (e == 0)
        return sign;                    /* |x| < 2^-1022: far below the bf16 subnormal range */
    int E = e - 1023;
    uint64_t sig = (1ULL << 52) | mant;
    if (E > 127)
        return (uint16_t)(sign | 0x7F80);
    if (E >= -126) {                    /* normal: 8 significant bits */
        int shift = 52 - 7;
        uint64_t q = sig >> shift;
        uint64_t rem = sig & ((1ULL << shift) - 1);
        uint64_t half = 1ULL << (shift - 1);
        if (rem > half || (rem == half && (q & 1)))
            q++;
        if (q == 256) {
            q = 128;
            E++;
        }
        if (E > 127)
            return (uint16_t)(sign | 0x7F80);
        return (uint16_t)(sign | (uint16_t)((E + 127) << 7) | (uint16_t)(q & 0x7F));
    }
    /* subnormal bf16: multiple q of 2^-133;  q = sig * 2^(E - 52 + 133) */
    int shift = 52 - 133 - E;           /* = -81 - E >= 46 */
    if (shift > 54)
        return sign;
    uint64_t q = sig >> shift;
    uint64_t rem = sig & ((1ULL << shift) - 1);
    uint64_t half = 1ULL << (shift - 1);
    if (rem > half || (rem == half && (q & 1)))
        q++;
    return (uint16_t)(sign | (uint16_t)q);
}

double orc_decbf16(uint16_t h)
{
    uint32_t w = (uint32_t)h << 16;
    float f;
    memcpy(&f, &w, sizeof f);
    return (double)f;                   /* bf16 is the top half of binary32: exact */
}

void orc_encbf16_array(int64_t n, const double *x, uint16_t *h)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++)
        h[i] = orc_encbf16(x[i]);
}

void orc_split_bf16x3(int64_t rows, int64_t cols, const float *X, int64_t ld,
                      uint16_t *p1, uint16_t *p2, uint16_t *p3, int64_t ldp)
{
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < rows; i++) {
        for (int64_t j = 0; j < cols; j++) {
            double x = (double)X[i * ld + j];
            uint16_t h1 = orc_encbf16(x);
            double r1 = x - orc_decbf16(h1);
            uint16_t h2 = orc_encbf16(r1);
            double r2 = r1 - orc_decbf16(h2);
            uint16_t h3 = orc_encbf16(r2);
            p1[i * ldp + j] = h1;
            p2[i * ldp + j] = h2;
            p3[i * ldp + j] = h3;
        }
    }
}

/* C = X1Y1 + (X1Y2 + X2Y1 + X1Y3 + X2Y2 + X3Y1), fp64 sums of exact products.
 * X planes M x K row-major (ldx), Y planes K x N row-major (ldy). */
void orc_gemm_bf16x3(int64_t M, int64_t N, int64_t K,
                     const uint16_t *X1, const uint16_t *X2, const uint16_t *X3, int64_t ldx,
                     const uint16_t *Y1, const uint16_t *Y2, const uint16_t *Y3, int64_t ldy,
                     double *C, int64_t ldc)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < M; i++) {
        for (int64_t j = 0; j < N; j++) {
            double hi = 0.0, rest = 0.0;
            for (int64_t k = 0; k < K; k++) {
                double x1 = orc_decbf16(X1[i * ldx + k]), x2 = orc_decbf16(X2[i * ldx + k]),
                       x3 = orc_decbf16(X3[i * ldx + k]);
                double y1 = orc_decbf16(Y1[k * ldy + j]), y2 = orc_decbf16(Y2[k * ldy + j]),
                       y3 = orc_decbf16(Y3[k * ldy + j]);
                hi += x1 * y1;
                rest += x1 * y2 + x2 * y1 + x1 * y3 + x2 * y2 + x3 * y1;
            }
            C[i * ldc + j] = hi + rest;
        }
    }
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_num_threads(int n)
{
#ifdef _OPENMP
    if (n > 0)
        omp_set_num_threads(n);
#else
    (void)n;
#endif
}
