/*
 * split3.h — C ABI of the B200 (sm_100a) split-FP16 SGEMM.
 *
 * The method (arXiv 2011.11188, Appendix A; "PAPER.md:L" = line L of the paper text):
 *   Eq. A_1:   A ~= a1*A1 + a2*A2,  B ~= b1*B1 + b2*B2   (A1, A2, B1, B2 in FP16)
 *   PAPER.md:18-20:           a2 = 2^-11 * a1,     b2 = 2^-11 * b1
 *   Eq. A_2: C ~= a1b1*A1B1 + a1b2*A1B2 + a2b1*A2B1 + a2b2*A2B2
 *   PAPER.md:21-24:           a2b2 = 2^-22 a1b1 "may be optionally dropped" -> 3 FP16 GEMMs
 *   PAPER.md:282-285:         FP16 inputs, FP32 accumulation on tensor cores
 * Scale rule (the paper gives only its purpose; DESIGN.md §3 R1):
 *   a1 = 2^sA, sA = 0 if max|A| == 0 else max(floor(log2 max|A|) - 14, -127), over finite entries.
 * Epilogue (DESIGN.md §3 R7): C = (D_hi + 2^-11 * D_mid [+ 2^-22 * D_lo]) * 2^(sA+sB)
 *   with D_hi = A1*B1, D_mid = A1*B2 + A2*B1, D_lo = A2*B2 accumulated in FP32 (TMEM).
 *
 * Conventions for every entry point:
 *  - Matrices are ROW-MAJOR.  A is M x K (lda >= max(1,K)), B is K x N (ldb >= max(1,N)),
 *    C is M x N (ldc >= max(1,N)).  Leading dimensions are in elements.
 *  - All matrix/workspace pointers are DEVICE pointers owned by the caller (e.g. PyTorch
 *    allocations), except where an entry point says HOST.  The library allocates no device
 *    memory of its own beyond a few bytes per handle.
 *  - Calls are asynchronous on the handle's stream unless stated; errors are returned as a
 *    split3_status (never printed, never aborted).  Argument errors are detected before any
 *    work is enqueued.  SPLIT3_ERR_CUDA reports a failed launch / CUDA API call.
 *  - C must not alias A, B or the workspace.  A handle is not thread-safe: use one per stream.
 *  - Requires an sm_100 device (B200); other devices -> SPLIT3_ERR_ARCH at create time.
 *  - CUDA-graph capture: every asynchronous entry point may be captured (stream capture) and
 *    replayed; SPLIT3_CHECK_FINITE synchronises and therefore cannot be captured.
 */
#ifndef SPLIT3_H
#define SPLIT3_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct split3_ctx *split3_handle_t;

typedef enum split3_status {
    SPLIT3_OK = 0,
    SPLIT3_ERR_INVALID_VALUE = 1,   /* bad dimension, leading dimension, pointer or flag */
    SPLIT3_ERR_NOT_FINITE = 2,      /* SPLIT3_CHECK_FINITE found a NaN/Inf input entry */
    SPLIT3_ERR_WORKSPACE = 3,       /* workspace missing or smaller than split3_sgemm_workspace_size */
    SPLIT3_ERR_CUDA = 4,            /* a CUDA runtime/driver call or a launch failed */
    SPLIT3_ERR_ARCH = 5,            /* device is not sm_100 */
    SPLIT3_ERR_NOT_IMPLEMENTED = 6  /* a combination this build does not support */
} split3_status;

/* flags (bitwise OR) */
#define SPLIT3_THREE_TERM   0u         /* default: A1B1 + 2^-11 (A1B2 + A2B1) */
#define SPLIT3_FOUR_TERM    (1u << 0)  /* keep the dropped 2^-22 A2B2 term (Eq. A_2 in full) */
#define SPLIT3_CHECK_FINITE (1u << 1)  /* synchronise; reject NaN/Inf inputs */
#define SPLIT3_ONE_TERM     (1u << 2)  /* control: a1b1 * A1B1 only (a scaled plain FP16 GEMM) */
#define SPLIT3_BF16X3       (1u << 3)  /* variant: x = X1 + X2 + X3 in bfloat16 (no
                                          scale), C = X1Y1 + (X1Y2 + X2Y1 + X1Y3 + X2Y2
                                          + X3Y1): 6 BF16 products; fp32 operands only (no pre-split);
                                          |x| >= 3.39e38 overflows bf16 */
#define SPLIT3_FLAGS_MASK   (SPLIT3_FOUR_TERM | SPLIT3_CHECK_FINITE | SPLIT3_ONE_TERM | SPLIT3_BF16X3)

/* ---- handle ------------------------------------------------------------------------ */

/* Create a handle bound to CUDA device `device` and stream `cuda_stream` (a cudaStream_t;
 * NULL = the legacy default stream).  Fails with SPLIT3_ERR_ARCH unless the device is sm_100.
 * Environment variables read here select internal paths for A/B measurements; none changes a
 * bit of any result (tests compare the paths bitwise):
 *   SPLIT3_MN_MAJOR=0     K-major planes for every operand (transposing splits) instead of
 *                         MN-major planes for a row-major B / a transposed A;
 *   SPLIT3_PREP_MAX=<n>   use the one-launch max-abs + split front end for eager calls whose
 *                         fp32 operands hold <= n elements together (default 4 Mi; 0 = never);
 *   SPLIT3_FUSE_B=0|1|2, SPLIT3_FUSE_B_MAX_M=<m>   the fused split of B (split3_set_fused_split). */
int split3_sgemm_create(split3_handle_t *h, int device, void *cuda_stream);

/* Rebind the handle to another stream of the same device. */
int split3_set_stream(split3_handle_t h, void *cuda_stream);

/* Destroy the handle (does not free caller-owned workspace).  NULL is a no-op. */
int split3_sgemm_destroy(split3_handle_t h);

/* Bytes of device workspace split3_sgemm / split3_sgemm_ex need for (M, N, K): 256 bytes of
 * scalars, the four FP16 planes with padded leading dimensions (a multiple of 8 elements; B's
 * region fits either its K-major N x K planes or the MN-major K x N planes a row-major B is split
 * into) and,
 * when the problem has fewer 256-wide C tiles than CTA pairs, S*M*N floats of split-K partials
 * (S <= 16 slices of K, reduced in a fixed order: results are deterministic), sized for the
 * largest plan over every GEMM SM count up to 148 (split3_set_max_sms). */
size_t split3_sgemm_workspace_size(int64_t M, int64_t N, int64_t K, uint32_t flags);

/* Attach caller-owned device workspace (256-byte aligned).  The handle keeps the pointer;
 * the caller keeps ownership and must keep it alive while calls are in flight. */
int split3_sgemm_set_workspace(split3_handle_t h, void *dptr, size_t bytes);

/* ---- the whole method --------------------------------------------------------------- */

/* C = A*B emulated by FP16 tensor-core GEMMs.  Enqueues: max-abs of A and B,
 * split of A and B into FP16 planes (A: M x K K-major; B: K x N MN-major, no transpose), and the
 * tcgen05 GEMM with fused rescaling epilogue — or, for small M (split3_set_fused_split), the
 * split of A and a GEMM that splits B's fp32 tiles in shared memory.  C is overwritten
 * (beta = 0).  M == 0 or N == 0: no-op.  K == 0: C is zero-filled.
 * Non-finite inputs: without SPLIT3_CHECK_FINITE they propagate into the rows/columns of C
 * that touch them (the max-abs skips them); with it the call synchronises and returns
 * SPLIT3_ERR_NOT_FINITE, the index then being available from split3_last_bad_index. */
int split3_sgemm(split3_handle_t h, int64_t M, int64_t N, int64_t K,
                 const float *A, int64_t lda, const float *B, int64_t ldb,
                 float *C, int64_t ldc, uint32_t flags);

/* Same computation with HOST buffers (pageable or pinned): copies A and B to the workspace
 * staging area of the handle's device, runs the method, copies C back, and synchronises
 * the handle's stream before returning.  Same planes and scales as split3_sgemm; C is bitwise
 * equal to it except where the device call cuts a tail wave into split-K slices (another
 * summation order; both within the oracle tolerance).
 * Pipelined: B is copied first, then A in up to 20 row blocks, each split and
 * multiplied as soon as it lands while the next one copies in, and C row blocks copy out
 * underneath (2-D: B in 2 column panels, the second right after the first A block, so C pieces
 * leave early); env SPLIT3_HOST_BLOCKS=<1..16> / SPLIT3_HOST_PANELS=<1..4> at handle creation fix
 * the block / panel counts.  Device staging for A, B and C is taken from the
 * workspace, which must hold split3_sgemm_host_workspace_size(M, N, K, flags) bytes.
 * Host layout is packed row-major (lda = K, ldb = N, ldc = N). */
size_t split3_sgemm_host_workspace_size(int64_t M, int64_t N, int64_t K, uint32_t flags);
int split3_sgemm_host(split3_handle_t h, int64_t M, int64_t N, int64_t K,
                      const float *A_host, const float *B_host, float *C_host, uint32_t flags);

/* Where the last split3_sgemm_host call of this handle left its FP16 planes (introspection for
 * tests: DESIGN.md §5e).  A was split in `nblk` row blocks [blk_r0, + blk_rows), each with its own
 * scale exponent d_sblk[b] — or the per-matrix *d_sA where d_redo[b] != 0 (the block was redone) —
 * into K-major M x K planes A1/A2 (ldpa); B in `npan` column panels [pan_c0, + pan_cols) with
 * exponents d_span[j] (or *d_sB where d_redo[32 + j] != 0) into MN-major K x N planes B1/B2
 * (ldpb) when b_mn, else K-major N x K.  d_redo is NULL for a one-block, one-panel call (the
 * per-matrix exponents were used).  All pointers are device pointers into the workspace, valid
 * until the next call that uses it.  nblk == 0 before the first host call. */
typedef struct split3_host_layout {
    int nblk, npan;
    int64_t blk_r0[32], blk_rows[32];
    int64_t pan_c0[4], pan_cols[4];
    const uint16_t *A1, *A2;
    int64_t ldpa;
    const uint16_t *B1, *B2;
    int64_t ldpb;
    int b_mn;
    const int32_t *d_sblk, *d_span, *d_redo, *d_sA, *d_sB;
} split3_host_layout;
int split3_host_last_layout(split3_handle_t h, split3_host_layout *out);

/* After SPLIT3_ERR_NOT_FINITE: first offending linear index (row*cols+col) of A, or
 * M*K + index within B; -1 if none recorded. */
int64_t split3_last_bad_index(split3_handle_t h);

/* Row blocks split3_sgemm_host has redone with the per-matrix scale since the handle was created
 * (the host pipeline splits each A row block with its own scale exponent as it
 * arrives; a block whose exponent is below the per-matrix one and that holds a nonzero
 * |a| < 2^(sA-12) is redone so that C keeps the per-matrix bits).  -1 for a NULL handle. */
int64_t split3_host_redo_count(split3_handle_t h);

const char *split3_status_string(int status);

/* ---- operand descriptors: transposes and pre-split reuse --------------- */

/* One GEMM operand.  op(X) = X (trans = 0) or X^T (trans = 1), with X row-major fp32 in device
 * memory (`data`, leading dimension `ld` of the STORED matrix) — or, when `hi` is non-NULL, the
 * operand is given pre-split: `hi`, `lo` FP16 planes (ldp elements per row, 16-byte aligned) and
 * its device scale exponent, either
 *   stored = 0: planes written by split3_presplit for this role (K-major: M x K for A, N x K for
 *               B; `trans` is ignored), or
 *   stored = 1: the plain split of the STORED matrix (split3_presplit_stored: planes have the
 *               stored matrix's shape) and `trans` relates op(X) to it exactly as for fp32 data.
 *               The same planes then serve any role and either op(): a dense layer splits W,
 *               H and dZ once each and uses them in X*W, H^T*dZ and dZ*W^T.
 * Pre-split planes are immutable inputs and may be reused across calls.
 * Zero-initialise unused fields (stored = 0 keeps the original meaning). */
typedef struct split3_matrix {
    const float *data;
    int64_t ld;
    int trans;
    const uint16_t *hi;
    const uint16_t *lo;
    int64_t ldp;
    const int32_t *d_sexp;
    int stored;
} split3_matrix;

/* C = op(A) * op(B), op(A) M x K, op(B) K x N (PAPER.md:2-24 with the transposes a dense layer's
 * forward X*W, backward dY*W^T and X^T*dY need).  Operands given as fp32 are max-abs'ed and split
 * in this call (their planes go to the workspace); pre-split ones are used as they are.  Flags,
 * K == 0 and error behaviour as split3_sgemm; with SPLIT3_CHECK_FINITE the reported index is the
 * linear index in the STORED fp32 matrix (A first, then M*K + index in B). */
int split3_sgemm_ex(split3_handle_t h, int64_t M, int64_t N, int64_t K, const split3_matrix *A,
                    const split3_matrix *B, float *C, int64_t ldc, uint32_t flags);

/* Workspace bytes split3_sgemm_ex needs when A and/or B are given pre-split (a_presplit,
 * b_presplit != 0): with both pre-split only the 256-byte scalars block and the split-K partials
 * (none if split3_set_split_k(h, 0)); otherwise split3_sgemm_workspace_size(M, N, K, flags). */
size_t split3_sgemm_ex_workspace_size(int64_t M, int64_t N, int64_t K, uint32_t flags, int a_presplit,
                                      int b_presplit);

/* Split an operand once for reuse (a1 + a2 on one matrix, Eq. A_1, scale rule R1).  role 0: op(X)
 * is an A operand, rows x cols = M x K, planes M x K; role 1: op(X) is a B operand, rows x cols =
 * K x N, planes N x K (= op(X)^T, K-major).  X stored row-major (rows x cols if trans == 0, else
 * cols x rows), leading dimension ldx.  ldp >= K, multiple of 8; d_sexp receives the exponent.
 * Uses a few bytes of handle-owned scratch; asynchronous on the handle's stream. */
int split3_presplit(split3_handle_t h, int role, int64_t rows, int64_t cols, const float *X, int64_t ldx,
                    int trans, uint16_t *hi, uint16_t *lo, int64_t ldp, int32_t *d_sexp);

/* Split the STORED matrix X (rows x cols, row-major, leading dimension ldx) once, without a
 * transpose: max-abs + Eq. A_1 with the scale rule R1 into planes hi/lo of the same shape
 * (ldp >= cols, multiple of 8, 16-byte aligned); d_sexp receives the exponent.  The result is a
 * split3_matrix with stored = 1 usable as A or B, transposed or not.  Asynchronous. */
int split3_presplit_stored(split3_handle_t h, int64_t rows, int64_t cols, const float *X, int64_t ldx,
                           uint16_t *hi, uint16_t *lo, int64_t ldp, int32_t *d_sexp);

/* ---- lower level: used by the multi-GPU driver and by the tests -------------------------- */

/* Max-abs over FINITE entries of X (rows x cols, ld), folded into *d_maxabs with an atomic
 * max on the float's bit pattern (exact and order-independent; non-finite entries are
 * skipped, DESIGN.md §3 R8).  d_maxabs: device float, caller initialises it to 0.0f.
 * If d_bad is non-NULL (device int64, caller initialises to INT64_MAX), the smallest
 * linear index of a non-finite entry is folded into it with an atomic min. */
int split3_maxabs(split3_handle_t h, int64_t rows, int64_t cols, const float *X, int64_t ldx,
                  float *d_maxabs, int64_t *d_bad);

/* Split X (rows x cols, ld) with the scale exponent derived on the device from *d_maxabs
 * (the GLOBAL max when X is a shard; reading R1) into FP16 planes hi/lo (uint16 binary16
 * bit patterns) per Eq. A_1.  transpose = 0: planes are rows x cols (ldp >= cols);
 * transpose = 1: planes are cols x rows (ldp >= rows) — the K-major layout the GEMM wants
 * for B.  ldp must be a multiple of 8 and the plane pointers 16-byte aligned.
 * If d_sexp is non-NULL the scale exponent s is written to *d_sexp (device int32). */
int split3_split(split3_handle_t h, int64_t rows, int64_t cols, const float *X, int64_t ldx,
                 const float *d_maxabs, uint16_t *hi, uint16_t *lo, int64_t ldp, int transpose,
                 int32_t *d_sexp);

/* bf16 x 3 planes of X (SPLIT3_BF16X3's split, no scale): p1..p3 rows x cols (transpose = 0) or
 * cols x rows (transpose = 1), bfloat16 bit patterns, ldp a multiple of 8, 16-byte aligned. */
int split3_split_bf16x3(split3_handle_t h, int64_t rows, int64_t cols, const float *X, int64_t ldx,
                        uint16_t *p1, uint16_t *p2, uint16_t *p3, int64_t ldp, int transpose);

/* GEMM from planes: A1, A2 are M x K (K-major, ldpa), B1t, B2t are N x K (K-major, ldpb),
 * i.e. the planes of B TRANSPOSED.  *d_sA, *d_sB are the device scale exponents.  Computes
 * C = (D_hi + 2^-11 D_mid [+ 2^-22 D_lo]) * 2^(sA+sB) (flags as for split3_sgemm; with
 * SPLIT3_ONE_TERM only A1/B1t are read and A2/B2t may be NULL).  ldpa, ldpb multiples of 8,
 * plane pointers 16-byte aligned, K >= 1. */
int split3_gemm_planes(split3_handle_t h, int64_t M, int64_t N, int64_t K,
                       const uint16_t *A1, const uint16_t *A2, int64_t ldpa, const int32_t *d_sA,
                       const uint16_t *B1t, const uint16_t *B2t, int64_t ldpb, const int32_t *d_sB,
                       float *C, int64_t ldc, uint32_t flags);

/* Number of kernels the last split3_sgemm / split3_gemm_planes call launched (for the bench's
 * gpu_launches count; memsets are not counted). */
int split3_last_launch_count(split3_handle_t h);

/* Which path the last split3_sgemm / split3_sgemm_ex call took (bitwise OR; 0 = the plain
 * sequential path: max-abs, separate splits, GEMM).  For tests and the benchmark's report. */
#define SPLIT3_PATH_FUSED_B 1   /* B split inside the GEMM (split3_set_fused_split) */
#define SPLIT3_PATH_FUSED_A 2   /* A split inside the GEMM, C^T = B^T A^T (split3_set_fused_split_a) */
#define SPLIT3_PATH_PREP    8   /* one-launch max-abs + split front end (small calls) */
#define SPLIT3_PATH_FOLD   16   /* folded accumulator (split3_set_fold) */
int split3_last_path(split3_handle_t h);

/* ---- dense-network step helpers ----------------------------
 * The GEMMs of a dense-layer training step go through split3_sgemm_ex; these FP32 kernels do the
 * rest (SPEC.md mlp ledger: bias, activations, softmax/cross-entropy never in fp16).  All are
 * deterministic (fixed reduction orders).  Device pointers, row-major, asynchronous on the
 * handle's stream. */

/* H = act(Z + b): b (length N, may be NULL) broadcast over the M rows; act = ReLU if relu != 0. */
int split3_bias_act(split3_handle_t h, int64_t M, int64_t N, const float *Z, int64_t ldz, const float *b,
                    float *H, int64_t ldh, int relu);

/* dZ = dH * 1[H > 0] (ReLU backward through its output), packed M x N. */
int split3_relu_backward(split3_handle_t h, int64_t M, int64_t N, const float *dH, const float *H, float *dZ);

/* Row-wise softmax cross-entropy of logits L (M x N, packed): P = softmax(L) with max-subtraction,
 * dL = (P - onehot(labels)) / M, and *d_loss = mean_r -log P[r, labels[r]] in fp64.
 * P, dL, labels, d_loss may be NULL (skipped); row_scratch: M doubles (device) when d_loss != NULL. */
int split3_softmax_xent(split3_handle_t h, int64_t M, int64_t N, const float *L, const int32_t *labels,
                        float *P, float *dL, double *row_scratch, double *d_loss_sum);

/* db[c] = sum_r dZ[r, c], dZ packed M x N, in a fixed order (deterministic): with an attached
 * workspace of >= chunks * N floats (chunks = min(ceil(M / 256), 64) >= 2) the rows are cut into
 * `chunks` contiguous chunks, each summed as 8 interleaved row groups (row order inside a group,
 * groups in order) and the chunk sums added in chunk order; otherwise 32 interleaved row groups,
 * then the group sums in order.  Uses the handle's workspace as scratch (dead between calls). */
int split3_bias_grad(split3_handle_t h, int64_t M, int64_t N, const float *dZ, float *db);

/* w -= lr * g over n elements. */
int split3_sgd_update(split3_handle_t h, int64_t n, float *w, const float *g, float lr);

/* ---- numerics knob ------------------------------------------------------------------- */

/* D_hi promotion period (DESIGN.md §3 R9): the tcgen05 FP32 accumulator truncates, so the
 * A1*B1 product is accumulated in TMEM for at most `kblocks` 64-wide k-blocks (4*kblocks
 * MMAs) and then added with round-to-nearest into an FP32 master.  0 = library default (2).
 * Smaller = more accurate, more epilogue work.  Range 0..1024. */
int split3_set_promotion(split3_handle_t h, int kblocks);

/* GEMM wave lockstep (default on): the persistent GEMM's producers wait — bounded, at most
 * 0.2 ms — for all CTA pairs at each tile boundary so that concurrent tiles share their K-window
 * in L2 (DRAM traffic).  A scheduling hint only: results are identical either way. */
int split3_set_wave_sync(split3_handle_t h, int enable);

/* GEMM tile schedule: raster group height in 256-row tile pairs (0 = default 8) and the L2
 * eviction policy of the A-plane and B-plane TMA loads (0 normal, 1 evict_first, 2 evict_last).
 * Scheduling only: results are identical for every setting. */
int split3_set_schedule(split3_handle_t h, int group_m, int l2_policy_a, int l2_policy_b);

/* Split-K tail (default on): when the last wave of 256-wide C tiles is partial (or there are fewer
 * tiles than CTA pairs), those tiles are cut along K into S <= 16 slices whose FP32 partials are
 * summed in a fixed slice order (deterministic, but another summation order than a whole tile).
 * enable = 0: whole tiles only — every C element is then accumulated over K in the same order
 * whatever the shape of the problem it belongs to, so a C piece computed by split3_gemm_planes
 * (the multi-GPU driver's pieces, always whole tiles) and the same rows/columns of one
 * split3_sgemm call are bitwise equal (SURVEY §8e invariant; tests/test_gpu_dist_gloo_cuda.py).
 * Scheduling only for the numerics contract: both modes meet the oracle tolerance. */
int split3_set_split_k(split3_handle_t h, int enable);

/* Cap on the SMs the persistent GEMM occupies (0 = all, else an even count >= 2; counts above
 * the device's are ignored).  The multi-GPU driver leaves SMs free this way while its plane
 * all-gathers run on another stream: the GEMM holds ~225 KB of shared memory per SM, so a
 * collective kernel finds no SM to run on until a full-width GEMM drains.  Results are
 * identical for every cap with split-K off; with split-K on the tail plan depends on the cap.
 * INVALID_VALUE for an odd or negative count. */
int split3_set_max_sms(split3_handle_t h, int sms);

/* Fused split of B (Eq. A_1, applied inside the GEMM): for a
 * 3-term call whose B is an fp32 matrix (not pre-split; row-major K x N, or stored N x K with
 * transB = 1), 16-byte aligned with ld % 4 == 0, the GEMM TMA-loads B's fp32 tiles into shared
 * memory and converter warps split them there in place, so B's planes never go through HBM (only
 * the max-abs pass reads B beforehand).  The planes, and therefore C, are bit-identical to the separate split.
 * mode 0: off; 1 (default): when M <= max_m (default 2048: each B tile is converted once per
 * 256-row tile row, and the extra shared-memory traffic slows the GEMM ~11 %, which the saved
 * 8 B/element of B's split outweighs for small M), when M <= 2 max_m and K * N <= 2^25 (B's split is
 * then a larger share of the call), or for any M when the call is small enough for
 * the one-launch front end (SPLIT3_PREP_MAX; fused B is 5-25 % faster there); 2: whenever
 * eligible.  max_m = 0 keeps the current threshold.  Env: SPLIT3_FUSE_B,
 * SPLIT3_FUSE_B_MAX_M at handle creation.  INVALID_VALUE for mode outside 0..2 or max_m < 0. */
int split3_set_fused_split(split3_handle_t h, int mode, int64_t max_m);

/* Folded accumulator (SURVEY §8f NEXT #2's D_lo fold, generalised): the 3-term
 * (4-term) products of each 64-wide k-block go into ONE TMEM accumulator T — [A2*B2 first], then
 * A1*B2 + A2*B1 entered with tcgen05's scale-input-d (T <- products + 2^-11 T), then A1*B1 likewise
 * — so T = D_hi + 2^-11 D_mid [+ 2^-22 D_lo] of the k-block, and the epilogue adds T into the FP32
 * master with one RN every k-block (the promotion period is 1 whatever split3_set_promotion says).
 * No separate D_mid / D_lo accumulators: two T buffers ping-pong in TMEM and the 4-term path keeps
 * 256-wide tiles (the unfolded 4-term kernel needs 256 TMEM columns more and runs 256 x 128
 * tiles).  Rounding differs from the unfolded kernel; same oracle tolerance.  mode 0: never;
 * 1 (default): 4-term calls with M*N*K >= 8192^3 (the power-capped regime, measured +5.4 % at
 * N = 16384; smaller single calls run 2-6 % slower folded); 2: every 4- and 3-term call (3-term:
 * -1.6 %).  Env: SPLIT3_FOLD.  INVALID_VALUE for mode outside 0..2. */
int split3_set_fold(split3_handle_t h, int mode);

/* Fused split of A (SURVEY §8f NEXT #2 for the other operand; Eq. A_1 applied inside the GEMM):
 * for a 3-term call whose A is an fp32 matrix (not pre-split; row-major M x K, or stored K x M
 * with transA = 1), 16-byte aligned with ld % 4 == 0, and whose C is 16-byte aligned with
 * ldc % 4 == 0, the call computes the transposed problem C^T = B^T A^T: B's planes are the GEMM's
 * A operand, A's fp32 tiles are TMA-loaded and split in shared memory as the fused B operand
 * above, and the epilogue writes each C^T tile transposed into C (TMA stores; the split-K tail
 * reduction likewise).  A's planes never go through HBM.  The planes equal the separate split's
 * bit for bit; C equals, bit for bit, C^T = B^T A^T computed with separately split planes, and
 * is within the same oracle tolerance as the untransposed call (the tensor core may sum a K = 16
 * step in another order when the operand roles swap).  mode 0 (default: every other path of
 * this library reproduces the untransposed call's bits, and this one would not): off; 1: when
 * N <= max_n (default 2048) and N < M (A is the larger operand: fused A is then chosen over fused
 * B) and the call is not a one-launch small call; 2: whenever eligible (takes precedence over
 * fused B).  max_n = 0 keeps the current threshold.  Env: SPLIT3_FUSE_A, SPLIT3_FUSE_A_MAX_N at
 * handle creation.  INVALID_VALUE for mode outside 0..2 or max_n < 0. */
int split3_set_fused_split_a(split3_handle_t h, int mode, int64_t max_n);

/* ---- debug build (libsplit3_debug.so: the same sources with -DSPLIT3_DEBUG=1) ----------------
 * The GEMM's synchronisation checks that compute-sanitizer would provide (it is not usable on this
 * GPU pool), built in: a watchdog on every mbarrier wait (2 s), checks of the TMEM
 * allocation, the shared-memory carve-out, tile coordinates and k-block ranges, D_hi chunks issued
 * vs drained, and the wave-lockstep counter.  The first failure is recorded (out8[0] = code,
 * [1] = detail, [2] = CTA, [3] = warp, [4] = number of failures) in host-mapped memory; a watchdog
 * trip then traps the kernel, so a broken pipeline ends with a launch error (the context is lost;
 * the record stays readable) instead of hanging the GPU.  Results of the debug build are bitwise
 * those of the release build.
 * split3_debug_read copies the record (reset != 0 clears it); split3_debug_fault(1) injects a
 * missing TMA load into the next GEMM launches (tests), 0 clears it.  Process-wide (device
 * globals of the current device).  Release build: SPLIT3_ERR_NOT_IMPLEMENTED. */
int split3_debug_read(uint64_t *out8, int reset);
int split3_debug_fault(int fault);

/* ---- measurement hooks (bench.py's roofline; no effect on results) ---------------------- */

/* enable != 0: every following split3_sgemm records CUDA events on the handle's stream around
 * its split phase (max-abs + split kernels) and its GEMM kernel. */
int split3_timing_enable(split3_handle_t h, int enable);

/* Synchronise the recorded events and return the summed durations (milliseconds) of the split
 * phase and of the GEMM kernel since the last read, and the number of calls timed; resets. */
int split3_timing_read(split3_handle_t h, double *split_ms, double *gemm_ms, int *calls);

#ifdef __cplusplus
}
#endif

#endif /* SPLIT3_H */
