// capi.cu — the extern "C" boundary declared in include/split3.h.
//
// Validation, workspace carving and launch orchestration only: every arithmetic step of the
// path runs in the kernels of split_kernels.cu (a1, a2) and gemm3.cu (a3, a4).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <new>
#include <algorithm>
#include <vector>

#include "../../include/split3.h"
#include "internal.h"

// handle-owned device scratch (byte offsets): [0] GEMM wave-lockstep counter, [4] max-abs ticket,
// [12] GEMM exit ticket (the last CTA zeroes [0] and [12]), [16] presplit max, [20] dummy max of
// the one-matrix ticketed max-abs, [48..55] grid barrier (arrival count, sense) of the one-launch
// front end,
// [64..] max-abs block partials (2 x kMaxPartials floats)
constexpr size_t kMaxPartials = 2048;
constexpr size_t kCounterBytes = 64 + 2 * kMaxPartials * 4;

struct split3_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    void* ws = nullptr;
    size_t ws_bytes = 0;
    long long last_bad = -1;
    int last_launches = 0;
    int last_path = 0;   // SPLIT3_PATH_* bits of the last split3_sgemm_ex call
    int promo_kb = 0;   // 0 = library default
    int wave_sync = 1;  // GEMM wave lockstep hint (L2 locality)
    int split_k = 1;    // split-K tail for partial last waves (0: whole tiles only, split3_set_split_k)
    int max_sms = 0;    // SMs the GEMM may occupy (0: all; split3_set_max_sms)
    int prep_ok = 1;    // the cooperative one-launch front end is accepted (cleared on rejection)
    int64_t prep_max = split3::kPrepMaxElems;   // elements of A + B up to which it is used (env SPLIT3_PREP_MAX)
    int mn_major = 1;   // MN-major planes for a row-major B / a transposed A (no transposing split);
                        // env SPLIT3_MN_MAJOR=0: off (K-major planes, transposing split)
    // fused B: an fp32 B is split inside the GEMM (converter warps) instead of
    // by a separate pass.  0 off, 1 auto (M <= fuse_b_max_m, M <= 2 fuse_b_max_m with K*N <= 2^25,
    // or a small call of any M),
    // 2 whenever eligible (measured: profiles/fused_b_r01.md).  env SPLIT3_FUSE_B, SPLIT3_FUSE_B_MAX_M
    int fuse_b = 1;
    int64_t fuse_b_max_m = 2048;
    // fused A: the same for an fp32 A, through the transposed problem C^T = B^T A^T (A^T is the
    // fused operand; the epilogue stores C^T's tiles transposed into C).  0 off (default: the
    // transposed product differs in the last bits from the untransposed one), 1 auto
    // (N <= fuse_a_max_n and N < M: A is the larger operand; not a one-launch small call), 2
    // whenever eligible (before fused B).  env SPLIT3_FUSE_A, SPLIT3_FUSE_A_MAX_N
    int fuse_a = 0;
    int64_t fuse_a_max_n = 2048;
    // folded accumulator (LAY_FOLD): 3-/4-term products of a k-block summed in ONE TMEM
    // accumulator with tcgen05's scale-input-d, promoted every k-block.  0 never, 1 (default)
    // 4-term calls of >= 8192^3 multiply-adds, 2 every 4- and 3-term call.  env SPLIT3_FOLD
    int fold = 1;
    split3::GemmTuneIn tune;
    unsigned* d_counters = nullptr;   // 256 B of device scratch owned by the handle
    // host-buffer entry: copy-in / copy-out streams and events, created on first use
    cudaStream_t s_in = nullptr, s_out = nullptr;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_done = nullptr;
    cudaEvent_t ev_rows[64] = {};      // C piece computed (ring)
    cudaEvent_t ev_arows[32] = {};     // A row block b copied in
    cudaEvent_t ev_pan[4] = {};        // B column panel j copied in
    int host_blocks = 0;               // row blocks of the host pipeline (0 = automatic; env SPLIT3_HOST_BLOCKS)
    long long host_redo = 0;           // row blocks redone with the per-matrix scale (split3_host_redo_count)
    int host_panels = 0;               // B column panels of the 2-D host schedule (0 = automatic; env SPLIT3_HOST_PANELS)
    split3_host_layout host_layout = {};   // the last host call's planes (split3_host_last_layout)
    // measurement hooks: event triples (start, after split, after gemm) per timed call
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
};

namespace {
cudaEvent_t next_event(split3_ctx* h) {
    if (h->ev_used == h->ev_pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        h->ev_pool.push_back(e);
    }
    return h->ev_pool[h->ev_used++];
}
void record(split3_ctx* h, cudaEvent_t e) {
    if (e) cudaEventRecord(e, h->stream);
}
}  // namespace

namespace {

using split3::plane_ld;

// Scalars block at the start of the workspace (256 B): [0] float maxA, [1] float maxB,
// [2] int32 sA, [3] int32 sB, [8..9] int64 badA, [10..11] int64 badB.
constexpr size_t kScalarBytes = 256;

struct Carve {
    float* maxA;
    float* maxB;
    int32_t* sA;
    int32_t* sB;
    long long* badA;
    long long* badB;
    uint16_t* A1;
    uint16_t* A2;
    uint16_t* B1t;
    uint16_t* B2t;
    int64_t ldpa, ldpb, ldpa_mn, ldpb_mn;
    size_t end;   // bytes used
};

inline size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

Carve carve(void* ws, int64_t M, int64_t N, int64_t K) {
    Carve c;
    uint8_t* b = static_cast<uint8_t*>(ws);
    c.maxA = reinterpret_cast<float*>(b);
    c.maxB = c.maxA + 1;
    c.sA = reinterpret_cast<int32_t*>(b + 8);
    c.sB = c.sA + 1;
    c.badA = reinterpret_cast<long long*>(b + 32);
    c.badB = c.badA + 1;
    c.ldpa = plane_ld(K);
    c.ldpb = plane_ld(K);
    size_t off = kScalarBytes;
    // planes K-major (A: M x plane_ld(K), B: N x plane_ld(K)) or MN-major (A: K x plane_ld(M),
    // B: K x plane_ld(N): the plain split of a stored A^T / row-major B); regions fit either
    c.ldpa_mn = plane_ld(M);
    const size_t pa = align256(std::max((size_t)M * (size_t)c.ldpa, (size_t)K * (size_t)c.ldpa_mn) * 2);
    c.ldpb_mn = plane_ld(N);
    const size_t pb = align256(std::max((size_t)N * (size_t)c.ldpb, (size_t)K * (size_t)c.ldpb_mn) * 2);
    c.A1 = reinterpret_cast<uint16_t*>(b + off); off += pa;
    c.A2 = reinterpret_cast<uint16_t*>(b + off); off += pa;
    c.B1t = reinterpret_cast<uint16_t*>(b + off); off += pb;
    c.B2t = reinterpret_cast<uint16_t*>(b + off); off += pb;
    c.end = off;
    return c;
}

// Split-K partials the workspace reserves: the largest plan over every SM count up to kMaxSms (a
// handle may run its GEMM on fewer SMs: split3_set_max_sms, MIG, green contexts), so the plan a
// call makes always fits; a device with more SMs would fall back to whole tiles (not sm_100).
constexpr int kMaxSms = 148;
int64_t partial_elems_bound(int64_t M, int64_t N, int64_t K, int terms) {
    int64_t mx = 0;
    for (int sms = 2; sms <= kMaxSms; sms += 2)
        for (int fold = 0; fold < 2; fold++)   // (the folded 4-term kernel has 256-wide tiles)
            mx = std::max(mx, split3::gemm3_partial_elems(split3::gemm3_split_plan(M, N, K, terms, sms, 0, fold != 0),
                                                          terms, fold != 0));
    return mx;
}

size_t ws_bytes_for(int64_t M, int64_t N, int64_t K, bool planesA, bool planesB, int terms_for_partials) {
    if (M < 0 || N < 0 || K < 0) return 0;
    (void)planesA; (void)planesB;   // plane regions are always carved (fixed layout)
    size_t b = kScalarBytes + 2 * align256(std::max((size_t)M * (size_t)plane_ld(K), (size_t)K * (size_t)plane_ld(M)) * 2) +
               2 * align256(std::max((size_t)N * (size_t)plane_ld(K), (size_t)K * (size_t)plane_ld(N)) * 2);
    if (terms_for_partials) b += align256((size_t)partial_elems_bound(M, N, K, terms_for_partials) * 4);
    return b;
}


// bf16 x 3: three planes per operand (scalars block as usual; sA = sB stay 0: no scale)
struct CarveBF3 {
    uint16_t *A[3], *B[3];
    int64_t ldp, ldpa_mn, ldpb_mn;
    size_t end;
};
CarveBF3 carve_bf3(void* ws, int64_t M, int64_t N, int64_t K) {
    CarveBF3 c;
    uint8_t* b = static_cast<uint8_t*>(ws);
    c.ldp = plane_ld(K);
    c.ldpa_mn = plane_ld(M);
    c.ldpb_mn = plane_ld(N);
    size_t off = kScalarBytes;
    const size_t pa = align256(std::max((size_t)M * (size_t)c.ldp, (size_t)K * (size_t)c.ldpa_mn) * 2);
    const size_t pb = align256(std::max((size_t)N * (size_t)c.ldp, (size_t)K * (size_t)c.ldpb_mn) * 2);
    for (int i = 0; i < 3; i++) { c.A[i] = reinterpret_cast<uint16_t*>(b + off); off += pa; }
    for (int i = 0; i < 3; i++) { c.B[i] = reinterpret_cast<uint16_t*>(b + off); off += pb; }
    c.end = off;
    return c;
}
size_t ws_bytes_bf3(int64_t M, int64_t N, int64_t K, bool partials) {
    size_t b = kScalarBytes + 3 * align256(std::max((size_t)M * (size_t)plane_ld(K), (size_t)K * (size_t)plane_ld(M)) * 2) +
               3 * align256(std::max((size_t)N * (size_t)plane_ld(K), (size_t)K * (size_t)plane_ld(N)) * 2);
    if (partials) b += align256((size_t)partial_elems_bound(M, N, K, 6) * 4);
    return b;
}

inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

inline int terms_of(uint32_t flags) {
    if (flags & SPLIT3_BF16X3) return 6;
    if (flags & SPLIT3_ONE_TERM) return 1;
    if (flags & SPLIT3_FOUR_TERM) return 4;
    return 3;
}

int set_dev(split3_ctx* h) {
    return cudaSetDevice(h->device) == cudaSuccess ? SPLIT3_OK : SPLIT3_ERR_CUDA;
}

// SMs the GEMM's persistent grid may occupy (split3_set_max_sms; an even count, >= 2)
int gemm_sms(const split3_ctx* h) {
    return h->max_sms > 0 && h->max_sms < h->num_sms ? h->max_sms : h->num_sms;
}

}  // namespace

extern "C" {

const char* split3_status_string(int status) {
    switch (status) {
        case SPLIT3_OK: return "SPLIT3_OK";
        case SPLIT3_ERR_INVALID_VALUE: return "SPLIT3_ERR_INVALID_VALUE";
        case SPLIT3_ERR_NOT_FINITE: return "SPLIT3_ERR_NOT_FINITE";
        case SPLIT3_ERR_WORKSPACE: return "SPLIT3_ERR_WORKSPACE";
        case SPLIT3_ERR_CUDA: return "SPLIT3_ERR_CUDA";
        case SPLIT3_ERR_ARCH: return "SPLIT3_ERR_ARCH";
        case SPLIT3_ERR_NOT_IMPLEMENTED: return "SPLIT3_ERR_NOT_IMPLEMENTED";
        default: return "SPLIT3_ERR_UNKNOWN";
    }
}

int split3_sgemm_create(split3_handle_t* h, int device, void* cuda_stream) {
    if (!h) return SPLIT3_ERR_INVALID_VALUE;
    *h = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess) return SPLIT3_ERR_CUDA;
    if (device < 0 || device >= ndev) return SPLIT3_ERR_INVALID_VALUE;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return SPLIT3_ERR_CUDA;
    if (prop.major != 10 || prop.minor != 0) return SPLIT3_ERR_ARCH;
    split3_ctx* c = new (std::nothrow) split3_ctx();
    if (!c) return SPLIT3_ERR_CUDA;
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    c->stream = static_cast<cudaStream_t>(cuda_stream);
    // creation may happen while another stream of this thread is being captured into a CUDA graph
    // (a binding creating the handle of a new stream lazily): relaxed mode lets the allocation and
    // the synchronous zeroing of the handle's counters through
    cudaStreamCaptureMode mode = cudaStreamCaptureModeRelaxed;
    cudaThreadExchangeStreamCaptureMode(&mode);
    const bool ok = cudaSetDevice(device) == cudaSuccess && cudaMalloc(&c->d_counters, kCounterBytes) == cudaSuccess &&
                    cudaMemset(c->d_counters, 0, kCounterBytes) == cudaSuccess &&
                    cudaStreamSynchronize(cudaStreamLegacy) == cudaSuccess;   // zeroed before any stream uses it
    const bool dbg_ok = !ok || split3::gemm3_debug_init() >= 0;   // debug build: map the check record
    cudaThreadExchangeStreamCaptureMode(&mode);
    if (!ok || !dbg_ok) {
        if (c->d_counters) cudaFree(c->d_counters);
        delete c;
        return SPLIT3_ERR_CUDA;
    }
    if (const char* e = getenv("SPLIT3_MN_MAJOR")) c->mn_major = atoi(e) != 0;
    if (const char* e = getenv("SPLIT3_PREP_MAX")) c->prep_max = atoll(e);
    if (const char* e = getenv("SPLIT3_FUSE_B")) c->fuse_b = atoi(e);
    if (const char* e = getenv("SPLIT3_HOST_BLOCKS")) c->host_blocks = std::min(std::max(atoi(e), 0), 16);
    if (const char* e = getenv("SPLIT3_HOST_PANELS")) c->host_panels = std::min(std::max(atoi(e), 0), 4);
    if (const char* e = getenv("SPLIT3_FUSE_B_MAX_M")) c->fuse_b_max_m = atoll(e);
    if (const char* e = getenv("SPLIT3_FUSE_A")) c->fuse_a = atoi(e);
    if (const char* e = getenv("SPLIT3_FOLD")) c->fold = std::min(std::max(atoi(e), 0), 2);
    if (const char* e = getenv("SPLIT3_FUSE_A_MAX_N")) c->fuse_a_max_n = atoll(e);
    *h = c;
    return SPLIT3_OK;
}

int split3_set_stream(split3_handle_t h, void* cuda_stream) {
    if (!h) return SPLIT3_ERR_INVALID_VALUE;
    h->stream = static_cast<cudaStream_t>(cuda_stream);
    return SPLIT3_OK;
}

int split3_sgemm_destroy(split3_handle_t h) {
    if (h) {
        for (cudaEvent_t e : h->ev_pool) cudaEventDestroy(e);
        if (h->d_counters) cudaFree(h->d_counters);
        if (h->s_in) cudaStreamDestroy(h->s_in);
        if (h->s_out) cudaStreamDestroy(h->s_out);
        for (cudaEvent_t e : {h->ev_a, h->ev_b, h->ev_done})
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : h->ev_rows)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : h->ev_arows)
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : h->ev_pan)
            if (e) cudaEventDestroy(e);
    }
    delete h;
    return SPLIT3_OK;
}

size_t split3_sgemm_workspace_size(int64_t M, int64_t N, int64_t K, uint32_t flags) {
    if (M < 0 || N < 0 || K < 0) return 0;
    if (flags & SPLIT3_BF16X3) return ws_bytes_bf3(M, N, K, true);
    return ws_bytes_for(M, N, K, true, true, terms_of(flags));
}

size_t split3_sgemm_ex_workspace_size(int64_t M, int64_t N, int64_t K, uint32_t flags, int a_presplit,
                                      int b_presplit) {
    if (M < 0 || N < 0 || K < 0) return 0;
    if (!(a_presplit && b_presplit) || (flags & SPLIT3_BF16X3)) return split3_sgemm_workspace_size(M, N, K, flags);
    return kScalarBytes + align256((size_t)partial_elems_bound(M, N, K, terms_of(flags)) * 4);
}

int split3_sgemm_set_workspace(split3_handle_t h, void* dptr, size_t bytes) {
    if (!h) return SPLIT3_ERR_INVALID_VALUE;
    if (bytes && (!dptr || !aligned(dptr, 256))) return SPLIT3_ERR_INVALID_VALUE;
    h->ws = dptr;
    h->ws_bytes = dptr ? bytes : 0;
    return SPLIT3_OK;
}

int64_t split3_last_bad_index(split3_handle_t h) { return h ? h->last_bad : -1; }

int split3_last_launch_count(split3_handle_t h) { return h ? h->last_launches : 0; }
int split3_last_path(split3_handle_t h) { return h ? h->last_path : 0; }
int64_t split3_host_redo_count(split3_handle_t h) { return h ? h->host_redo : -1; }

int split3_maxabs(split3_handle_t h, int64_t rows, int64_t cols, const float* X, int64_t ldx,
                  float* d_maxabs, int64_t* d_bad) {
    if (!h || rows < 0 || cols < 0 || !d_maxabs) return SPLIT3_ERR_INVALID_VALUE;
    if (rows == 0 || cols == 0) return SPLIT3_OK;
    if (!X || ldx < cols || !aligned(d_maxabs, 4)) return SPLIT3_ERR_INVALID_VALUE;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    int n = split3::launch_maxabs(h->stream, rows, cols, X, ldx, d_maxabs,
                                  reinterpret_cast<long long*>(d_bad), h->num_sms);
    if (n < 0) return SPLIT3_ERR_CUDA;
    h->last_launches = n;
    return SPLIT3_OK;
}

int split3_split(split3_handle_t h, int64_t rows, int64_t cols, const float* X, int64_t ldx,
                 const float* d_maxabs, uint16_t* hi, uint16_t* lo, int64_t ldp, int transpose,
                 int32_t* d_sexp) {
    if (!h || rows < 0 || cols < 0 || !d_maxabs) return SPLIT3_ERR_INVALID_VALUE;
    if (transpose != 0 && transpose != 1) return SPLIT3_ERR_INVALID_VALUE;
    if (rows == 0 || cols == 0) return SPLIT3_OK;
    const int64_t need = transpose ? rows : cols;
    if (!X || !hi || !lo || ldx < cols || ldp < need || ldp % 8 != 0 || !aligned(hi, 16) ||
        !aligned(lo, 16))
        return SPLIT3_ERR_INVALID_VALUE;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    int n = transpose
                ? split3::launch_split_t(h->stream, rows, cols, X, ldx, d_maxabs, hi, lo, ldp, d_sexp, h->num_sms)
                : split3::launch_split(h->stream, rows, cols, X, ldx, d_maxabs, hi, lo, ldp, d_sexp, h->num_sms);
    if (n < 0) return SPLIT3_ERR_CUDA;
    h->last_launches = n;
    return SPLIT3_OK;
}

int split3_split_bf16x3(split3_handle_t h, int64_t rows, int64_t cols, const float* X, int64_t ldx,
                        uint16_t* p1, uint16_t* p2, uint16_t* p3, int64_t ldp, int transpose) {
    if (!h || rows < 0 || cols < 0 || (transpose != 0 && transpose != 1)) return SPLIT3_ERR_INVALID_VALUE;
    if (rows == 0 || cols == 0) return SPLIT3_OK;
    const int64_t need = transpose ? rows : cols;
    if (!X || !p1 || !p2 || !p3 || ldx < cols || ldp < need || ldp % 8 || !aligned(p1, 16) || !aligned(p2, 16) ||
        !aligned(p3, 16))
        return SPLIT3_ERR_INVALID_VALUE;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    int n = split3::launch_split_bf16x3(h->stream, rows, cols, X, ldx, p1, p2, p3, ldp, transpose, h->num_sms);
    if (n < 0) return SPLIT3_ERR_CUDA;
    h->last_launches = n;
    return SPLIT3_OK;
}

int split3_gemm_planes(split3_handle_t h, int64_t M, int64_t N, int64_t K, const uint16_t* A1,
                       const uint16_t* A2, int64_t ldpa, const int32_t* d_sA, const uint16_t* B1t,
                       const uint16_t* B2t, int64_t ldpb, const int32_t* d_sB, float* C,
                       int64_t ldc, uint32_t flags) {
    if (!h || M < 0 || N < 0 || K < 1) return SPLIT3_ERR_INVALID_VALUE;
    if (flags & ~SPLIT3_FLAGS_MASK) return SPLIT3_ERR_INVALID_VALUE;
    if ((flags & SPLIT3_ONE_TERM) && (flags & SPLIT3_FOUR_TERM)) return SPLIT3_ERR_INVALID_VALUE;
    if (M == 0 || N == 0) { h->last_launches = 0; return SPLIT3_OK; }
    const int terms = terms_of(flags);
    if (!A1 || !B1t || !C || !d_sA || !d_sB || ldc < N || ldpa < K || ldpb < K || ldpa % 8 ||
        ldpb % 8 || !aligned(A1, 16) || !aligned(B1t, 16))
        return SPLIT3_ERR_INVALID_VALUE;
    if (terms != 1 && (!A2 || !B2t || !aligned(A2, 16) || !aligned(B2t, 16)))
        return SPLIT3_ERR_INVALID_VALUE;
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return SPLIT3_ERR_NOT_IMPLEMENTED;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    cudaEvent_t ev0 = nullptr, ev2 = nullptr;
    if (h->timing && h->ev_used + 3 <= 3 * 4096) {
        ev0 = next_event(h);
        cudaEvent_t ev1 = next_event(h);
        ev2 = next_event(h);
        if (!ev0 || !ev1 || !ev2) return SPLIT3_ERR_CUDA;
        record(h, ev0);
        record(h, ev1);   // empty split phase
    }
    int err = 0;
    int n = split3::launch_gemm3(h->stream, M, N, K, A1, A2, ldpa, d_sA, B1t, B2t, ldpb, d_sB, C,
                                 ldc, terms, gemm_sms(h), h->promo_kb,
                                 h->wave_sync ? h->d_counters : nullptr, h->tune, nullptr, 0, &err, nullptr, nullptr,
                                 0, nullptr, 0, nullptr, 0, h->fold);
    if (n < 0) return err ? err : SPLIT3_ERR_CUDA;
    record(h, ev2);
    h->last_launches = n;
    return SPLIT3_OK;
}

// op(X) of a split3_matrix is X (trans = 0) or X^T (trans = 1).  The GEMM consumes K-major planes:
// A as M x K, B as N x K (= op(B)^T).  The split kernel that produces them directly: for A the
// transposing one iff trans; for B the transposing one iff !trans (B^T planes from row-major B).
static int split_operand(split3_ctx* h, int role, int64_t opr, int64_t opc, const split3_matrix* X,
                         float* d_max, uint16_t* hi, uint16_t* lo, int64_t ldp, int32_t* d_sexp, int* launches) {
    const bool tr = role == 0 ? X->trans != 0 : X->trans == 0;
    // stored matrix: rows x cols with ld
    const int64_t rows = X->trans ? opc : opr, cols = X->trans ? opr : opc;
    int n = tr ? split3::launch_split_t(h->stream, rows, cols, X->data, X->ld, d_max, hi, lo, ldp, d_sexp, h->num_sms)
               : split3::launch_split(h->stream, rows, cols, X->data, X->ld, d_max, hi, lo, ldp, d_sexp, h->num_sms);
    if (n < 0) return SPLIT3_ERR_CUDA;
    *launches += n;
    return SPLIT3_OK;
}

static bool operand_ok(const split3_matrix* X, int64_t opr, int64_t opc, int role, int terms) {
    if (!X || (X->trans != 0 && X->trans != 1)) return false;
    if (X->hi) {   // pre-split planes
        // stored: the plain split of the stored matrix (row length: op cols, or op rows if trans);
        // else split3_presplit's K-major planes (rows = M (A) or N (B), K columns)
        const int64_t need = X->stored ? (X->trans ? opr : opc) : (role == 0 ? opc : opr);
        if (X->stored != 0 && X->stored != 1) return false;
        if (!X->d_sexp || X->ldp < need || X->ldp % 8 || !aligned(X->hi, 16)) return false;
        if (terms != 1 && (!X->lo || !aligned(X->lo, 16))) return false;
        return true;
    }
    if (!X->data) return false;
    const int64_t stored_cols = X->trans ? opr : opc;
    return X->ld >= (stored_cols > 1 ? stored_cols : 1);
}

// bf16 x 3 variant of split3_sgemm_ex (NEXT #4): fp32 operands only, no scale pass.
static int sgemm_bf16x3(split3_ctx* h, int64_t M, int64_t N, int64_t K, const split3_matrix* A,
                        const split3_matrix* B, float* C, int64_t ldc, uint32_t flags) {
    if (A->hi || B->hi) return SPLIT3_ERR_NOT_IMPLEMENTED;     // pre-split planes are FP16 x 2
    if (h->ws_bytes < ws_bytes_bf3(M, N, K, false)) return SPLIT3_ERR_WORKSPACE;
    CarveBF3 w = carve_bf3(h->ws, M, N, K);
    Carve sc = carve(h->ws, M, N, K);    // the scalars block (sA = sB = 0, bad indices)
    if (cudaMemsetAsync(h->ws, 0, 32, h->stream) != cudaSuccess) return SPLIT3_ERR_CUDA;
    int launches = 0, n;
    if (flags & SPLIT3_CHECK_FINITE) {
        if (cudaMemsetAsync(sc.badA, 0xFF, 16, h->stream) != cudaSuccess ||
            cudaMemsetAsync(reinterpret_cast<uint8_t*>(sc.badA) + 7, 0x7F, 1, h->stream) != cudaSuccess ||
            cudaMemsetAsync(reinterpret_cast<uint8_t*>(sc.badB) + 7, 0x7F, 1, h->stream) != cudaSuccess)
            return SPLIT3_ERR_CUDA;
        const int64_t ra = A->trans ? K : M, ca = A->trans ? M : K, rb = B->trans ? N : K, cb = B->trans ? K : N;
        if ((n = split3::launch_maxabs(h->stream, ra, ca, A->data, A->ld, sc.maxA, sc.badA, h->num_sms)) < 0 ||
            (launches += n, n = split3::launch_maxabs(h->stream, rb, cb, B->data, B->ld, sc.maxB, sc.badB, h->num_sms)) < 0)
            return SPLIT3_ERR_CUDA;
        launches += n;
        long long bad[2];
        if (cudaMemcpyAsync(bad, sc.badA, 16, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
            cudaStreamSynchronize(h->stream) != cudaSuccess)
            return SPLIT3_ERR_CUDA;
        if (bad[0] != INT64_MAX || bad[1] != INT64_MAX) {
            h->last_bad = bad[0] != INT64_MAX ? bad[0] : M * K + bad[1];
            h->last_launches = launches;
            return SPLIT3_ERR_NOT_FINITE;
        }
    }
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    if (h->timing && h->ev_used + 3 <= 3 * 4096) {
        ev0 = next_event(h); ev1 = next_event(h); ev2 = next_event(h);
        if (!ev0 || !ev1 || !ev2) return SPLIT3_ERR_CUDA;
        record(h, ev0);
    }
    const bool b_mn = !B->trans && h->mn_major, a_mn = A->trans && h->mn_major;
    {   // K-major planes (A: M x K, transposing split iff transA; B: N x K, iff !transB), or
        // MN-major planes (no transpose) for a stored A^T / a row-major B
        const int64_t ra = A->trans ? K : M, ca = A->trans ? M : K;
        if ((n = split3::launch_split_bf16x3(h->stream, ra, ca, A->data, A->ld, w.A[0], w.A[1], w.A[2],
                                             a_mn ? w.ldpa_mn : w.ldp, a_mn ? 0 : A->trans, h->num_sms)) < 0)
            return SPLIT3_ERR_CUDA;
        launches += n;
        const int64_t rb = B->trans ? N : K, cb = B->trans ? K : N;
        // a row-major K x N B: MN-major K x N planes without a transpose (as in the FP16 path)
        if ((n = split3::launch_split_bf16x3(h->stream, rb, cb, B->data, B->ld, w.B[0], w.B[1], w.B[2],
                                             b_mn ? w.ldpb_mn : w.ldp, b_mn ? 0 : !B->trans, h->num_sms)) < 0)
            return SPLIT3_ERR_CUDA;
        launches += n;
    }
    record(h, ev1);
    float* partial = reinterpret_cast<float*>(static_cast<uint8_t*>(h->ws) + w.end);
    size_t reserved = ws_bytes_bf3(M, N, K, true) - w.end;
    if (reserved > h->ws_bytes - w.end) reserved = h->ws_bytes - w.end;
    int err = 0;
    n = split3::launch_gemm3(h->stream, M, N, K, w.A[0], w.A[1], a_mn ? w.ldpa_mn : w.ldp, sc.sA, w.B[0], w.B[1],
                             b_mn ? w.ldpb_mn : w.ldp, sc.sB, C, ldc, 6, gemm_sms(h), h->promo_kb,
                             h->wave_sync ? h->d_counters : nullptr, h->tune, h->split_k ? partial : nullptr,
                             (int64_t)(reserved / 4), &err,
                             w.A[2], w.B[2], (b_mn ? 1 : 0) | (a_mn ? 2 : 0));
    if (n < 0) return err ? err : SPLIT3_ERR_CUDA;
    record(h, ev2);
    h->last_launches = launches + n;
    return SPLIT3_OK;
}

int split3_sgemm_ex(split3_handle_t h, int64_t M, int64_t N, int64_t K, const split3_matrix* A,
                    const split3_matrix* B, float* C, int64_t ldc, uint32_t flags) {
    if (!h || M < 0 || N < 0 || K < 0 || !A || !B) return SPLIT3_ERR_INVALID_VALUE;
    if (flags & ~SPLIT3_FLAGS_MASK) return SPLIT3_ERR_INVALID_VALUE;
    if ((flags & SPLIT3_ONE_TERM) && (flags & SPLIT3_FOUR_TERM)) return SPLIT3_ERR_INVALID_VALUE;
    if ((flags & SPLIT3_BF16X3) && (flags & (SPLIT3_ONE_TERM | SPLIT3_FOUR_TERM))) return SPLIT3_ERR_INVALID_VALUE;
    h->last_launches = 0;
    h->last_bad = -1;
    h->last_path = 0;
    if (M == 0 || N == 0) return SPLIT3_OK;
    if (!C || ldc < N) return SPLIT3_ERR_INVALID_VALUE;
    const int terms = terms_of(flags);
    if (K > 0 && (!operand_ok(A, M, K, 0, terms) || !operand_ok(B, K, N, 1, terms))) return SPLIT3_ERR_INVALID_VALUE;
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return SPLIT3_ERR_NOT_IMPLEMENTED;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    if (K == 0) {   // empty sum: C = 0
        if (cudaMemset2DAsync(C, (size_t)ldc * 4, 0, (size_t)N * 4, (size_t)M, h->stream) != cudaSuccess)
            return SPLIT3_ERR_CUDA;
        return SPLIT3_OK;
    }
    if (!h->ws || h->ws_bytes < kScalarBytes) return SPLIT3_ERR_WORKSPACE;
    if (flags & SPLIT3_BF16X3) return sgemm_bf16x3(h, M, N, K, A, B, C, ldc, flags);
    const bool needA = A->hi == nullptr, needB = B->hi == nullptr;
    // planes carved only when an operand is split here; two pre-split operands need the scalars
    // block (and split-K partials right after it)
    const bool planes_ws = needA || needB;
    const size_t need = planes_ws ? ws_bytes_for(M, N, K, needA, needB, 0) : kScalarBytes;
    if (h->ws_bytes < need) return SPLIT3_ERR_WORKSPACE;
    Carve w = carve(h->ws, M, N, K);
    const bool check = (flags & SPLIT3_CHECK_FINITE) != 0;
    // scalars: maxA = maxB = 0.0f, sA = sB = 0, badA = badB = INT64_MAX.  The common path (both
    // operands fp32, no check) needs no reset: the two-matrix max-abs writes maxA/maxB itself.
    const bool fast_max = needA && needB && !check;
    // fused B (NEXT #2): 3-term, fp32 B (row-major K x N, or stored N x K for transB) that TMA
    // can read (16-B aligned, ld % 4 == 0)
    const bool small_call = fast_max && h->mn_major && h->prep_ok && h->prep_max >= M * K + K * N;
    // fused A (NEXT #2 for A): the transposed problem C^T = B^T A^T with A^T as the fused operand
    // (an fp32 A of either storage TMA can read) and C written transposed (TMA stores: C 16-B
    // aligned, ldc % 4 == 0); preferred over fused B when A is the larger operand (N < M)
    const bool fuse_a = needA && terms == 3 && aligned(A->data, 16) && (A->ld % 4) == 0 && aligned(C, 16) &&
                        (ldc % 4) == 0 &&
                        (h->fuse_a == 2 || (h->fuse_a == 1 && N <= h->fuse_a_max_n && N < M && !small_call));
    // fused B: M <= fuse_b_max_m; or M <= 2 fuse_b_max_m with a B of at most 2^25 elements (its
    // split is then a larger share of the call: 4096^3 +1.6 %, 4096 x 8192 x 4096 +3.5 %, while
    // 4096 x 8192^2 loses 0.5-6.5 %: profiles/fused_b_bench_midM_r02.json); or any M for a small
    // call (faster than the one-launch front end at every small shape, 5-25 %:
    // profiles/small_fused_bench_r02.json)
    const bool mid_m = M <= 2 * h->fuse_b_max_m && N * K <= ((int64_t)1 << 25);
    const bool fuse_b = !fuse_a && needB && terms == 3 && aligned(B->data, 16) && (B->ld % 4) == 0 &&
                        (h->fuse_b == 2 || (h->fuse_b == 1 && (M <= h->fuse_b_max_m || mid_m || small_call)));
    // (both operands pre-split: no max-abs at all, nothing to reset)
    if (!fast_max && (needA || needB) && cudaMemsetAsync(h->ws, 0, 32, h->stream) != cudaSuccess)
        return SPLIT3_ERR_CUDA;
    int launches = 0, n;
    if (check) {
        if (cudaMemsetAsync(w.badA, 0xFF, 16, h->stream) != cudaSuccess ||
            cudaMemsetAsync(reinterpret_cast<uint8_t*>(w.badA) + 7, 0x7F, 1, h->stream) != cudaSuccess ||
            cudaMemsetAsync(reinterpret_cast<uint8_t*>(w.badB) + 7, 0x7F, 1, h->stream) != cudaSuccess)
            return SPLIT3_ERR_CUDA;
    }
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    if (h->timing && h->ev_used + 3 <= 3 * 4096) {
        ev0 = next_event(h); ev1 = next_event(h); ev2 = next_event(h);
        if (!ev0 || !ev1 || !ev2) return SPLIT3_ERR_CUDA;
        record(h, ev0);
    }
    // small problems: a1 + a2 of both operands in ONE cooperative launch (all splits are plain
    // with MN-major planes); a rejected cooperative launch switches the handle to the 3 kernels
    // (eager calls only: under CUDA-graph capture the separate kernels' programmatic edges
    // replay faster than one cooperative node: 0.361 vs 0.403 ms per small-MLP step)
    bool prepped = false;
    cudaStreamCaptureStatus cap_st = cudaStreamCaptureStatusNone;
    if (!fuse_b && !fuse_a && small_call &&
        cudaStreamIsCapturing(h->stream, &cap_st) == cudaSuccess && cap_st == cudaStreamCaptureStatusNone) {
        const split3::PrepOperand pa{A->data, A->trans ? K : M, A->trans ? M : K, A->ld, w.A1, w.A2,
                                     A->trans ? w.ldpa_mn : w.ldpa, w.maxA, w.sA};
        const split3::PrepOperand pb{B->data, B->trans ? N : K, B->trans ? K : N, B->ld, w.B1t, w.B2t,
                                     B->trans ? w.ldpb : w.ldpb_mn, w.maxB, w.sB};
        unsigned* parts_u = reinterpret_cast<unsigned*>(reinterpret_cast<uint8_t*>(h->d_counters) + 64);
        n = split3::launch_prep2(h->stream, pa, pb, parts_u, h->d_counters + 12, h->num_sms);
        if (n == -2) {
            h->prep_ok = 0;
        } else if (n < 0) {
            return SPLIT3_ERR_CUDA;
        } else {
            launches += n;
            prepped = true;
        }
    }
    // a1: per-matrix max-abs (reading R1) of the fp32 operands (max|op(X)| = max|X|)
    if (prepped) {
    } else if (fast_max) {
        const int64_t ra = A->trans ? K : M, ca = A->trans ? M : K;
        const int64_t rb = B->trans ? N : K, cb = B->trans ? K : N;
        float* parts = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(h->d_counters) + 64);
        unsigned* ticket = h->d_counters + 1;
        if ((n = split3::launch_maxabs2(h->stream, ra, ca, A->data, A->ld, w.maxA, rb, cb, B->data, B->ld, w.maxB,
                                        h->num_sms, parts, (int)kMaxPartials, ticket)) < 0)
            return SPLIT3_ERR_CUDA;
        launches += n;
    } else if (needA) {
        const int64_t r = A->trans ? K : M, c = A->trans ? M : K;
        if ((n = split3::launch_maxabs(h->stream, r, c, A->data, A->ld, w.maxA, check ? w.badA : nullptr, h->num_sms)) < 0)
            return SPLIT3_ERR_CUDA;
        launches += n;
    }
    if (needB && !(needA && !check) && !prepped) {
        const int64_t r = B->trans ? N : K, c = B->trans ? K : N;
        if ((n = split3::launch_maxabs(h->stream, r, c, B->data, B->ld, w.maxB, check ? w.badB : nullptr, h->num_sms)) < 0)
            return SPLIT3_ERR_CUDA;
        launches += n;
    }
    if (check) {
        long long bad[2];
        if (cudaMemcpyAsync(bad, w.badA, 16, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
            cudaStreamSynchronize(h->stream) != cudaSuccess)
            return SPLIT3_ERR_CUDA;
        if (bad[0] != INT64_MAX || bad[1] != INT64_MAX) {   // linear index in the STORED matrix
            h->last_bad = bad[0] != INT64_MAX ? bad[0] : M * K + bad[1];
            h->last_launches = launches;
            return SPLIT3_ERR_NOT_FINITE;
        }
    }
    h->last_path = (fuse_b ? SPLIT3_PATH_FUSED_B : 0) | (fuse_a ? SPLIT3_PATH_FUSED_A : 0) | (prepped ? SPLIT3_PATH_PREP : 0) |
                   (split3::gemm3_fold_chosen(M, N, K, terms, h->fold) ? SPLIT3_PATH_FOLD : 0);
    // a2: split into K-major planes (A: M x K, B: N x K)
    const uint16_t *A1 = A->hi, *A2 = A->lo, *B1t = B->hi, *B2t = B->lo;
    const int32_t *sA = A->d_sexp, *sB = B->d_sexp;
    int64_t ldpa = A->ldp, ldpb = B->ldp;
    // pre-split planes of the stored matrix: A stored K x M (trans) is MN-major, B stored K x N
    // (not trans) is MN-major; the other two cases are K-major
    const bool a_mn = (needA && A->trans && h->mn_major) || (!needA && A->stored && A->trans);
    if (fuse_a) {
        sA = w.sA;   // written by the GEMM (A's planes never reach HBM)
    } else if (prepped) {
        A1 = w.A1; A2 = w.A2; sA = w.sA; ldpa = a_mn ? w.ldpa_mn : w.ldpa;
    } else if (needA && a_mn) {
        if ((n = split3::launch_split(h->stream, K, M, A->data, A->ld, w.maxA, w.A1, w.A2, w.ldpa_mn, w.sA,
                                      h->num_sms)) < 0)
            return SPLIT3_ERR_CUDA;
        launches += n;
        A1 = w.A1; A2 = w.A2; sA = w.sA; ldpa = w.ldpa_mn;
    } else if (needA) {
        int st = split_operand(h, 0, M, K, A, w.maxA, w.A1, w.A2, w.ldpa, w.sA, &launches);
        if (st) return st;
        A1 = w.A1; A2 = w.A2; sA = w.sA; ldpa = w.ldpa;
    }
    const bool b_mn = (needB && !B->trans && (h->mn_major || fuse_b)) || (!needB && B->stored && !B->trans);
    if (fuse_b) {
        sB = w.sB;   // written by the GEMM (the planes never reach HBM)
    } else if (prepped) {
        B1t = w.B1t; B2t = w.B2t; sB = w.sB; ldpb = b_mn ? w.ldpb_mn : w.ldpb;
    } else if (needB && b_mn) {
        if ((n = split3::launch_split(h->stream, K, N, B->data, B->ld, w.maxB, w.B1t, w.B2t, w.ldpb_mn, w.sB,
                                      h->num_sms)) < 0)
            return SPLIT3_ERR_CUDA;
        launches += n;
        B1t = w.B1t; B2t = w.B2t; sB = w.sB; ldpb = w.ldpb_mn;
    } else if (needB) {
        int st = split_operand(h, 1, K, N, B, w.maxB, w.B1t, w.B2t, w.ldpb, w.sB, &launches);
        if (st) return st;
        B1t = w.B1t; B2t = w.B2t; sB = w.sB; ldpb = w.ldpb;
    }
    record(h, ev1);
    // a3 + a4: tensor-core products with the fused epilogue (split-K partials after the planes)
    // split-K partials: only the region split3_sgemm_workspace_size reserves for them (whatever
    // follows it in the workspace may be staging buffers of split3_sgemm_host)
    const size_t pend = planes_ws ? w.end : kScalarBytes;
    float* partial = reinterpret_cast<float*>(static_cast<uint8_t*>(h->ws) + pend);
    size_t reserved = planes_ws ? ws_bytes_for(M, N, K, true, true, terms) - w.end
                                : align256((size_t)partial_elems_bound(M, N, K, terms) * 4);
    if (reserved > h->ws_bytes - pend) reserved = h->ws_bytes - pend;
    const int64_t partial_elems = (int64_t)(reserved / 4);
    int err = 0;
    if (fuse_a)   // C^T (N x M) = B^T A^T: B's planes are the A operand (MN-major iff B's are), the
                  // fp32 A is the fused B operand (MN-major iff A is stored K x M), C stored transposed
        n = split3::launch_gemm3(h->stream, N, M, K, B1t, B2t, ldpb, sB, nullptr, nullptr, 0, sA, C, ldc, terms,
                                 gemm_sms(h), h->promo_kb, h->wave_sync ? h->d_counters : nullptr, h->tune,
                                 h->split_k ? partial : nullptr, partial_elems, &err, nullptr, nullptr,
                                 (A->trans ? 1 : 0) | (b_mn ? 2 : 0), A->data, A->ld, w.maxA, 1, h->fold);
    else
        n = split3::launch_gemm3(h->stream, M, N, K, A1, A2, ldpa, sA, B1t, B2t, ldpb, sB, C, ldc, terms,
                                 gemm_sms(h), h->promo_kb, h->wave_sync ? h->d_counters : nullptr, h->tune,
                                 h->split_k ? partial : nullptr, partial_elems, &err, nullptr, nullptr,
                                 (b_mn ? 1 : 0) | (a_mn ? 2 : 0), fuse_b ? B->data : nullptr, B->ld, w.maxB, 0,
                                 h->fold);
    if (n < 0) return err ? err : SPLIT3_ERR_CUDA;
    record(h, ev2);
    launches += n;
    h->last_launches = launches;
    return SPLIT3_OK;
}

int split3_sgemm(split3_handle_t h, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                 const float* B, int64_t ldb, float* C, int64_t ldc, uint32_t flags) {
    if (!h) return SPLIT3_ERR_INVALID_VALUE;
    if (K > 0 && M > 0 && N > 0 && (!A || !B)) return SPLIT3_ERR_INVALID_VALUE;
    split3_matrix a = {A, lda, 0, nullptr, nullptr, 0, nullptr, 0};
    split3_matrix b = {B, ldb, 0, nullptr, nullptr, 0, nullptr, 0};
    return split3_sgemm_ex(h, M, N, K, &a, &b, C, ldc, flags);
}

int split3_presplit(split3_handle_t h, int role, int64_t rows, int64_t cols, const float* X, int64_t ldx,
                    int trans, uint16_t* hi, uint16_t* lo, int64_t ldp, int32_t* d_sexp) {
    if (!h || (role != 0 && role != 1) || (trans != 0 && trans != 1) || rows < 0 || cols < 0)
        return SPLIT3_ERR_INVALID_VALUE;
    if (rows == 0 || cols == 0) return SPLIT3_OK;
    const int64_t prow = role == 0 ? rows : cols, pk = role == 0 ? cols : rows;   // planes prow x pk
    const int64_t stored_cols = trans ? rows : cols;
    if (!X || !hi || !lo || !d_sexp || ldx < stored_cols || ldp < pk || ldp % 8 || !aligned(hi, 16) ||
        !aligned(lo, 16))
        return SPLIT3_ERR_INVALID_VALUE;
    (void)prow;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    float* d_max = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(h->d_counters) + 16);
    if (cudaMemsetAsync(d_max, 0, 4, h->stream) != cudaSuccess) return SPLIT3_ERR_CUDA;
    int launches = 0;
    const int64_t sr = trans ? cols : rows, sc = trans ? rows : cols;
    int n = split3::launch_maxabs(h->stream, sr, sc, X, ldx, d_max, nullptr, h->num_sms);
    if (n < 0) return SPLIT3_ERR_CUDA;
    launches += n;
    split3_matrix m = {X, ldx, trans, nullptr, nullptr, 0, nullptr, 0};
    int st = split_operand(h, role, rows, cols, &m, d_max, hi, lo, ldp, d_sexp, &launches);
    if (st) return st;
    h->last_launches = launches;
    return SPLIT3_OK;
}

int split3_presplit_stored(split3_handle_t h, int64_t rows, int64_t cols, const float* X, int64_t ldx, uint16_t* hi,
                           uint16_t* lo, int64_t ldp, int32_t* d_sexp) {
    if (!h || rows < 0 || cols < 0) return SPLIT3_ERR_INVALID_VALUE;
    if (rows == 0 || cols == 0) return SPLIT3_OK;
    if (!X || !hi || !lo || !d_sexp || ldx < cols || ldp < cols || ldp % 8 || !aligned(hi, 16) || !aligned(lo, 16))
        return SPLIT3_ERR_INVALID_VALUE;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    float* d_max = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(h->d_counters) + 16);
    int launches = 0, n;
    if (ldx == cols && aligned(X, 16) && cols >= 4) {
        // ticketed max-abs (writes *d_max itself: no memset node, so the programmatic edge to the
        // split survives under graph capture); the second operand is a 4-element dummy
        float* dummy = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(h->d_counters) + 20);
        float* parts = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(h->d_counters) + 64);
        if ((n = split3::launch_maxabs2(h->stream, rows, cols, X, ldx, d_max, 1, 4, X, 4, dummy, h->num_sms, parts,
                                        (int)kMaxPartials, h->d_counters + 1)) < 0)
            return SPLIT3_ERR_CUDA;
    } else {
        if (cudaMemsetAsync(d_max, 0, 4, h->stream) != cudaSuccess) return SPLIT3_ERR_CUDA;
        if ((n = split3::launch_maxabs(h->stream, rows, cols, X, ldx, d_max, nullptr, h->num_sms)) < 0)
            return SPLIT3_ERR_CUDA;
    }
    launches += n;
    if ((n = split3::launch_split(h->stream, rows, cols, X, ldx, d_max, hi, lo, ldp, d_sexp, h->num_sms)) < 0)
        return SPLIT3_ERR_CUDA;
    h->last_launches = launches + n;
    return SPLIT3_OK;
}

int split3_bias_act(split3_handle_t h, int64_t M, int64_t N, const float* Z, int64_t ldz, const float* b,
                    float* H, int64_t ldh, int relu) {
    if (!h || M < 0 || N < 0) return SPLIT3_ERR_INVALID_VALUE;
    if (M == 0 || N == 0) return SPLIT3_OK;
    if (!Z || !H || ldz < N || ldh < N) return SPLIT3_ERR_INVALID_VALUE;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    return split3::launch_bias_act(h->stream, M, N, Z, ldz, b, H, ldh, relu != 0, h->num_sms) < 0 ? SPLIT3_ERR_CUDA
                                                                                                  : SPLIT3_OK;
}

int split3_relu_backward(split3_handle_t h, int64_t M, int64_t N, const float* dH, const float* H, float* dZ) {
    if (!h || M < 0 || N < 0) return SPLIT3_ERR_INVALID_VALUE;
    if (M == 0 || N == 0) return SPLIT3_OK;
    if (!dH || !H || !dZ) return SPLIT3_ERR_INVALID_VALUE;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    return split3::launch_relu_bwd(h->stream, M, N, dH, H, dZ, h->num_sms) < 0 ? SPLIT3_ERR_CUDA : SPLIT3_OK;
}

int split3_softmax_xent(split3_handle_t h, int64_t M, int64_t N, const float* L, const int32_t* labels, float* P,
                        float* dL, double* row_scratch, double* d_loss_sum) {
    if (!h || M < 0 || N < 0) return SPLIT3_ERR_INVALID_VALUE;
    if (M == 0 || N == 0) return SPLIT3_OK;
    if (!L || (d_loss_sum && (!row_scratch || !labels)) || (dL && !labels)) return SPLIT3_ERR_INVALID_VALUE;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    return split3::launch_softmax_xent(h->stream, M, N, L, labels, P, dL, d_loss_sum ? row_scratch : nullptr,
                                       d_loss_sum) < 0
               ? SPLIT3_ERR_CUDA
               : SPLIT3_OK;
}

int split3_bias_grad(split3_handle_t h, int64_t M, int64_t N, const float* dZ, float* db) {
    if (!h || M < 0 || N < 0) return SPLIT3_ERR_INVALID_VALUE;
    if (N == 0) return SPLIT3_OK;
    if (!dZ || !db) return SPLIT3_ERR_INVALID_VALUE;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    // the attached workspace is scratch between calls on this stream: the two-stage form uses it
    return split3::launch_col_sum(h->stream, M, N, dZ, db, h->num_sms, static_cast<float*>(h->ws), h->ws_bytes) < 0
               ? SPLIT3_ERR_CUDA
               : SPLIT3_OK;
}

int split3_sgd_update(split3_handle_t h, int64_t n, float* w, const float* g, float lr) {
    if (!h || n < 0) return SPLIT3_ERR_INVALID_VALUE;
    if (n == 0) return SPLIT3_OK;
    if (!w || !g) return SPLIT3_ERR_INVALID_VALUE;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    return split3::launch_sgd(h->stream, n, w, g, lr, h->num_sms) < 0 ? SPLIT3_ERR_CUDA : SPLIT3_OK;
}

int split3_set_schedule(split3_handle_t h, int group_m, int l2_policy_a, int l2_policy_b) {
    if (!h || group_m < 0 || group_m > 4096 || l2_policy_a < 0 || l2_policy_a > 2 || l2_policy_b < 0 ||
        l2_policy_b > 2)
        return SPLIT3_ERR_INVALID_VALUE;
    h->tune.group_m = group_m;
    h->tune.pol_a = l2_policy_a;
    h->tune.pol_b = l2_policy_b;
    return SPLIT3_OK;
}

int split3_set_wave_sync(split3_handle_t h, int enable) {
    if (!h) return SPLIT3_ERR_INVALID_VALUE;
    h->wave_sync = enable != 0;
    return SPLIT3_OK;
}

int split3_debug_read(uint64_t* out8, int reset) {
    if (!out8) return SPLIT3_ERR_INVALID_VALUE;
    const int r = split3::gemm3_debug_read(reinterpret_cast<unsigned long long*>(out8), reset);
    return r > 0 ? SPLIT3_OK : (r == 0 ? SPLIT3_ERR_NOT_IMPLEMENTED : SPLIT3_ERR_CUDA);
}

int split3_debug_fault(int fault) {
    if (fault < 0 || fault > 1) return SPLIT3_ERR_INVALID_VALUE;
    const int r = split3::gemm3_debug_fault(fault);
    return r > 0 ? SPLIT3_OK : (r == 0 ? SPLIT3_ERR_NOT_IMPLEMENTED : SPLIT3_ERR_CUDA);
}

int split3_set_split_k(split3_handle_t h, int enable) {
    if (!h) return SPLIT3_ERR_INVALID_VALUE;
    h->split_k = enable != 0;
    return SPLIT3_OK;
}

int split3_set_max_sms(split3_handle_t h, int sms) {
    if (!h || sms < 0 || sms == 1 || (sms & 1)) return SPLIT3_ERR_INVALID_VALUE;
    h->max_sms = sms;
    return SPLIT3_OK;
}

int split3_set_fused_split(split3_handle_t h, int mode, int64_t max_m) {
    if (!h || mode < 0 || mode > 2 || max_m < 0) return SPLIT3_ERR_INVALID_VALUE;
    h->fuse_b = mode;
    if (max_m > 0) h->fuse_b_max_m = max_m;
    return SPLIT3_OK;
}

int split3_set_fold(split3_handle_t h, int mode) {
    if (!h || mode < 0 || mode > 2) return SPLIT3_ERR_INVALID_VALUE;
    h->fold = mode;
    return SPLIT3_OK;
}

int split3_set_fused_split_a(split3_handle_t h, int mode, int64_t max_n) {
    if (!h || mode < 0 || mode > 2 || max_n < 0) return SPLIT3_ERR_INVALID_VALUE;
    h->fuse_a = mode;
    if (max_n > 0) h->fuse_a_max_n = max_n;
    return SPLIT3_OK;
}

int split3_set_promotion(split3_handle_t h, int kblocks) {
    if (!h || kblocks < 0 || kblocks > 1024) return SPLIT3_ERR_INVALID_VALUE;
    h->promo_kb = kblocks;
    return SPLIT3_OK;
}

int split3_timing_enable(split3_handle_t h, int enable) {
    if (!h) return SPLIT3_ERR_INVALID_VALUE;
    h->timing = enable != 0;
    return SPLIT3_OK;
}

int split3_timing_read(split3_handle_t h, double* split_ms, double* gemm_ms, int* calls) {
    if (!h) return SPLIT3_ERR_INVALID_VALUE;
    double s = 0.0, g = 0.0;
    int n = 0;
    for (size_t i = 0; i + 3 <= h->ev_used; i += 3) {
        float a = 0.f, b = 0.f;
        if (cudaEventSynchronize(h->ev_pool[i + 2]) != cudaSuccess ||
            cudaEventElapsedTime(&a, h->ev_pool[i], h->ev_pool[i + 1]) != cudaSuccess ||
            cudaEventElapsedTime(&b, h->ev_pool[i + 1], h->ev_pool[i + 2]) != cudaSuccess)
            return SPLIT3_ERR_CUDA;
        s += a;
        g += b;
        n++;
    }
    h->ev_used = 0;
    if (split_ms) *split_ms = s;
    if (gemm_ms) *gemm_ms = g;
    if (calls) *calls = n;
    return SPLIT3_OK;
}

// host pipeline: per-row-block scalars after the staging buffers
constexpr int kMaxHostBlocks = 32;
constexpr int kMaxPanels = 4;
static_assert(sizeof(((split3_host_layout*)nullptr)->blk_r0) / sizeof(int64_t) == kMaxHostBlocks &&
                  sizeof(((split3_host_layout*)nullptr)->pan_c0) / sizeof(int64_t) == kMaxPanels,
              "split3_host_layout arrays match the host pipeline's limits");
constexpr int kMaxPieceEvents = 64;   // ring of "C piece computed" events (ev_rows)
constexpr size_t kHostScalarBytes = 4 * 4 * (kMaxHostBlocks + kMaxPanels);

size_t split3_sgemm_host_workspace_size(int64_t M, int64_t N, int64_t K, uint32_t flags) {
    if (M < 0 || N < 0 || K < 0) return 0;
    return split3_sgemm_workspace_size(M, N, K, flags) + align256((size_t)M * K * 4) +
           align256((size_t)K * N * 4) + align256((size_t)M * N * 4) + kHostScalarBytes;
}

int split3_sgemm_host(split3_handle_t h, int64_t M, int64_t N, int64_t K, const float* A_host,
                      const float* B_host, float* C_host, uint32_t flags) {
    if (!h || M < 0 || N < 0 || K < 0) return SPLIT3_ERR_INVALID_VALUE;
    if (flags & ~SPLIT3_FLAGS_MASK) return SPLIT3_ERR_INVALID_VALUE;
    if ((flags & SPLIT3_ONE_TERM) && (flags & SPLIT3_FOUR_TERM)) return SPLIT3_ERR_INVALID_VALUE;
    if (M == 0 || N == 0) return SPLIT3_OK;
    if (!C_host || (K > 0 && (!A_host || !B_host))) return SPLIT3_ERR_INVALID_VALUE;
    if (!h->ws || h->ws_bytes < split3_sgemm_host_workspace_size(M, N, K, flags))
        return SPLIT3_ERR_WORKSPACE;
    if (set_dev(h)) return SPLIT3_ERR_CUDA;
    uint8_t* base = static_cast<uint8_t*>(h->ws) + split3_sgemm_workspace_size(M, N, K, flags);
    float* dA = reinterpret_cast<float*>(base);
    float* dB = reinterpret_cast<float*>(base + align256((size_t)M * K * 4));
    float* dC = reinterpret_cast<float*>(base + align256((size_t)M * K * 4) + align256((size_t)K * N * 4));
    if (K == 0 || (flags & (SPLIT3_CHECK_FINITE | SPLIT3_BF16X3))) {   // serial path
        if (K > 0 &&
            (cudaMemcpyAsync(dA, A_host, (size_t)M * K * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess ||
             cudaMemcpyAsync(dB, B_host, (size_t)K * N * 4, cudaMemcpyHostToDevice, h->stream) != cudaSuccess))
            return SPLIT3_ERR_CUDA;
        int st = split3_sgemm(h, M, N, K, dA, K, dB, N, dC, N, flags);
        if (st != SPLIT3_OK) return st;
        if (cudaMemcpyAsync(C_host, dC, (size_t)M * N * 4, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess ||
            cudaStreamSynchronize(h->stream) != cudaSuccess)
            return SPLIT3_ERR_CUDA;
        return SPLIT3_OK;
    }
    // Pipelined path.  B first (its split needs all of B), then A in row blocks:
    // each block is split with its OWN scale exponent as soon as it lands and multiplied while the
    // next block copies in, and C row blocks copy out underneath (copy engines run both directions).
    // A block exponent below the per-matrix one (reading R1) scales the block's planes, products and
    // C partial sums by an exact power of two, so C gets the per-matrix bits, unless the block holds
    // a nonzero |x| < 2^(sA-12) (fp16-subnormal planes): a check kernel flags such blocks after the
    // last copy and they are redone with the per-matrix scale before the call returns.
    if (!h->s_in) {
        if (cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_a, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_b, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_done, cudaEventDisableTiming) != cudaSuccess)
            return SPLIT3_ERR_CUDA;
        for (cudaEvent_t& e : h->ev_rows)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return SPLIT3_ERR_CUDA;
        for (cudaEvent_t& e : h->ev_arows)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return SPLIT3_ERR_CUDA;
        for (cudaEvent_t& e : h->ev_pan)
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return SPLIT3_ERR_CUDA;
    }
    cudaStream_t s0 = h->stream;
    // row blocks: multiples of the 256-row pair tile, each >= 2 waves of tiles (more blocks shorten
    // the exposed tail: the last block's split + GEMM + copy-out)
    const int64_t tiles_n = (N + 255) / 256;
    int nblk = 1;
    if (h->host_blocks > 0) {
        nblk = h->host_blocks;
    } else {
        while (nblk < 16 && ((M / (2 * nblk)) / 256) * tiles_n >= h->num_sms / 2) nblk *= 2;
    }
    const int64_t rows_per = ((M + nblk - 1) / nblk + 255) / 256 * 256;
    // blocks (r0, rows): rows_per each (>= 1 wave of tiles; <= 16 blocks: the copy-out of C trails
    // the copy-in of A by about one block); with >= 4 blocks the first one is cut into 1/4 + 1/4 + 1/2
    // (the GEMMs, and so the copy-out, start a quarter block after B has landed) and the last
    // into 1/2 + 1/4 + 1/4 (short exposed tail: the last piece's split, GEMM and copy-out)
    int64_t blk_r0[kMaxHostBlocks], blk_mr[kMaxHostBlocks];
    const bool cut = h->host_blocks == 0 && M >= 4 * rows_per && rows_per % 1024 == 0;
    const int64_t q = rows_per / 4;
    nblk = 0;
    for (int64_t r0 = 0; r0 < M; r0 += rows_per) {
        const int64_t mr = std::min(rows_per, M - r0);
        if (cut && r0 == 0) {
            blk_r0[nblk] = 0; blk_mr[nblk++] = q;
            blk_r0[nblk] = q; blk_mr[nblk++] = q;
            blk_r0[nblk] = 2 * q; blk_mr[nblk++] = 2 * q;
        } else if (cut && r0 + rows_per == M) {
            blk_r0[nblk] = r0; blk_mr[nblk++] = 2 * q;
            blk_r0[nblk] = r0 + 2 * q; blk_mr[nblk++] = q;
            blk_r0[nblk] = r0 + 3 * q; blk_mr[nblk++] = q;
        } else {
            blk_r0[nblk] = r0; blk_mr[nblk++] = mr;
        }
    }
    Carve w = carve(h->ws, M, N, K);
    const bool b_mn = h->mn_major != 0;  // MN-major B planes (plain split) unless disabled
    const int64_t ldpb = b_mn ? w.ldpb_mn : w.ldpb;
    // 2-D schedule: with >= 4 A blocks and a wide B, B is copied in column panels interleaved with
    // the A blocks at equal byte rates, each panel split with its own exponent, and the C piece
    // (A block i, B panel j) is multiplied and copied out as soon as both have landed — C starts
    // leaving a fraction of B in, not after all of it (§5e).  Panels are multiples of 256 columns.
    int nbp = 1;
    if (b_mn && nblk >= 4 && h->host_blocks == 0 && N >= 4 * 1024)
        nbp = h->host_panels > 0 ? std::min(h->host_panels, kMaxPanels) : 2;
    const int64_t cols_per = ((N + nbp - 1) / nbp + 255) / 256 * 256;
    int64_t pan_c0[kMaxPanels], pan_nc[kMaxPanels];
    nbp = 0;
    for (int64_t c0 = 0; c0 < N; c0 += cols_per) {
        pan_c0[nbp] = c0;
        pan_nc[nbp++] = std::min(cols_per, N - c0);
    }
    // scalars after the staging buffers: per A block and per B panel max bits, min-nonzero bits,
    // exponents, redo flags
    uint8_t* sc = reinterpret_cast<uint8_t*>(dC) + align256((size_t)M * N * 4);
    constexpr int kSlots = kMaxHostBlocks + kMaxPanels;
    unsigned* maxblk = reinterpret_cast<unsigned*>(sc);
    unsigned* minblk = reinterpret_cast<unsigned*>(sc + 4 * kSlots);
    int32_t* sblk = reinterpret_cast<int32_t*>(sc + 8 * kSlots);
    int32_t* flags_d = reinterpret_cast<int32_t*>(sc + 12 * kSlots);
    unsigned* maxpan = maxblk + kMaxHostBlocks;
    unsigned* minpan = minblk + kMaxHostBlocks;
    int32_t* span = sblk + kMaxHostBlocks;
    // transfer order: B panel 0, A block 0, B panel 1, A block 1, ... until B is in, then the rest
    // of A (the first A blocks are the small quarter cuts: B still lands almost as early as in
    // one piece, while the first C pieces can already leave)
    int order[kMaxHostBlocks + kMaxPanels];
    int nitems = 0;
    {
        int next_pan = 0;
        order[nitems++] = -1 - next_pan++;
        for (int b = 0; b < nblk; b++) {
            order[nitems++] = b;
            if (next_pan < nbp) order[nitems++] = -1 - next_pan++;
        }
        while (next_pan < nbp) order[nitems++] = -1 - next_pan++;
    }
    // copy-in must not overwrite the staging buffers while an earlier call on s0 still reads them
    if (cudaEventRecord(h->ev_done, s0) != cudaSuccess || cudaStreamWaitEvent(h->s_in, h->ev_done, 0) != cudaSuccess)
        return SPLIT3_ERR_CUDA;
    for (int it = 0; it < nitems; it++) {
        const int x = order[it];
        if (x < 0) {
            const int j = -1 - x;
            if (cudaMemcpy2DAsync(dB + pan_c0[j], (size_t)N * 4, B_host + pan_c0[j], (size_t)N * 4, (size_t)pan_nc[j] * 4,
                                  (size_t)K, cudaMemcpyHostToDevice, h->s_in) != cudaSuccess ||
                cudaEventRecord(h->ev_pan[j], h->s_in) != cudaSuccess)
                return SPLIT3_ERR_CUDA;
        } else {
            const int64_t r0 = blk_r0[x], mr = blk_mr[x];
            if (cudaMemcpyAsync(dA + r0 * K, A_host + r0 * K, (size_t)mr * K * 4, cudaMemcpyHostToDevice, h->s_in) !=
                    cudaSuccess ||
                cudaEventRecord(h->ev_arows[x], h->s_in) != cudaSuccess)
                return SPLIT3_ERR_CUDA;
        }
    }
    int launches = 0, n;
    if (cudaMemsetAsync(h->ws, 0, 32, s0) != cudaSuccess || cudaMemsetAsync(maxblk, 0, 4 * kSlots, s0) != cudaSuccess ||
        cudaMemsetAsync(minblk, 0xFF, 4 * kSlots, s0) != cudaSuccess)
        return SPLIT3_ERR_CUDA;
    // every piece takes the whole problem's accumulator (folded or not): the device call's bits
    const int fold_whole = split3::gemm3_fold_chosen(M, N, K, terms_of(flags), h->fold) ? 2 : 0;
    auto gemm_piece = [&](int b, int j, const int32_t* d_sA, const int32_t* d_sB) {
        const int64_t r0 = blk_r0[b], mr = blk_mr[b], c0 = pan_c0[j], nc = pan_nc[j];
        int err = 0;
        // MN-major B planes: columns [c0, c0 + nc) of the K x N planes; K-major (one panel): all
        int r = split3::launch_gemm3(s0, mr, nc, K, w.A1 + r0 * w.ldpa, w.A2 + r0 * w.ldpa, w.ldpa, d_sA, w.B1t + c0,
                                     w.B2t + c0, ldpb, d_sB, dC + r0 * N + c0, N, terms_of(flags), gemm_sms(h),
                                     h->promo_kb, h->wave_sync ? h->d_counters : nullptr, h->tune, nullptr, 0, &err,
                                     nullptr, nullptr, b_mn ? 1 : 0, nullptr, 0, nullptr, 0, fold_whole);
        return r < 0 ? -(err ? err : SPLIT3_ERR_CUDA) : r;
    };
    auto copy_out = [&](int b, int j, cudaStream_t st) {
        const int64_t r0 = blk_r0[b], mr = blk_mr[b], c0 = pan_c0[j], nc = pan_nc[j];
        return cudaMemcpy2DAsync(C_host + r0 * N + c0, (size_t)N * 4, dC + r0 * N + c0, (size_t)N * 4, (size_t)nc * 4,
                                 (size_t)mr, cudaMemcpyDeviceToHost, st) == cudaSuccess;
    };
    bool have_a[kMaxHostBlocks] = {false}, have_b[kMaxPanels] = {false};
    int nev = 0;
    auto piece = [&](int b, int j) {      // GEMM of (block b, panel j), then its copy-out on s_out
        int r = gemm_piece(b, j, sblk + b, span + j);
        if (r < 0) return r;
        launches += r;
        cudaEvent_t e = h->ev_rows[nev++ % kMaxPieceEvents];
        if (cudaEventRecord(e, s0) != cudaSuccess || cudaStreamWaitEvent(h->s_out, e, 0) != cudaSuccess ||
            !copy_out(b, j, h->s_out))
            return -SPLIT3_ERR_CUDA;
        return 0;
    };
    for (int it = 0; it < nitems; it++) {
        const int x = order[it];
        if (x < 0) {   // B panel j: max/min, split with its own exponent, then its pieces
            const int j = -1 - x;
            const float* Bp = dB + pan_c0[j];
            if (cudaStreamWaitEvent(s0, h->ev_pan[j], 0) != cudaSuccess) return SPLIT3_ERR_CUDA;
            if ((n = split3::launch_maxmin2d(s0, K, pan_nc[j], Bp, N, maxpan + j, minpan + j, h->num_sms)) < 0)
                return SPLIT3_ERR_CUDA;
            launches += n;
            const float* pmax = reinterpret_cast<const float*>(maxpan + j);
            if ((n = b_mn ? split3::launch_split(s0, K, pan_nc[j], Bp, N, pmax, w.B1t + pan_c0[j], w.B2t + pan_c0[j],
                                                 ldpb, span + j, h->num_sms)
                          : split3::launch_split_t(s0, K, N, dB, N, pmax, w.B1t, w.B2t, ldpb, span + j, h->num_sms)) < 0)
                return SPLIT3_ERR_CUDA;
            launches += n;
            have_b[j] = true;
            for (int b = 0; b < nblk; b++)
                if (have_a[b] && (n = piece(b, j)) < 0) return -n;
        } else {       // A block b: max/min, split with its own exponent, then its pieces
            const int b = x;
            const int64_t r0 = blk_r0[b], mr = blk_mr[b];
            if (cudaStreamWaitEvent(s0, h->ev_arows[b], 0) != cudaSuccess) return SPLIT3_ERR_CUDA;
            const float* Ab = dA + r0 * K;
            if ((n = split3::launch_maxmin(s0, mr * K, Ab, maxblk + b, minblk + b, h->num_sms)) < 0) return SPLIT3_ERR_CUDA;
            launches += n;
            if ((n = split3::launch_split(s0, mr, K, Ab, K, reinterpret_cast<const float*>(maxblk + b),
                                          w.A1 + r0 * w.ldpa, w.A2 + r0 * w.ldpa, w.ldpa, sblk + b, h->num_sms)) < 0)
                return SPLIT3_ERR_CUDA;
            launches += n;
            have_a[b] = true;
            for (int j = 0; j < nbp; j++)
                if (have_b[j] && (n = piece(b, j)) < 0) return -n;
        }
    }
    // per-matrix scales from the block / panel maxima, and the pieces to redo (rare)
    if (nblk > 1 || nbp > 1) {
        int32_t fa[kMaxHostBlocks] = {0}, fb[kMaxPanels] = {0};
        if ((n = split3::launch_host_scale_check(s0, maxblk, minblk, sblk, nblk, w.maxA, w.sA, flags_d)) < 0)
            return SPLIT3_ERR_CUDA;
        launches += n;
        if ((n = split3::launch_host_scale_check(s0, maxpan, minpan, span, nbp, w.maxB, w.sB, flags_d + kMaxHostBlocks)) < 0)
            return SPLIT3_ERR_CUDA;
        launches += n;
        if (cudaMemcpyAsync(fa, flags_d, (size_t)nblk * 4, cudaMemcpyDeviceToHost, s0) != cudaSuccess ||
            cudaMemcpyAsync(fb, flags_d + kMaxHostBlocks, (size_t)nbp * 4, cudaMemcpyDeviceToHost, s0) != cudaSuccess ||
            cudaStreamSynchronize(s0) != cudaSuccess || cudaStreamSynchronize(h->s_out) != cudaSuccess)
            return SPLIT3_ERR_CUDA;
        bool any = false;
        for (int b = 0; b < nblk; b++) any |= fa[b] != 0;
        for (int j = 0; j < nbp; j++) any |= fb[j] != 0;
        if (any) {
            for (int b = 0; b < nblk; b++) {   // re-split flagged blocks / panels with the per-matrix scale
                if (!fa[b]) continue;
                const int64_t r0 = blk_r0[b], mr = blk_mr[b];
                if ((n = split3::launch_split(s0, mr, K, dA + r0 * K, K, w.maxA, w.A1 + r0 * w.ldpa, w.A2 + r0 * w.ldpa,
                                              w.ldpa, w.sA, h->num_sms)) < 0)
                    return SPLIT3_ERR_CUDA;
                launches += n;
                h->host_redo++;
            }
            for (int j = 0; j < nbp; j++) {
                if (!fb[j]) continue;
                if ((n = split3::launch_split(s0, K, pan_nc[j], dB + pan_c0[j], N, w.maxB, w.B1t + pan_c0[j],
                                              w.B2t + pan_c0[j], ldpb, w.sB, h->num_sms)) < 0)
                    return SPLIT3_ERR_CUDA;
                launches += n;
                h->host_redo++;
            }
            for (int b = 0; b < nblk; b++)
                for (int j = 0; j < nbp; j++) {
                    if (!fa[b] && !fb[j]) continue;
                    if ((n = gemm_piece(b, j, fa[b] ? w.sA : sblk + b, fb[j] ? w.sB : span + j)) < 0) return -n;
                    launches += n;
                    if (!copy_out(b, j, s0)) return SPLIT3_ERR_CUDA;
                }
        }
    }
    if (cudaStreamSynchronize(h->s_out) != cudaSuccess || cudaStreamSynchronize(s0) != cudaSuccess)
        return SPLIT3_ERR_CUDA;
    h->last_launches = launches;
    split3_host_layout& L = h->host_layout;   // where the planes of this call live (introspection)
    L = split3_host_layout{};
    L.nblk = nblk;
    L.npan = nbp;
    for (int b = 0; b < nblk; b++) { L.blk_r0[b] = blk_r0[b]; L.blk_rows[b] = blk_mr[b]; }
    for (int j = 0; j < nbp; j++) { L.pan_c0[j] = pan_c0[j]; L.pan_cols[j] = pan_nc[j]; }
    L.A1 = w.A1; L.A2 = w.A2; L.ldpa = w.ldpa;
    L.B1 = w.B1t; L.B2 = w.B2t; L.ldpb = ldpb; L.b_mn = b_mn ? 1 : 0;
    L.d_sblk = sblk; L.d_span = span;
    L.d_redo = (nblk > 1 || nbp > 1) ? flags_d : nullptr;
    L.d_sA = w.sA; L.d_sB = w.sB;
    return SPLIT3_OK;
}

int split3_host_last_layout(split3_handle_t h, split3_host_layout* out) {
    if (!h || !out) return SPLIT3_ERR_INVALID_VALUE;
    *out = h->host_layout;
    return SPLIT3_OK;
}

}  // extern "C"
