"""Host-buffer pipeline (split3_sgemm_host): A arrives in row blocks, each split with
its own scale exponent; a block whose exponent is below the per-matrix one (reading R1) gives the
per-matrix bits by exact power-of-two scaling unless it holds a nonzero |a| < 2^(sA-12), in which
case the library redoes it.  C must be BIT-identical to the one-block host call (per-matrix scale,
same whole-tile GEMM plan) in every case, and match the device-buffer call (whose small problems
may use split-K slices, another summation order) to the oracle tolerance."""
import os

import numpy as np
import pytest
import torch

import paper_2011_11188_b200 as s3
from workloads import numpy_matrix

pytestmark = pytest.mark.gpu


def _handle(blocks):
    old = os.environ.get("SPLIT3_HOST_BLOCKS")
    os.environ["SPLIT3_HOST_BLOCKS"] = str(blocks)
    try:
        return s3.Handle(0)
    finally:
        if old is None:
            os.environ.pop("SPLIT3_HOST_BLOCKS", None)
        else:
            os.environ["SPLIT3_HOST_BLOCKS"] = old


@pytest.fixture(scope="module")
def hb():
    return _handle(4)


@pytest.fixture(scope="module")
def hd():
    return _handle(1)     # one block: the per-matrix scale for all of A


def _device(hd, A, B, **kw):
    C1 = hd.sgemm_host(A, B, **kw)
    Cd = hd.sgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), **kw).cpu().numpy()
    fin = np.isfinite(Cd)
    assert np.array_equal(fin, np.isfinite(C1))
    if fin.any():
        d = Cd[fin].astype(np.float64)
        assert np.linalg.norm(C1[fin] - d) <= 1e-6 * max(np.linalg.norm(d), 1e-300)
    return C1


def _same(x, y):
    return np.array_equal(x.view(np.int32), y.view(np.int32))


@pytest.mark.parametrize("kw", [{}, {"four_term": True}, {"one_term": True}])
@pytest.mark.parametrize("M,N,K", [(2048, 512, 700), (1100, 300, 257), (1024, 1024, 64)])
def test_blocks_equal_device(hb, hd, M, N, K, kw):
    A = numpy_matrix("uniform", M, K, seed=40)
    B = numpy_matrix("glorot", K, N, seed=41)
    assert _same(hb.sgemm_host(A, B, **kw), _device(hd, A, B, **kw))


def test_block_exponents_differ_no_redo(hb, hd):
    """block 0 five binades below the rest: its planes are the per-matrix ones x 2^5 exactly"""
    M, N, K = 2048, 512, 700
    A = numpy_matrix("uniform", M, K, seed=42)
    A[:512] = np.sign(A[:512]) * np.maximum(np.abs(A[:512]), np.float32(2.0 ** -20))
    A[:512] *= 2.0 ** -5
    assert np.abs(A).min() >= 2.0 ** -27 and np.abs(A).max() >= 0.5   # nothing below 2^(sA-12), sA = -15
    B = numpy_matrix("loguni", K, N, seed=43)
    r0 = hb.host_redo_count()
    C = hb.sgemm_host(A, B)
    assert hb.host_redo_count() == r0
    assert _same(C, _device(hd, A, B))


@pytest.mark.parametrize("tiny", [2.0 ** -40, 2.0 ** -30, 1e-45])
def test_block_with_tiny_entry_is_redone(hb, hd, tiny):
    """a low-exponent block with a nonzero entry below 2^(sA-12) is redone with the per-matrix scale"""
    M, N, K = 2048, 512, 700
    A = numpy_matrix("uniform", M, K, seed=44)
    A[:512] *= 2.0 ** -5
    A[3, 5] = np.float32(tiny)
    A[100, 7] = -np.float32(tiny) * 3
    B = numpy_matrix("uniform", K, N, seed=45)
    r0 = hb.host_redo_count()
    C = hb.sgemm_host(A, B)
    assert hb.host_redo_count() == r0 + 1
    assert _same(C, _device(hd, A, B))


def test_wide_range_blocks(hb, hd):
    """log-uniform magnitudes (2^-20..2^20) in every block: exponents and tiny entries everywhere"""
    M, N, K = 2048, 384, 512
    A = numpy_matrix("loguni", M, K, seed=46)
    A[512:1024] *= 2.0 ** -30
    B = numpy_matrix("loguni", K, N, seed=47)
    assert _same(hb.sgemm_host(A, B), _device(hd, A, B))


def test_zero_and_nonfinite_blocks(hb, hd):
    """an all-zero block (exponent 0) and a block with Inf/NaN (skipped by the max, propagated)"""
    M, N, K = 2048, 256, 320
    A = numpy_matrix("uniform", M, K, seed=48)
    A[:512] = 0.0
    A[1500, 3] = np.inf
    A[1700, 9] = np.nan
    B = numpy_matrix("uniform", K, N, seed=49)
    C = hb.sgemm_host(A, B)
    Cd = _device(hd, A, B)
    assert _same(C, Cd)
    assert np.isnan(C[1700]).all() and not np.isfinite(C[1500]).any()


def test_auto_blocks_with_tail(hd):
    """automatic blocking (4 blocks, the last cut into 1/2 + 1/4 + 1/4) with differing block scales"""
    M, N, K = 8192, 16384, 320
    A = numpy_matrix("uniform", M, K, seed=50)
    A[2048:4096] *= 2.0 ** -3
    A[7000, 1] = np.float32(2.0 ** -45)       # a tiny entry in a tail block with the top exponent
    B = numpy_matrix("uniform", K, N, seed=51)
    h = s3.Handle(0)
    C = h.sgemm_host(A, B)
    assert h.last_launch_count() > 6 * 3          # 6 row blocks: max/min, split, GEMM each
    assert _same(C, hd.sgemm_host(A, B))


@pytest.mark.parametrize("case", ["plain", "b_panel_scaled", "b_tiny", "a_and_b_tiny"])
def test_2d_schedule_b_panels(hd, case):
    """automatic 2-D schedule (2 B column panels interleaved with the first A blocks, each panel
    split with its own exponent): bitwise equal to the one-block call, pieces redone when needed"""
    M, N, K = 8192, 16384, 256
    A = numpy_matrix("uniform", M, K, seed=56)
    B = numpy_matrix("uniform", K, N, seed=57)
    half = N // 2                                    # B panel 0
    if case != "plain":                              # panel 0 six binades below panel 1
        B[:, :half] = np.sign(B[:, :half]) * np.maximum(np.abs(B[:, :half]), np.float32(2.0 ** -20))
        B[:, :half] *= 2.0 ** -6
    if case in ("b_tiny", "a_and_b_tiny"):
        B[17, 100] = np.float32(2.0 ** -50)         # a tiny entry in the low-exponent panel
    if case == "a_and_b_tiny":
        A[:2048] = np.sign(A[:2048]) * np.maximum(np.abs(A[:2048]), np.float32(2.0 ** -20))
        A[:2048] *= 2.0 ** -4
        A[5, 5] = np.float32(2.0 ** -60)
    h = s3.Handle(0)
    r0 = h.host_redo_count()
    C = h.sgemm_host(A, B)
    redo = h.host_redo_count() - r0
    assert redo == {"plain": 0, "b_panel_scaled": 0, "b_tiny": 1, "a_and_b_tiny": 2}[case], redo
    assert _same(C, hd.sgemm_host(A, B))


def _dev_view(h, ptr, rows, ld, cols):
    """rows x cols int16 plane view (ld elements per row) of the handle's workspace at device ptr"""
    ws = h._ws
    off = ptr - ws.data_ptr()
    assert 0 <= off and off + rows * ld * 2 <= ws.numel()
    return ws[off:off + rows * ld * 2].view(torch.int16).view(rows, ld)[:, :cols].cpu().numpy().view(np.uint16)


def _dev_i32(h, ptr, n):
    ws = h._ws
    off = ptr - ws.data_ptr()
    return ws[off:off + 4 * n].view(torch.int32).cpu().numpy()


@pytest.mark.parametrize("case", ["uniform", "blocks_scaled", "tiny_redo", "loguni", "panels"])
def test_host_planes_vs_oracle(orc, case):
    """the planes the host pipeline multiplied (split3_host_last_layout): every A row block and B
    column panel bit-exact vs the ORACLE's split of that block with the exponent the pipeline used
    — its own R1 exponent, or the per-matrix one where the block was redone — and that choice
    itself recomputed from oracle.maxabs / oracle.scale_exp"""
    h = _handle(4)
    if case == "panels":
        h = s3.Handle(0)        # automatic blocks + 2 B panels (2-D schedule)
    M, N, K = (8192, 8192, 320) if case == "panels" else (2048, 512, 700)
    kind = "loguni" if case == "loguni" else "uniform"
    A = numpy_matrix(kind, M, K, seed=60)
    B = numpy_matrix("uniform" if case != "panels" else "loguni", K, N, seed=61)
    if case in ("blocks_scaled", "tiny_redo"):
        A[:512] *= np.float32(2.0 ** -6)
    if case == "tiny_redo":
        A[5, 9] = np.float32(2.0 ** -44)
    if case == "panels":
        B[:, N // 2:] *= np.float32(2.0 ** -9)
    h.sgemm_host(A, B)
    torch.cuda.synchronize()
    L = h.host_last_layout()
    assert L.nblk >= 1 and L.npan >= 1
    sA = orc.scale_exp(orc.maxabs(A)[0])
    sB = orc.scale_exp(orc.maxabs(B)[0])
    assert _dev_i32(h, L.d_sA, 1)[0] == sA and _dev_i32(h, L.d_sB, 1)[0] == sB
    sblk = _dev_i32(h, L.d_sblk, L.nblk)
    span = _dev_i32(h, L.d_span, L.npan)
    redo = _dev_i32(h, L.d_redo, 36) if L.d_redo else np.zeros(36, np.int32)

    def rule(X, s_mat):
        s_b = orc.scale_exp(orc.maxabs(np.ascontiguousarray(X))[0])
        a = np.abs(X.astype(np.float64))
        tiny = np.any((a > 0) & (a < 2.0 ** (s_mat - 12)))
        return s_b, bool(s_b != s_mat and tiny)

    A1 = _dev_view(h, L.A1, M, L.ldpa, K)
    A2 = _dev_view(h, L.A2, M, L.ldpa, K)
    n_redo = 0
    for b in range(L.nblk):
        r0, mr = L.blk_r0[b], L.blk_rows[b]
        blk = A[r0:r0 + mr]
        s_b, must_redo = rule(blk, sA)
        if L.d_redo:
            assert bool(redo[b]) == must_redo, (b, redo[b], must_redo)
        assert sblk[b] == s_b, (b, sblk[b], s_b)
        s_used = sA if (L.d_redo and redo[b]) else s_b
        n_redo += int(bool(L.d_redo) and bool(redo[b]))
        hi, lo, _ = orc.split(blk, s=s_used)
        assert np.array_equal(A1[r0:r0 + mr], hi) and np.array_equal(A2[r0:r0 + mr], lo), b
    assert L.b_mn == 1
    B1 = _dev_view(h, L.B1, K, L.ldpb, N)
    B2 = _dev_view(h, L.B2, K, L.ldpb, N)
    for j in range(L.npan):
        c0, nc = L.pan_c0[j], L.pan_cols[j]
        pan = np.ascontiguousarray(B[:, c0:c0 + nc])
        s_j, must_redo = rule(pan, sB)
        if L.d_redo:
            assert bool(redo[32 + j]) == must_redo, (j, must_redo)
        assert span[j] == s_j
        s_used = sB if (L.d_redo and redo[32 + j]) else s_j
        hi, lo, _ = orc.split(pan, s=s_used)
        assert np.array_equal(B1[:, c0:c0 + nc], hi) and np.array_equal(B2[:, c0:c0 + nc], lo), j
    if case == "tiny_redo":
        assert n_redo == 1
    if case == "panels":
        assert L.npan == 2 and L.nblk >= 4
