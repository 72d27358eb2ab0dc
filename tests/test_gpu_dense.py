"""NEXT #1: transposes, pre-split operand reuse and split-K for dense-layer shapes.

Every variant is checked against the oracle (E_or <= 1e-6) AND, where the planes are the same
by construction, bitwise against the plain split3_sgemm on explicitly transposed copies.
"""
import numpy as np
import pytest
import torch

from workloads import numpy_matrix, torch_matrix

pytestmark = pytest.mark.gpu
E_OR_TOL = 1e-6


@pytest.fixture(scope="module")
def h():
    import paper_2011_11188_b200 as s3

    assert torch.cuda.is_available(), "GPU tests need a B200"
    return s3.Handle(0)


def _eor(C, Cs):
    return float(np.linalg.norm(C.astype(np.float64) - Cs) / np.linalg.norm(Cs))


@pytest.mark.parametrize("transA,transB", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(300, 200, 500), (1024, 768, 640), (65, 1030, 129)])
def test_transposes(h, orc, transA, transB, M, N, K):
    opA = numpy_matrix("uniform", M, K, seed=M + K)
    opB = numpy_matrix("loguni", K, N, seed=N + K)
    As = np.ascontiguousarray(opA.T) if transA else opA     # stored matrices
    Bs = np.ascontiguousarray(opB.T) if transB else opB
    C = h.sgemm_ex(torch.from_numpy(As).cuda(), torch.from_numpy(Bs).cuda(), transA=bool(transA),
                   transB=bool(transB))
    ref = h.sgemm(torch.from_numpy(opA).cuda(), torch.from_numpy(opB).cuda())
    assert torch.equal(C.view(torch.int32), ref.view(torch.int32))
    assert _eor(C.cpu().numpy(), orc.sgemm(opA, opB)) <= E_OR_TOL


@pytest.mark.parametrize("role,trans", [(0, False), (0, True), (1, False), (1, True)])
def test_presplit_planes_and_reuse(h, orc, role, trans):
    rows, cols = (384, 520) if role == 0 else (520, 700)      # op(X) shape
    opX = numpy_matrix("glorot", rows, cols, seed=role * 10 + int(trans))
    Xs = np.ascontiguousarray(opX.T) if trans else opX
    P = h.presplit(torch.from_numpy(Xs).cuda(), role=role, trans=trans)
    torch.cuda.synchronize()
    hi_o, lo_o, s_o = orc.split(opX)
    assert int(P.sexp.item()) == s_o
    ghi = P.hi.cpu().numpy().view(np.uint16)
    glo = P.lo.cpu().numpy().view(np.uint16)
    if role == 0:    # planes M x K
        assert np.array_equal(ghi[:, :cols], hi_o) and np.array_equal(glo[:, :cols], lo_o)
    else:            # planes N x K = op(X)^T
        assert np.array_equal(ghi[:, :rows], hi_o.T) and np.array_equal(glo[:, :rows], lo_o.T)
    # reuse: the pre-split operand gives the same bits as splitting in the call, twice
    if role == 0:
        other = torch_matrix("uniform", cols, 333, seed=9, device="cuda")
        ref = h.sgemm(torch.from_numpy(opX).cuda(), other)
        for _ in range(2):
            C = h.sgemm_ex(P, other)
            assert torch.equal(C.view(torch.int32), ref.view(torch.int32))
    else:
        other = torch_matrix("uniform", 333, rows, seed=9, device="cuda")
        ref = h.sgemm(other, torch.from_numpy(opX).cuda())
        for _ in range(2):
            C = h.sgemm_ex(other, P)
            assert torch.equal(C.view(torch.int32), ref.view(torch.int32))


@pytest.mark.parametrize("M,N,K", [(256, 1024, 1024), (256, 8192, 8192), (300, 500, 4096),
                                   (1024, 4096, 4096), (200, 300, 64)])
def test_split_k_parity_and_determinism(h, orc, M, N, K):
    """Few C tiles -> split-K (fixed-order reduction): oracle parity + bitwise repeatability."""
    A = numpy_matrix("uniform", M, K, seed=1)
    B = numpy_matrix("glorot", K, N, seed=2)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    C1 = h.sgemm(Ad, Bd).clone()
    n1 = h.last_launch_count()
    C2 = h.sgemm(Ad, Bd)
    assert torch.equal(C1.view(torch.int32), C2.view(torch.int32))
    if M * N <= 300 * 1024:
        Cs = orc.sgemm(A, B)
    else:   # sampled oracle
        rows = np.arange(0, M, max(1, M // 40))
        cols = np.arange(0, N, max(1, N // 40))
        Cs, _, _ = orc.sgemm_sampled(A, B, rows, cols)
        C1 = C1[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()]
    assert _eor(C1.cpu().numpy(), Cs) <= E_OR_TOL, n1
    for four in (True,):
        C4 = h.sgemm(Ad, Bd, four_term=four)
        if M * N <= 300 * 1024:
            assert _eor(C4.cpu().numpy(), orc.sgemm(A, B, terms=4)) <= E_OR_TOL


def test_dense_layer_forward_backward(h, orc):
    """Y = X W, dX = dY W^T, dW = X^T dY with W pre-split once per role (MagmaDNN dense layer)."""
    batch, fin, fout = 512, 1024, 768
    X = numpy_matrix("uniform", batch, fin, seed=11)
    W = numpy_matrix("glorot", fin, fout, seed=12)
    dY = numpy_matrix("uniform", batch, fout, seed=13)
    Xd, Wd, dYd = (torch.from_numpy(v).cuda() for v in (X, W, dY))
    W_fwd = h.presplit(Wd, role=1)                 # op(B) = W
    W_bwd = h.presplit(Wd, role=1, trans=True)     # op(B) = W^T
    Y = h.sgemm_ex(Xd, W_fwd).cpu().numpy()
    dX = h.sgemm_ex(dYd, W_bwd).cpu().numpy()
    dW = h.sgemm_ex(Xd, dYd, transA=True).cpu().numpy()
    assert _eor(Y, orc.sgemm(X, W)) <= E_OR_TOL
    assert _eor(dX, orc.sgemm(dY, np.ascontiguousarray(W.T))) <= E_OR_TOL
    assert _eor(dW, orc.sgemm(np.ascontiguousarray(X.T), dY)) <= E_OR_TOL


def test_ex_check_finite_index_in_stored_matrix(h):
    import paper_2011_11188_b200 as s3

    A = torch.ones((20, 30), device="cuda")       # stored K x M for transA
    A[4, 7] = float("inf")
    with pytest.raises(s3.NotFiniteError) as ei:
        h.sgemm_ex(A, torch.ones((20, 5), device="cuda"), transA=True, check_finite=True)
    assert ei.value.index == 4 * 30 + 7


@pytest.mark.parametrize("M,N,K,kw", [(300, 200, 500, {}), (257, 1030, 129, {"four_term": True}),
                                      (256, 8192, 4096, {}), (700, 900, 1500, {"transA": True}),
                                      (1, 1, 1, {}), (2048, 2560, 128, {"one_term": True})])
def test_canaries_around_output_and_workspace(h, M, N, K, kw):
    """No write outside C (rows/cols around a strided view) or past the declared workspace size
    (compute-sanitizer is not available on this pool: guard regions instead)."""
    import ctypes

    import paper_2011_11188_b200.split3 as s3

    transA = kw.pop("transA", False)
    A = torch_matrix("uniform", K if transA else M, M if transA else K, seed=3, device="cuda")
    B = torch_matrix("loguni", K, N, seed=4, device="cuda")
    big = torch.full((M + 16, N + 12), 12345.0, device="cuda")
    C = big[8:8 + M, 4:4 + N]
    flags = (s3.FOUR_TERM if kw.get("four_term") else 0) | (s3.ONE_TERM if kw.get("one_term") else 0)
    need = h.workspace_size(M, N, K, flags)
    ws = torch.full((need + 4096,), 0x5A, dtype=torch.uint8, device="cuda")
    st = h._lib.split3_sgemm_set_workspace(h._h, ctypes.c_void_p(ws.data_ptr()), need)
    assert st == 0
    h._ws = ws      # keep alive; the binding will not shrink it
    try:
        h.sgemm_ex(A, B, transA=transA, out=C, **kw)
        torch.cuda.synchronize()
        assert torch.all(ws[need:] == 0x5A)
        outside = big.clone()
        outside[8:8 + M, 4:4 + N] = 12345.0          # everything but C must still be the canary
        assert torch.all(outside == 12345.0)
        assert torch.isfinite(C).all()
    finally:
        h._ws = None
        h._ensure_ws(256)


def test_ex_error_paths(h):
    import ctypes

    import paper_2011_11188_b200.split3 as s3

    A = torch.ones((64, 32), device="cuda")
    B = torch.ones((32, 48), device="cuda")
    PB = h.presplit(B, role=1)
    PA = h.presplit(A, role=0)
    with pytest.raises(ValueError):                      # planes split for the other role
        h.sgemm_ex(PB, B)
    with pytest.raises(s3.Split3Error) as ei:            # bf16x3 takes fp32 operands only
        h.sgemm_ex(A, PB, bf16x3=True)
    assert ei.value.status == s3.ERR_NOT_IMPLEMENTED
    with pytest.raises(s3.Split3Error) as ei:            # exclusive flags
        h.sgemm_ex(A, B, bf16x3=True, four_term=True)
    assert ei.value.status == s3.ERR_INVALID_VALUE
    lib = s3.load()
    hi = torch.empty((48, 32), dtype=torch.int16, device="cuda")
    sx = torch.zeros(1, dtype=torch.int32, device="cuda")
    # ldp not a multiple of 8 / smaller than K / bad role
    assert lib.split3_presplit(h._h, 1, 32, 48, B.data_ptr(), 48, 0, hi.data_ptr(), hi.data_ptr(), 30, sx.data_ptr()) \
        == s3.ERR_INVALID_VALUE
    assert lib.split3_presplit(h._h, 2, 32, 48, B.data_ptr(), 48, 0, hi.data_ptr(), hi.data_ptr(), 32, sx.data_ptr()) \
        == s3.ERR_INVALID_VALUE
    assert lib.split3_presplit(h._h, 1, 32, 48, B.data_ptr(), 47, 0, hi.data_ptr(), hi.data_ptr(), 32, sx.data_ptr()) \
        == s3.ERR_INVALID_VALUE
    # a pre-split A with pre-split B works and equals the fp32 call
    C = h.sgemm_ex(PA, PB)
    assert torch.equal(C, h.sgemm(A, B))
    # check-finite under bf16x3 reports the index in the stored matrix
    A2 = A.clone()
    A2[5, 7] = float("nan")
    with pytest.raises(s3.NotFiniteError) as ei:
        h.sgemm_ex(A2, B, bf16x3=True, check_finite=True)
    assert ei.value.index == 5 * 32 + 7
    del ctypes
