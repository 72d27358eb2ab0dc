"""Folded accumulator (split3_set_fold; SURVEY §8f NEXT #2's D_lo fold, generalised):
per 64-wide k-block one TMEM accumulator takes [A2*B2], then A1*B2 + A2*B1 entered with tcgen05's
scale-input-d (T <- P + 2^-11 T), then A1*B1 likewise, i.e. T = D_hi + 2^-11 D_mid [+ 2^-22 D_lo]
of Eq. A_2, promoted into the FP32 master every k-block.

Pins: the oracle (E_or, E64, the fold's per-element bound on every element); the dropped term:
C_4 - C_3 from the folded kernel reproduces the oracle's 2^-22 a1 b1 A2 B2 (so the 2^-11 scaling is
applied exactly twice to D_lo and once to D_mid); integer inputs are exact; fused B and the
separate split give the same bits through the folded kernel."""
import numpy as np
import pytest
import torch

import paper_2011_11188_b200 as s3
from split3_bounds import _assert_elementwise
from workloads import numpy_matrix, torch_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hf():
    h = s3.Handle(0)
    h.set_fold(2)            # 3- and 4-term calls folded (the default folds 4-term only)
    return h


@pytest.fixture(scope="module")
def hfs():
    h = s3.Handle(0)
    h.set_fold(2)
    h.set_fused_split(0)
    return h


def _bits(C):
    return C.view(torch.int32)


SHAPES = [(1, 1, 1), (64, 64, 64), (128, 128, 64), (200, 300, 100), (257, 129, 1000), (130, 390, 77),
          (512, 512, 512), (1024, 1024, 1024), (33, 1000, 2000), (2304, 2304, 1536)]


@pytest.mark.parametrize("terms", [3, 4])
@pytest.mark.parametrize("shape", SHAPES)
def test_fold_vs_oracle(hf, orc, shape, terms):
    M, N, K = shape
    A = numpy_matrix("uniform", M, K, seed=M + 11)
    B = numpy_matrix("uniform", K, N, seed=N + 12)
    C = hf.sgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), four_term=terms == 4).cpu().numpy()
    Cs = orc.sgemm(A, B, terms=terms)
    C64 = orc.gemm64(A, B)
    e_or = np.linalg.norm(C - Cs) / np.linalg.norm(Cs)
    e64 = np.linalg.norm(C - C64) / (np.linalg.norm(A.astype(np.float64)) * np.linalg.norm(B.astype(np.float64)))
    e64rel = np.linalg.norm(C - C64) / np.linalg.norm(C64)
    assert e_or <= 1e-6 and e64 <= 2e-6 and e64rel <= 1e-6, (e_or, e64, e64rel)
    _assert_elementwise(orc, C, Cs, A, B, terms, fold=True)


@pytest.mark.parametrize("kind", ["loguni", "glorot", "fp16"])
def test_fold_distributions(hf, orc, kind):
    M, N, K = 192, 160, 700
    A = numpy_matrix(kind, M, K, seed=5)
    B = numpy_matrix(kind, K, N, seed=6)
    for terms in (3, 4):
        C = hf.sgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), four_term=terms == 4).cpu().numpy()
        Cs = orc.sgemm(A, B, terms=terms)
        assert np.linalg.norm(C - Cs) / np.linalg.norm(Cs) <= 1e-6
        _assert_elementwise(orc, C, Cs, A, B, terms, fold=True)


def _exact_split_inputs(M, N, K, seed):
    """Entries in {+-16392, +-16408}: s = 0, x = A1 + 2^-11 A2 exactly with A1 in {16384, 16416},
    A2 = +-16384 (ties to even), all products and partial sums of a K <= 2 dot product — in every
    group order and after each 2^-11 scaling — exact in FP32 (<= 24 significant bits), and a
    dropped term 2^-22 A2 B2 of 2^6 per product against C as small as |x|*16."""
    rng = np.random.default_rng(seed)
    vals = np.array([16392, -16392, 16408, -16408], dtype=np.float32)
    return vals[rng.integers(0, 4, (M, K))], vals[rng.integers(0, 4, (K, N))]


@pytest.mark.parametrize("fold", [2, 0])
def test_fold_dropped_term_exact(orc, fold):
    """C_4 = A B exactly and C_3 = the oracle's 3-term value exactly (both kernels): the folded
    accumulator applies 2^-11 once to D_mid and twice to D_lo, bit for bit"""
    h = s3.Handle(0)
    h.set_fold(fold)
    M, N, K = 256, 384, 2
    A, B = _exact_split_inputs(M, N, K, seed=31)
    exact = A.astype(np.float64) @ B.astype(np.float64)
    assert np.array_equal(exact.astype(np.float32).astype(np.float64), exact)
    c3_oracle = orc.sgemm(A, B, terms=3)
    assert np.array_equal(c3_oracle.astype(np.float32).astype(np.float64), c3_oracle)
    assert np.count_nonzero(exact - c3_oracle) > M * N // 4       # the dropped term is visible
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    c4 = h.sgemm(Ad, Bd, four_term=True).cpu().numpy()
    c3 = h.sgemm(Ad, Bd).cpu().numpy()
    assert np.array_equal(c4, exact.astype(np.float32))
    assert np.array_equal(c3, c3_oracle.astype(np.float32))


def test_unfolded_four_term_still_available(orc):
    """set_fold(0): the 256 x 128-tile 4-term kernel with its own D_lo accumulator"""
    h = s3.Handle(0)
    h.set_fold(0)
    M, N, K = 300, 520, 3000
    A = numpy_matrix("uniform", M, K, seed=32)
    B = numpy_matrix("loguni", K, N, seed=33)
    C = h.sgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), four_term=True).cpu().numpy()
    Cs = orc.sgemm(A, B, terms=4)
    assert np.linalg.norm(C - Cs) / np.linalg.norm(Cs) <= 1e-6
    _assert_elementwise(orc, C, Cs, A, B, 4, fold=False)


@pytest.mark.parametrize("M,N,K", [(64, 64, 64), (300, 200, 4096), (256, 256, 16384)])
def test_fold_integer_inputs_exact(hf, M, N, K):
    A = numpy_matrix("int2", M, K, seed=1)
    B = numpy_matrix("int2", K, N, seed=2)
    exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float32)
    for terms in (3, 4):
        C = hf.sgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), four_term=terms == 4).cpu().numpy()
        assert np.array_equal(C, exact)


@pytest.mark.parametrize("M,N,K", [(256, 4096, 4096), (300, 200, 500), (2048, 2048, 2048), (7, 4096, 8192)])
def test_fold_fused_b_equals_separate(hf, hfs, M, N, K):
    A = torch_matrix("uniform", M, K, seed=23)
    B = torch_matrix("loguni", K, N, seed=24)
    C1 = hf.sgemm(A, B).clone()
    assert hf.last_path() & 1 or M > 2048
    C2 = hfs.sgemm(A, B)
    assert torch.equal(_bits(C1), _bits(C2))


@pytest.mark.parametrize("transA,transB", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_fold_transposes_and_split_k(hf, orc, transA, transB):
    M, N, K = 300, 520, 8192          # 4 tiles: every tile cut into K slices
    A = torch_matrix("uniform", K if transA else M, M if transA else K, seed=25)
    B = torch_matrix("uniform", N if transB else K, K if transB else N, seed=26)
    for terms in (3, 4):
        C = hf.sgemm_ex(A, B, transA=bool(transA), transB=bool(transB), four_term=terms == 4).cpu().numpy()
        An = (A.t() if transA else A).contiguous().cpu().numpy()
        Bn = (B.t() if transB else B).contiguous().cpu().numpy()
        Cs = orc.sgemm(An, Bn, terms=terms)
        assert np.linalg.norm(C - Cs) / np.linalg.norm(Cs) <= 1e-6
        _assert_elementwise(orc, C, Cs, An, Bn, terms, fold=True)


def test_fold_full_4096_every_element(hf, orc):
    N = 4096
    A = torch_matrix("uniform", N, N, seed=41, device="cuda")
    B = torch_matrix("uniform", N, N, seed=42, device="cuda")
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    for terms in (3, 4):
        C = hf.sgemm(A, B, four_term=terms == 4).cpu().numpy()
        Cs = orc.sgemm(An, Bn, terms=terms)
        assert np.linalg.norm(C - Cs) / np.linalg.norm(Cs) <= 1e-6
        _assert_elementwise(orc, C, Cs, An, Bn, terms, fold=True)


def test_fold_repeatable_and_graph(hf):
    M, N, K = 1024, 1024, 2048
    A = torch_matrix("uniform", M, K, seed=27)
    B = torch_matrix("uniform", K, N, seed=28)
    C0 = hf.sgemm(A, B, four_term=True).clone()
    for _ in range(3):
        assert torch.equal(_bits(hf.sgemm(A, B, four_term=True)), _bits(C0))
    C = torch.empty(M, N, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        hf.sgemm(A, B, out=C, four_term=True)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            hf.sgemm(A, B, out=C, four_term=True)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(_bits(C), _bits(C0))


@pytest.mark.parametrize("N", [8192, 16384])
def test_fold_accuracy_full_size(orc, N):
    """folded vs unfolded accumulator at full size (64 x 64 sampled outputs vs the oracle's 3- /
    4-term emulation and fp64): both within the tolerance, within 1.5x of each other — the fold
    rounds the mid group at the k-block sum's precision and promotes every k-block (K/64 RN adds
    instead of K/128); measured 8192: 2.27e-7 folded vs 2.38e-7, 16384: 3.11e-7 vs 2.78e-7
    (profiles/fold_accuracy_r02.json)"""
    import json
    import os

    A = torch_matrix("uniform", N, N, seed=11, device="cuda")
    B = torch_matrix("uniform", N, N, seed=12, device="cuda")
    rng = np.random.Generator(np.random.PCG64(N))
    R = 64
    rows = np.sort(rng.choice(N, R, replace=False))
    cols = np.sort(rng.choice(N, R, replace=False))
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    C64 = An[rows].astype(np.float64) @ Bn[:, cols].astype(np.float64)
    rec = {}
    for terms, fold in ((3, 0), (4, 0), (4, 2), (3, 2)):
        h = s3.Handle(0)
        h.set_fold(fold)
        C = h.sgemm(A, B, four_term=terms == 4)
        Cg = C[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy().astype(np.float64)
        Cs, _, _ = orc.sgemm_sampled(An, Bn, rows, cols, terms=terms)
        rec[f"t{terms}_fold{fold}"] = {"E_or": float(np.linalg.norm(Cg - Cs) / np.linalg.norm(Cs)),
                                       "E64rel": float(np.linalg.norm(Cg - C64) / np.linalg.norm(C64))}
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, f"fold_accuracy_N{N}.json"), "w") as f:
        json.dump(rec, f)
    for k, v in rec.items():
        assert v["E_or"] <= 1e-6 and v["E64rel"] <= 1e-6, (k, v)
    for t in (3, 4):
        a, b = rec[f"t{t}_fold2"]["E_or"], rec[f"t{t}_fold0"]["E_or"]
        assert max(a, b) <= 1.5 * min(a, b), rec


def test_fold_default_rule():
    """default handle: 4-term calls of >= 8192^3 multiply-adds fold (SPLIT3_PATH_FOLD), smaller
    4-term calls and every 3-term call do not"""
    h = s3.Handle(0)
    A = torch_matrix("uniform", 8192, 8192, seed=51)
    B = torch_matrix("uniform", 8192, 8192, seed=52)
    h.sgemm(A, B, four_term=True)
    assert h.last_path() & 16
    h.sgemm(A, B)
    assert not h.last_path() & 16
    h.sgemm(A[:4096].contiguous(), B, four_term=True)
    assert not h.last_path() & 16


def test_fold_validation(hf):
    assert s3.split3.load().split3_set_fold(hf._h, 3) == 1      # SPLIT3_ERR_INVALID_VALUE
    with pytest.raises(s3.Split3Error):
        hf.set_fold(-1)
