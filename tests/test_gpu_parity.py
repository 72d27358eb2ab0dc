"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle, element by element.

Bars (BASELINE.json north_star):
  * planes: bit-exact vs oracle/;  max-abs and scale exponent: exact;
  * C: ||C - C_split||_F / ||C_split||_F <= 1e-6  (C_split: oracle's fp64 split emulation)
       ||C - C64||_F / (||A||_F ||B||_F) <= 2e-6  (C64: oracle's fp64 GEMM)
  * integer inputs {-2..2}: C == exact product, bitwise.
"""
import json
import os

import numpy as np
import pytest
import torch

from split3_bounds import _assert_elementwise, _elementwise_bound  # noqa: F401
from workloads import numpy_matrix, torch_matrix

pytestmark = pytest.mark.gpu

E_OR_TOL = 1e-6
E64_TOL = 2e-6
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


@pytest.fixture(scope="module")
def h():
    import paper_2011_11188_b200 as s3

    assert torch.cuda.is_available(), "GPU tests need a B200"
    return s3.Handle(0)


def _planes_np(t, rows, cols):
    return t[:rows, :cols].cpu().numpy().view(np.uint16)


def _gpu_split(h, X, transpose):
    d_max = torch.zeros(1, dtype=torch.float32, device="cuda")
    h.maxabs(X, d_max)
    hi, lo, sexp = h.split(X, d_max, transpose=transpose)
    torch.cuda.synchronize()
    return hi, lo, int(sexp.item()), float(d_max.item())


def _metrics(C, Csplit, C64, A, B):
    C = C.astype(np.float64)
    e_or = np.linalg.norm(C - Csplit) / max(np.linalg.norm(Csplit), 1e-300)
    e64 = np.linalg.norm(C - C64) / max(np.linalg.norm(A.astype(np.float64)) * np.linalg.norm(B.astype(np.float64)), 1e-300)
    e64rel = np.linalg.norm(C - C64) / max(np.linalg.norm(C64), 1e-300)
    return e_or, e64, e64rel


# ----------------------------------------------------------- a1 + a2: planes -----

SPLIT_SHAPES = [(1, 1), (3, 5), (64, 64), (65, 129), (200, 333), (256, 1000), (1000, 72)]


@pytest.mark.parametrize("kind", ["uniform", "loguni", "glorot", "int2", "fp16"])
@pytest.mark.parametrize("shape", SPLIT_SHAPES)
def test_planes_bit_exact(h, orc, kind, shape):
    rows, cols = shape
    X = numpy_matrix(kind, rows, cols, seed=rows * 7 + cols)
    hi_o, lo_o, s_o = orc.split(X)
    Xd = torch.from_numpy(X).cuda()
    for transpose in (False, True):
        hi, lo, s, m = _gpu_split(h, Xd, transpose)
        assert m == float(np.max(np.abs(X)))
        assert s == s_o
        if transpose:
            assert np.array_equal(_planes_np(hi, cols, rows), hi_o.T)
            assert np.array_equal(_planes_np(lo, cols, rows), lo_o.T)
        else:
            assert np.array_equal(_planes_np(hi, rows, cols), hi_o)
            assert np.array_equal(_planes_np(lo, rows, cols), lo_o)


@pytest.mark.parametrize("scale", [2.0 ** -20, 1.0, 2.0 ** 14, 2.0 ** -126, 2.0 ** 100])
def test_planes_scale_family(h, orc, scale):
    X = (numpy_matrix("uniform", 97, 131, seed=3) * np.float32(scale)).astype(np.float32)
    hi_o, lo_o, s_o = orc.split(X)
    for transpose in (False, True):
        hi, lo, s, _ = _gpu_split(h, torch.from_numpy(X).cuda(), transpose)
        assert s == s_o
        got_hi = _planes_np(hi, 131, 97).T if transpose else _planes_np(hi, 97, 131)
        got_lo = _planes_np(lo, 131, 97).T if transpose else _planes_np(lo, 97, 131)
        assert np.array_equal(got_hi, hi_o) and np.array_equal(got_lo, lo_o)


def test_planes_strided_and_unaligned(h, orc):
    """Leading dimension > cols and a misaligned base: scalar paths, same bits."""
    big = numpy_matrix("loguni", 70, 103, seed=9)
    Xd = torch.from_numpy(big).cuda()
    sub = Xd[:, 1:100]            # ld = 103, base offset 4 bytes (not 16-B aligned)
    X = big[:, 1:100].copy()
    hi_o, lo_o, s_o = orc.split(X)
    for transpose in (False, True):
        hi, lo, s, _ = _gpu_split(h, sub, transpose)
        assert s == s_o
        got = _planes_np(hi, 99, 70).T if transpose else _planes_np(hi, 70, 99)
        assert np.array_equal(got, hi_o)
        got = _planes_np(lo, 99, 70).T if transpose else _planes_np(lo, 70, 99)
        assert np.array_equal(got, lo_o)


def test_maxabs_skips_nonfinite_and_reports_index(h):
    X = numpy_matrix("uniform", 50, 60, seed=1)
    X[7, 9] = np.nan
    X[30, 2] = np.inf
    Xd = torch.from_numpy(X).cuda()
    d_max = torch.zeros(1, dtype=torch.float32, device="cuda")
    d_bad = torch.full((1,), np.iinfo(np.int64).max, dtype=torch.int64, device="cuda")
    h.maxabs(Xd, d_max, d_bad)
    fin = np.isfinite(X)
    assert float(d_max.item()) == float(np.max(np.abs(X[fin])))
    assert int(d_bad.item()) == 7 * 60 + 9


# ------------------------------------------------------- a3 + a4: the product -----

GEMM_SHAPES = [(1, 1, 1), (64, 64, 64), (128, 128, 64), (200, 300, 100), (257, 129, 1000),
               (130, 390, 77), (512, 512, 512), (1024, 1024, 1024), (33, 1000, 2000)]


@pytest.mark.parametrize("terms", [3, 4, 1])
@pytest.mark.parametrize("shape", GEMM_SHAPES)
def test_sgemm_vs_oracle(h, orc, shape, terms):
    M, N, K = shape
    A = numpy_matrix("uniform", M, K, seed=M + 1)
    B = numpy_matrix("uniform", K, N, seed=N + 2)
    C = h.sgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(),
                four_term=terms == 4, one_term=terms == 1).cpu().numpy()
    Cs = orc.sgemm(A, B, terms=terms)
    C64 = orc.gemm64(A, B)
    e_or, e64, e64rel = _metrics(C, Cs, C64, A, B)
    assert e_or <= E_OR_TOL, (e_or, e64, e64rel)
    if terms != 1:
        assert e64 <= E64_TOL and e64rel <= 1e-6, (e_or, e64, e64rel)
    _assert_elementwise(orc, C, Cs, A, B, terms)     # every element, not only the norm


@pytest.mark.parametrize("kind", ["loguni", "glorot", "fp16"])
def test_sgemm_distributions(h, orc, kind):
    M, N, K = 192, 160, 700
    A = numpy_matrix(kind, M, K, seed=5)
    B = numpy_matrix(kind, K, N, seed=6)
    C = h.sgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()).cpu().numpy()
    Cs = orc.sgemm(A, B, terms=3)
    e_or, _, _ = _metrics(C, Cs, orc.gemm64(A, B), A, B)
    assert e_or <= E_OR_TOL
    _assert_elementwise(orc, C, Cs, A, B, 3)


@pytest.mark.parametrize("kind", ["uniform", "loguni"])
def test_full_4096_every_element_vs_oracle(h, orc, kind):
    """N = 4096 (configs[1] small size), launched as bench.py does: EVERY element of C against the
    oracle's full fp64 emulation (no sampling) — E_or, E64 and the per-element bound"""
    N = 4096
    A = torch_matrix(kind, N, N, seed=41, device="cuda")
    B = torch_matrix(kind, N, N, seed=42, device="cuda")
    C = h.sgemm(A, B).cpu().numpy()
    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    Cs = orc.sgemm(An, Bn, terms=3)
    C64 = orc.gemm64(An, Bn)
    e_or, e64, e64rel = _metrics(C, Cs, C64, An, Bn)
    worst = _assert_elementwise(orc, C, Cs, An, Bn, 3)
    rec = {"N": N, "kind": kind, "E_or": e_or, "E64": e64, "E64rel": e64rel, "max_err_over_bound": worst,
           "elements": N * N}
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"parity_full4096_{kind}.json"), "w") as f:
        json.dump(rec, f)
    print(rec)
    assert e_or <= E_OR_TOL, rec
    if kind == "uniform":
        assert e64 <= E64_TOL, rec


@pytest.mark.parametrize("M,N,K", [(64, 64, 64), (300, 200, 4096), (256, 256, 16384)])
def test_integer_inputs_bit_exact(h, M, N, K):
    """Entries in {-2..2}: A2 = B2 = 0, every partial sum is an integer < 2^24: exact."""
    A = numpy_matrix("int2", M, K, seed=1)
    B = numpy_matrix("int2", K, N, seed=2)
    exact = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float32)
    for terms in (3, 4, 1):
        C = h.sgemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(),
                    four_term=terms == 4, one_term=terms == 1).cpu().numpy()
        assert np.array_equal(C, exact)


def test_three_term_equals_one_term_when_residual_zero(h):
    """fp16-representable inputs: D_mid == 0, so 3-term C == 1-term C bitwise."""
    A = numpy_matrix("fp16", 200, 512, seed=1) * np.float32(2.0 ** -10)
    B = numpy_matrix("fp16", 512, 150, seed=2) * np.float32(2.0 ** -10)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    c3 = h.sgemm(Ad, Bd).cpu().numpy()
    c1 = h.sgemm(Ad, Bd, one_term=True).cpu().numpy()
    assert np.array_equal(c3.view(np.uint32), c1.view(np.uint32))


@pytest.mark.parametrize("shape", [(300, 200, 1000), (256, 256, 4096), (2304, 520, 640)])
@pytest.mark.parametrize("e", [-70, -60, 56])
def test_epilogue_scale_outside_fp32_normal_range(h, shape, e):
    """a4's final factor 2^(sA+sB) outside the fp32 normal range (the epilogue's fp64 path; the
    split-K reduction's too): A, B scaled by 2^e have the same planes as A, B (per-matrix power of
    two, R1), so C_e must equal RN32(C * 2^(2e)) bit for bit — one rounding of the exact product.
    e = -70 / -60: sA + sB ~ -170 / -150 (subnormal and flushed results); e = 56: ~ +82 (fast path,
    control).  Shapes: fused B (M <= 2048), a split-K single tile, whole tiles; TMA-store C and a
    strided C (scalar stores)."""
    M, N, K = shape
    A = numpy_matrix("uniform", M, K, seed=M + 7)
    B = numpy_matrix("uniform", K, N, seed=N + 8)
    f = np.float32(2.0 ** e)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    Ae, Be = torch.from_numpy(A * f).cuda(), torch.from_numpy(B * f).cuda()
    for terms in (3, 4, 1):
        kw = dict(four_term=terms == 4, one_term=terms == 1)
        C = h.sgemm(Ad, Bd, **kw).cpu().numpy()
        want = (C.astype(np.float64) * 2.0 ** (2 * e)).astype(np.float32)
        got = h.sgemm(Ae, Be, **kw).cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (terms, e)
        Cbig = torch.full((M, N + 3), 7.0, device="cuda")
        h.sgemm(Ae, Be, out=Cbig[:, 1:1 + N], **kw)
        assert np.array_equal(Cbig[:, 1:1 + N].cpu().numpy().view(np.uint32), want.view(np.uint32)), (terms, e)
    if e < 0:
        assert np.count_nonzero(want) > 0 and np.any(np.abs(want[want != 0]) < np.float32(2.0 ** -126))


def test_default_call_planes_vs_oracle(orc):
    """The planes the default call leaves in its workspace (A: M x K K-major, B: K x N MN-major,
    both split without a transpose; capi.cu carve) equal the oracle's bit for bit; the call is the
    two-matrix max-abs, the two splits and the GEMM (+ split-K reduction)"""
    import paper_2011_11188_b200 as s3

    hh = s3.Handle(0)
    M, N, K = 4100, 1028, 1032                 # not small, M > 4096: no fused B
    A = torch_matrix("loguni", M, K, seed=61, device="cuda")
    B = torch_matrix("loguni", K, N, seed=62, device="cuda")
    hh.sgemm(A, B)
    torch.cuda.synchronize()
    assert hh.last_path() == 0 and hh.last_launch_count() <= 5, (hh.last_path(), hh.last_launch_count())
    pl = s3.split3.plane_ld
    pa = (max(M * pl(K), K * pl(M)) * 2 + 255) // 256 * 256
    pb = (max(N * pl(K), K * pl(N)) * 2 + 255) // 256 * 256
    raw = hh._ws.view(torch.uint8)

    def plane(off, rows, ld, cols):
        return raw[off:off + rows * ld * 2].view(torch.int16).view(rows, ld)[:, :cols].cpu().numpy().view(np.uint16)

    a1, a2, _ = orc.split(A.cpu().numpy())
    b1, b2, _ = orc.split(B.cpu().numpy())
    assert np.array_equal(plane(256, M, pl(K), K), a1) and np.array_equal(plane(256 + pa, M, pl(K), K), a2)
    o = 256 + 2 * pa
    assert np.array_equal(plane(o, K, pl(N), N), b1) and np.array_equal(plane(o + pb, K, pl(N), N), b2)


def test_strided_operands_and_output(h, orc):
    M, N, K = 100, 90, 130
    Abig = torch.from_numpy(numpy_matrix("uniform", M, K + 6, seed=1)).cuda()
    Bbig = torch.from_numpy(numpy_matrix("uniform", K, N + 3, seed=2)).cuda()
    A, B = Abig[:, 2:2 + K], Bbig[:, :N]
    Cbig = torch.full((M, N + 5), 7.0, device="cuda")
    C = Cbig[:, 1:1 + N]
    h.sgemm(A, B, out=C)
    Cs = orc.sgemm(A.cpu().numpy(), B.cpu().numpy(), terms=3)
    e_or = np.linalg.norm(C.cpu().numpy() - Cs) / np.linalg.norm(Cs)
    assert e_or <= E_OR_TOL
    cb = Cbig.cpu().numpy()
    assert np.all(cb[:, 0] == 7.0) and np.all(cb[:, N + 1:] == 7.0)


def test_edge_cases(h):
    import paper_2011_11188_b200 as s3

    A = torch.ones((3, 0), device="cuda")
    B = torch.ones((0, 4), device="cuda")
    C = torch.full((3, 4), 5.0, device="cuda")
    h.sgemm(A, B, out=C)                                    # K == 0: zero-fill
    assert torch.all(C == 0)
    h.sgemm(torch.ones((0, 5), device="cuda"), torch.ones((5, 4), device="cuda"))   # M == 0
    z = h.sgemm(torch.zeros((70, 33), device="cuda"), torch.zeros((33, 20), device="cuda"))
    assert torch.all(z == 0)
    with pytest.raises(ValueError):
        h.sgemm(torch.ones((3, 4), device="cuda"), torch.ones((5, 4), device="cuda"))
    # check-finite: first offending index
    A = torch.ones((10, 10), device="cuda")
    A[3, 4] = float("nan")
    with pytest.raises(s3.NotFiniteError) as ei:
        h.sgemm(A, torch.ones((10, 6), device="cuda"), check_finite=True)
    assert ei.value.index == 34
    B = torch.ones((10, 6), device="cuda")
    B[2, 5] = float("inf")
    with pytest.raises(s3.NotFiniteError) as ei:
        h.sgemm(torch.ones((10, 10), device="cuda"), B, check_finite=True)
    assert ei.value.index == 100 + 17
    # without the flag, non-finite values propagate only to the rows/cols that touch them
    A = torch.ones((130, 64), device="cuda")
    A[5, 3] = float("inf")
    C = h.sgemm(A, torch.ones((64, 140), device="cuda")).cpu().numpy()
    assert not np.all(np.isfinite(C[5])) and np.all(np.isfinite(np.delete(C, 5, axis=0)))
    assert np.all(np.delete(C, 5, axis=0) == 64.0)


def test_capi_error_codes(h):
    import ctypes

    import paper_2011_11188_b200.split3 as s3

    lib = s3.load()
    hd = h._h
    assert lib.split3_sgemm(hd, 4, 4, 4, 1, 3, 1, 4, 1, 4, 0) == s3.ERR_INVALID_VALUE   # lda < K
    assert lib.split3_sgemm(hd, 4, 4, 4, 1, 4, 1, 4, 1, 4, 1 << 7) == s3.ERR_INVALID_VALUE   # flag
    assert lib.split3_sgemm(hd, -1, 4, 4, 1, 4, 1, 4, 1, 4, 0) == s3.ERR_INVALID_VALUE
    assert lib.split3_sgemm(hd, 4, 4, 4, None, 4, 1, 4, 1, 4, 0) == s3.ERR_INVALID_VALUE
    h2 = s3.Handle(0)
    A = torch.ones((64, 64), device="cuda")
    st = lib.split3_sgemm(h2._h, 64, 64, 64, A.data_ptr(), 64, A.data_ptr(), 64, A.data_ptr(), 64, 0)
    assert st == s3.ERR_WORKSPACE
    assert lib.split3_sgemm_set_workspace(h2._h, ctypes.c_void_p(A.data_ptr() + 4), 1024) == s3.ERR_INVALID_VALUE


def test_host_buffers_roundtrip(h, orc):
    A = numpy_matrix("uniform", 300, 200, seed=1)
    B = numpy_matrix("uniform", 200, 100, seed=2)
    C = h.sgemm_host(A, B)
    Cs = orc.sgemm(A, B)
    assert np.linalg.norm(C - Cs) / np.linalg.norm(Cs) <= E_OR_TOL


# ------------------------------------------------ tensor-core numerics probe -----

def _probe(h, a_vals, b_vals, K=64):
    """D_hi[0,0] for A1 row 0 = a_vals, B1 column 0 = b_vals (1-term, scales 2^0)."""
    M = N = 128
    A1 = np.zeros((M, K), np.float16)
    B1t = np.zeros((N, K), np.float16)
    A1[0, :len(a_vals)] = a_vals
    B1t[0, :len(b_vals)] = b_vals
    A1d = torch.from_numpy(A1.view(np.int16)).cuda()
    B1d = torch.from_numpy(B1t.view(np.int16)).cuda()
    z = torch.zeros(1, dtype=torch.int32, device="cuda")
    C = h.gemm_planes(M, N, K, A1d, A1d, z, B1d, B1d, z, one_term=True)
    return float(C[0, 0].item())


def test_tc_accumulation_probe(h):
    """Records how tcgen05 kind::f16 rounds its FP32 accumulation (DESIGN.md §3 R9).

    Values are (D - 1)/ulp(1).  Written to gpurun_out/tc_probe.json; asserts only what every
    plausible model agrees on (exact products, subnormal fp16 inputs not flushed).
    """
    u = 2.0 ** -23
    t = 2.0 ** -12
    res = {}
    res["P1_0.75ulp"] = (_probe(h, [1, t], [1, 1.5 * t]) - 1) / u
    res["P1n"] = (_probe(h, [-1, -t], [1, 1.5 * t]) + 1) / u
    res["P2_tie"] = (_probe(h, [1, t], [1, t]) - 1) / u
    q = 2.0 ** -13
    res["P3_1.875ulp"] = (_probe(h, [1] + [q] * 15, [1] + [q] * 15) - 1) / u
    res["P4_two_halves"] = (_probe(h, [1, t, t], [1, t, t]) - 1) / u
    a = [1] + [0] * 15 + [t]
    b = [1] + [0] * 15 + [1.5 * t]
    res["P5_cross_mma_0.75ulp"] = (_probe(h, a, b) - 1) / u
    a = [1] + [0] * 63 + [t]
    b = [1] + [0] * 63 + [1.5 * t]
    res["P5b_cross_stage_0.75ulp"] = (_probe(h, a, b, K=128) - 1) / u
    sub = _probe(h, [2.0 ** -24], [2.0 ** -24])
    res["P6_subnormal_product"] = sub
    # alignment width: 1 + 2^-(23+j) * 1.5 for j = 1..8 -> does the addend survive?
    for j in range(0, 9):
        small = 1.5 * 2.0 ** -(23 + j)
        # split small into two fp16 factors
        res[f"P7_align_j{j}"] = (_probe(h, [1, 2.0 ** -12], [1, small * 2 ** 12]) - 1) / u
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "tc_probe.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))
    assert sub == 2.0 ** -48
    assert res["P2_tie"] == 0.0


# --------------------------------------------- full size (bench configuration) -----

@pytest.mark.parametrize("N,terms", [(4096, 3), (4096, 4), (16384, 3), (16384, 4)])
def test_full_size_sampled_parity(h, orc, N, terms):
    """configs[1] sizes, launched exactly as bench.py does (16384 4-term: the folded accumulator);
    oracle on sampled outputs."""
    A = torch_matrix("uniform", N, N, seed=11, device="cuda")
    B = torch_matrix("uniform", N, N, seed=12, device="cuda")
    C = h.sgemm(A, B, four_term=terms == 4)
    torch.cuda.synchronize()
    rng = np.random.Generator(np.random.PCG64(N))
    R = 48
    rows = np.sort(rng.choice(N, R, replace=False))
    cols = np.sort(rng.choice(N, R, replace=False))
    An = A.cpu().numpy()
    Bn = B.cpu().numpy()
    Cs, sA, sB = orc.sgemm_sampled(An, Bn, rows, cols, terms=terms)
    Cg = C[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy().astype(np.float64)
    # fp64 reference on the sample
    C64 = An[rows].astype(np.float64) @ Bn[:, cols].astype(np.float64)
    e_or = np.linalg.norm(Cg - Cs) / np.linalg.norm(Cs)
    e64rel = np.linalg.norm(Cg - C64) / np.linalg.norm(C64)
    # E64 over the sample, normalised as the full metric would be (unbiased Frobenius estimate)
    scale = (N * N) / (R * R)
    e64 = np.sqrt(scale) * np.linalg.norm(Cg - C64) / (np.linalg.norm(An.astype(np.float64)) *
                                                      np.linalg.norm(Bn.astype(np.float64)))
    rec = {"N": N, "terms": terms, "E_or": e_or, "E64": e64, "E64rel": e64rel, "sA": sA, "sB": sB}
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"parity_N{N}_t{terms}.json"), "w") as f:
        json.dump(rec, f)
    print(rec)
    assert e_or <= E_OR_TOL, rec
    assert e64 <= E64_TOL, rec


def test_promotion_sweep(h, orc):
    """E_or vs the D_hi promotion period at K = 8192 (records gpurun_out/promo_sweep.json).

    The default period must meet the 1e-6 bar; longer periods must not be more accurate
    than shorter ones by more than noise (the truncation error grows with the chain length).
    """
    M, N, K = 256, 256, 8192
    A = numpy_matrix("uniform", M, K, seed=31)
    B = numpy_matrix("uniform", K, N, seed=32)
    Cs = orc.sgemm(A, B, terms=3)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    res = {}
    try:
        for p in (1, 2, 4, 8, 16, 1024):
            h.set_promotion(p)
            C = h.sgemm(Ad, Bd).cpu().numpy()
            res[p] = float(np.linalg.norm(C - Cs) / np.linalg.norm(Cs))
    finally:
        h.set_promotion(0)
    C = h.sgemm(Ad, Bd).cpu().numpy()
    res["default"] = float(np.linalg.norm(C - Cs) / np.linalg.norm(Cs))
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "promo_sweep.json"), "w") as f:
        json.dump(res, f, indent=1)
    print(res)
    assert res["default"] <= E_OR_TOL
    assert res[1] <= res[1024]


def test_schedule_knobs_do_not_change_bits(h):
    """Wave lockstep, raster group and L2 policies are scheduling only: C is bitwise identical."""
    M, N, K = 700, 900, 1500
    A = torch.from_numpy(numpy_matrix("uniform", M, K, seed=3)).cuda()
    B = torch.from_numpy(numpy_matrix("loguni", K, N, seed=4)).cuda()
    ref = h.sgemm(A, B).cpu().numpy().view(np.uint32)
    try:
        for wave, sched in ((False, (0, 0, 0)), (True, (1, 2, 1)), (True, (3, 1, 2)), (False, (16, 0, 0))):
            h.set_wave_sync(wave)
            h.set_schedule(*sched)
            got = h.sgemm(A, B).cpu().numpy().view(np.uint32)
            assert np.array_equal(got, ref), (wave, sched)
    finally:
        h.set_wave_sync(True)
        h.set_schedule(0, 0, 0)


def test_repeatable_bitwise(h):
    """Same inputs, same launch configuration: bitwise identical C (no atomics in the product)."""
    A = torch_matrix("uniform", 2048, 1536, seed=5, device="cuda")
    B = torch_matrix("uniform", 1536, 2304, seed=6, device="cuda")
    c1 = h.sgemm(A, B).clone()
    c2 = h.sgemm(A, B)
    assert torch.equal(c1.view(torch.int32), c2.view(torch.int32))


@pytest.mark.parametrize("M,N", [(256 * 37, 512), (256 * 74 - 100, 256)])
def test_host_pipeline_bitwise_equals_device(h, M, N):
    """split3_sgemm_host (copy streams, row-block GEMMs, overlapped copy-out) == split3_sgemm.

    Shapes with a multiple of 74 C tiles, so the device path splits no tile along K (split
    tiles sum K in another, also fixed, order) and the host path never does."""
    K = 700
    A = torch_matrix("uniform", M, K, seed=M, device="cuda")
    B = torch_matrix("loguni", K, N, seed=M + 1, device="cuda")
    ref = h.sgemm(A, B).cpu()
    Ah = A.cpu().pin_memory()
    Bh = B.cpu().pin_memory()
    Ch = torch.empty((M, N), dtype=torch.float32).pin_memory()
    for flags in (0, 0):   # twice: reuse of the handle's streams/events
        h.sgemm_host_ptr(M, N, K, Ah.data_ptr(), Bh.data_ptr(), Ch.data_ptr(), flags)
        assert torch.equal(Ch.view(torch.int32), ref.view(torch.int32))


def test_host_pipeline_bitwise_equals_device_folded_four_term():
    """A 4-term call of 8192^3 multiply-adds folds (split3_set_fold's default rule): the host
    pipeline's row-block GEMMs take the WHOLE problem's choice, so its C is the device call's bit
    for bit (device handle with split-K off: whole tiles, as the host pieces)"""
    import paper_2011_11188_b200 as s3

    n = 8192
    hd = s3.Handle(0)
    hd.set_split_k(False)
    A = torch_matrix("uniform", n, n, seed=3, device="cuda")
    B = torch_matrix("uniform", n, n, seed=4, device="cuda")
    ref = hd.sgemm(A, B, four_term=True).cpu()
    assert hd.last_path() & 16                      # SPLIT3_PATH_FOLD
    Ah, Bh = A.cpu().pin_memory(), B.cpu().pin_memory()
    Ch = torch.empty((n, n), dtype=torch.float32).pin_memory()
    hd.sgemm_host_ptr(n, n, n, Ah.data_ptr(), Bh.data_ptr(), Ch.data_ptr(), 1)   # SPLIT3_FOUR_TERM
    assert torch.equal(Ch.view(torch.int32), ref.view(torch.int32))


def test_planes_exhaustive_fp32_range(h, orc):
    """Every fp32 bit pattern with |x| < 2^15 (2 x 0x47000000 ~ 2.4e9 values, in 2^28-pattern
    chunks): GPU planes == oracle planes, bit for bit (the GPU cvt.rn.f16.f32 pin).
    Each chunk is split with its own max-abs scale on both sides."""
    chunk = 1 << 28
    checked = 0
    for sign in (0, 0x80000000):
        for start in range(0, 0x47000000, chunk):
            n = min(chunk, 0x47000000 - start)
            bits = torch.arange(start, start + n, dtype=torch.int64, device="cuda") + sign
            X = bits.to(torch.int32).view(torch.float32).view(n // 4096, 4096) if n % 4096 == 0 else None
            assert X is not None
            del bits
            hi, lo, s, _ = _gpu_split(h, X, transpose=False)
            hi_o, lo_o, s_o = orc.split(X.cpu().numpy())
            assert s == s_o
            assert np.array_equal(_planes_np(hi, X.shape[0], 4096), hi_o)
            assert np.array_equal(_planes_np(lo, X.shape[0], 4096), lo_o)
            checked += n
            del X, hi, lo
            torch.cuda.empty_cache()
    assert checked == 2 * 0x47000000


def test_planes_exhaustive_fp32_large(h, orc):
    """The rest of the finite fp32 patterns, 2^15 <= |x| <= FLT_MAX (2 x 0x38800000 ~ 1.9e9
    values): each 2^28-pattern chunk's max sets a large scale exponent (up to the s = 113 of
    FLT_MAX), so most of the chunk lands in the fp16 subnormal / zero range after the exact
    2^-s scaling — GPU planes == oracle planes, bit for bit, with the two pins above covering
    every finite fp32 pattern."""
    chunk = 1 << 28
    lo_pat, hi_pat = 0x47000000, 0x7F800000
    checked = 0
    for sign in (0, 0x80000000):
        for start in range(lo_pat, hi_pat, chunk):
            n = min(chunk, hi_pat - start)
            assert n % 4096 == 0
            bits = torch.arange(start, start + n, dtype=torch.int64, device="cuda") + sign
            X = bits.to(torch.int32).view(torch.float32).view(n // 4096, 4096)
            del bits
            hi, lo, s, _ = _gpu_split(h, X, transpose=False)
            hi_o, lo_o, s_o = orc.split(X.cpu().numpy())
            assert s == s_o
            assert np.array_equal(_planes_np(hi, X.shape[0], 4096), hi_o)
            assert np.array_equal(_planes_np(lo, X.shape[0], 4096), lo_o)
            checked += n
            del X, hi, lo
            torch.cuda.empty_cache()
    assert checked == 2 * (hi_pat - lo_pat)


@pytest.mark.parametrize("shape,kw", [((2048, 2048, 1024), {}), ((256, 1024, 4096), {}),
                                      ((700, 900, 1500), {"bf16x3": True})])
def test_cuda_graph_capture_replay(h, shape, kw):
    """split3_sgemm captured into a CUDA graph and replayed == eager, bitwise (wave-lockstep slot
    and max-abs ticket are capture-safe); replays interleaved with eager calls stay correct."""
    M, N, K = shape
    A = torch_matrix("uniform", M, K, seed=1, device="cuda")
    B = torch_matrix("uniform", K, N, seed=2, device="cuda")
    ref = h.sgemm(A, B, **kw).clone()
    C = torch.empty((M, N), device="cuda")
    h.sgemm(A, B, out=C, **kw)           # allocate the workspace outside the capture
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            h.sgemm(A, B, out=C, **kw)
    torch.cuda.current_stream().wait_stream(s)
    for _ in range(3):
        C.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(C.view(torch.int32), ref.view(torch.int32))
        eager = h.sgemm(A, B, **kw)
        assert torch.equal(eager.view(torch.int32), ref.view(torch.int32))


def test_wave_counter_many_launches(h):
    """100 back-to-back launches (the eager wave counter is resynchronised every 64) stay bitwise
    identical and fast (no lockstep timeouts)."""
    import time

    A = torch_matrix("uniform", 4096, 2048, seed=1, device="cuda")
    B = torch_matrix("uniform", 2048, 4096, seed=2, device="cuda")
    ref = h.sgemm(A, B).clone()
    C = torch.empty_like(ref)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(100):
        h.sgemm(A, B, out=C)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 100
    assert torch.equal(C.view(torch.int32), ref.view(torch.int32))
    assert dt < 2e-3, dt      # ~0.2 ms of work; a desynchronised counter would cost 0.2 ms per wave
