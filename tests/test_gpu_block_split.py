"""Block-scaled single-pass split (split3_set_block_scale, split3_split_blocks).

Every 128-row block of A and 128-column block of B is split with its own scale exponent (rule R1
on the block's max) in one pass over HBM; a block whose exponent is below the per-matrix one and
that holds a nonzero |x| < 2^(s_matrix - 12) keeps the per-matrix exponent.  Checked here:
  * the block planes bit-exact vs the oracle's split of each block with that exponent (the
    exponent rule itself recomputed from oracle.maxabs / oracle.scale_exp);
  * C bitwise equal to the per-matrix-scale path (block scaling off) for 1/3/4 terms, ragged
    shapes, split-K tails, differing block binades, blocks that need the per-matrix exponent,
    zero blocks, non-finite entries and CUDA-graph replays;
  * the oracle tolerance on top.
"""
import numpy as np
import pytest
import torch

from workloads import numpy_matrix, torch_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hb():
    """handle on which every non-tiny call takes the block-scaled path: the one-launch front end is
    off (SPLIT3_PREP_MAX=0, read when a stream's library handle is created, so it stays set for the
    module: the graph test's capture stream gets its own handle)"""
    import os

    import paper_2011_11188_b200 as s3

    old = os.environ.get("SPLIT3_PREP_MAX")
    os.environ["SPLIT3_PREP_MAX"] = "0"
    yield s3.Handle(0)
    if old is None:
        del os.environ["SPLIT3_PREP_MAX"]
    else:
        os.environ["SPLIT3_PREP_MAX"] = old


def _block_scaled(kind, rows, cols, seed, axis):
    """a matrix whose 128-blocks along `axis` (0: row blocks, 1: column blocks) have different binades"""
    X = numpy_matrix(kind, rows, cols, seed)
    nb = (X.shape[axis] + 127) // 128
    for b in range(nb):
        sl = (slice(128 * b, 128 * b + 128), slice(None)) if axis == 0 else (slice(None), slice(128 * b, 128 * b + 128))
        X[sl] *= np.float32(2.0 ** (-7 * (b % 4) + 3 * (b % 3)))
    return X


def _expected_exp(orc, block, s_mat):
    m, _ = orc.maxabs(np.ascontiguousarray(block))
    s_b = orc.scale_exp(m)
    a = np.abs(block[np.isfinite(block)].astype(np.float64))
    tiny = np.any((a > 0) & (a < 2.0 ** (s_mat - 12)))
    return s_mat if (s_b != s_mat and tiny) else s_b


CASES = [(300, 200, 1000, "uniform"), (128, 128, 64, "uniform"), (1, 1, 1, "uniform"), (257, 385, 333, "loguni"),
         (1024, 640, 2048, "glorot"), (200, 300, 100, "fp16"), (384, 256, 512, "int2"), (640, 520, 700, "blocks")]


@pytest.mark.parametrize("M,N,K,kind", CASES)
def test_block_planes_vs_oracle(hb, orc, M, N, K, kind):
    if kind == "blocks":
        A = _block_scaled("uniform", M, K, 1, 0)
        B = _block_scaled("loguni", K, N, 2, 1)
    else:
        A = numpy_matrix(kind, M, K, seed=M)
        B = numpy_matrix(kind, K, N, seed=N + 1)
    A1, A2, B1, B2, sblk, smat = hb.split_blocks(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    torch.cuda.synchronize()
    sblk, smat = sblk.cpu().numpy(), smat.cpu().numpy()
    sA, sB = orc.scale_exp(orc.maxabs(A)[0]), orc.scale_exp(orc.maxabs(B)[0])
    assert (smat[0], smat[1]) == (sA, sB)
    nbA = (M + 127) // 128
    A1n, A2n = A1.cpu().numpy().view(np.uint16), A2.cpu().numpy().view(np.uint16)
    B1n, B2n = B1.cpu().numpy().view(np.uint16), B2.cpu().numpy().view(np.uint16)
    for b in range(nbA):
        blk = A[128 * b:128 * b + 128]
        s = _expected_exp(orc, blk, sA)
        assert sblk[b] == s, (b, sblk[b], s)
        hi, lo, _ = orc.split(blk, s=s)
        assert np.array_equal(A1n[128 * b:128 * b + 128, :K], hi) and np.array_equal(A2n[128 * b:128 * b + 128, :K], lo)
    for b in range((N + 127) // 128):
        blk = np.ascontiguousarray(B[:, 128 * b:128 * b + 128])
        s = _expected_exp(orc, blk, sB)
        assert sblk[nbA + b] == s, (b, sblk[nbA + b], s)
        hi, lo, _ = orc.split(blk, s=s)
        w = blk.shape[1]
        assert np.array_equal(B1n[:, 128 * b:128 * b + w], hi) and np.array_equal(B2n[:, 128 * b:128 * b + w], lo)


def _both(hb, A, B, **kw):
    hb.set_block_scale(True)
    c1 = hb.sgemm(A, B, **kw).clone()
    hb.set_block_scale(False)
    c0 = hb.sgemm(A, B, **kw).clone()
    hb.set_block_scale(True)
    torch.cuda.synchronize()
    return c1, c0


@pytest.mark.parametrize("terms", [3, 4, 1])
@pytest.mark.parametrize("M,N,K,kind", CASES + [(2304, 1152, 777, "uniform"), (4096, 4096, 1024, "loguni")])
def test_block_scale_C_bitwise(hb, orc, M, N, K, kind, terms):
    if kind == "blocks":
        A = torch.from_numpy(_block_scaled("uniform", M, K, 1, 0)).cuda()
        B = torch.from_numpy(_block_scaled("loguni", K, N, 2, 1)).cuda()
    elif M * N > 4 << 20:
        A = torch_matrix(kind, M, K, seed=3)
        B = torch_matrix(kind, K, N, seed=4)
    else:
        A = torch.from_numpy(numpy_matrix(kind, M, K, seed=5)).cuda()
        B = torch.from_numpy(numpy_matrix(kind, K, N, seed=6)).cuda()
    c1, c0 = _both(hb, A, B, four_term=terms == 4, one_term=terms == 1)
    assert torch.equal(c1.view(torch.int32), c0.view(torch.int32))
    if M * N * K <= 1 << 30:
        Cs = orc.sgemm(A.cpu().numpy(), B.cpu().numpy(), terms=terms)
        e = np.linalg.norm(c1.cpu().numpy() - Cs) / max(np.linalg.norm(Cs), 1e-300)
        assert e <= 1e-6, e


def test_tiny_entries_force_matrix_exponent(hb, orc):
    """block 1 of A sits 5 binades below the matrix max and holds an entry 2^(s_A - 20): its
    fp16-subnormal rounding would differ under the block exponent, so it is re-split with s_A
    (the fix-up kernel); block 2 is as low but has no tiny entries and keeps its own exponent"""
    M, N, K = 512, 384, 640
    A = numpy_matrix("uniform", M, K, seed=7)
    A[128:384] *= np.float32(2.0 ** -5)
    sA = orc.scale_exp(orc.maxabs(A)[0])
    A[130, 17] = np.float32(2.0 ** (sA - 20))
    A[131, 18] = np.float32(-(2.0 ** (sA - 13)) * 1.5)
    B = numpy_matrix("glorot", K, N, seed=8)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    *_, sblk, smat = hb.split_blocks(Ad, Bd)
    sblk = sblk.cpu().numpy()
    assert sblk[1] == sA and sblk[2] == sA - 5 and sblk[0] == sA
    c1, c0 = _both(hb, Ad, Bd)
    assert torch.equal(c1.view(torch.int32), c0.view(torch.int32))


def test_zero_and_nonfinite_blocks(hb):
    M, N, K = 512, 512, 384
    A = numpy_matrix("uniform", M, K, seed=9)
    A[128:256] = 0.0                       # a zero block: exponent 0, zero planes
    A[300, 5] = np.inf
    B = numpy_matrix("uniform", K, N, seed=10)
    B[7, 200] = np.nan
    c1, c0 = _both(hb, torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda())
    a, b = c1.cpu().numpy(), c0.cpu().numpy()
    assert np.array_equal(np.isfinite(a), np.isfinite(b))
    fin = np.isfinite(a)
    assert np.array_equal(a[fin].view(np.uint32), b[fin].view(np.uint32))
    assert not fin[300].any() and not fin[:, 200].any() and fin.sum() == (M - 1) * (N - 1)


def test_graph_replay_changing_scales(hb):
    """captured block-scaled calls replay with new inputs (other binades, other flagged blocks)"""
    M, N, K = 1024, 768, 512
    A = torch_matrix("uniform", M, K, seed=11)
    B = torch_matrix("uniform", K, N, seed=12)
    C = torch.empty((M, N), device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        hb.sgemm(A, B, out=C)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            hb.sgemm(A, B, out=C)
    for t in range(4):
        An = torch_matrix("loguni" if t % 2 else "uniform", M, K, seed=20 + t)
        Bn = torch_matrix("uniform", K, N, seed=30 + t)
        An[128 * t:128 * t + 128] *= 2.0 ** (-6 - t)
        if t == 3:
            An[128 * t + 1, 3] = 2.0 ** -60      # forces the fix-up path inside the replay
        A.copy_(An)
        B.copy_(Bn)
        g.replay()
        torch.cuda.synchronize()
        hb.set_block_scale(False)
        ref = hb.sgemm(A, B)
        hb.set_block_scale(True)
        torch.cuda.synchronize()
        assert torch.equal(C.view(torch.int32), ref.view(torch.int32)), t


def test_full_size_block_split_matches_per_matrix(hb):
    """the bench's configs[1] size: the block-scaled call (default) == the two-pass call, bitwise"""
    N = 16384
    A = torch_matrix("uniform", N, N, seed=0)
    B = torch_matrix("uniform", N, N, seed=1)
    c1, c0 = _both(hb, A, B)
    assert torch.equal(c1.view(torch.int32), c0.view(torch.int32))
