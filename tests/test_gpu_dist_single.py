"""The 2-D tile driver (dist.py) on ONE GPU over a one-rank NCCL group: exercises
CudaOps (max-abs + all_reduce(MAX), plane splits, all-gathers, per-row-block GEMMs on a side
stream) with the real kernels.  Multi-rank logic is covered by tests/test_dist_gloo.py on CPU."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_one_rank():
    import torch.distributed as dist

    created = False
    if not dist.is_initialized():
        dist.init_process_group("nccl", store=dist.HashStore(), world_size=1, rank=0,
                                device_id=torch.device("cuda", 0))
        created = True
    yield
    if created:
        dist.destroy_process_group()


def _oracle_errors(C, A, B, terms=3, R=192):
    """E_or / E64 of C on R x R seeded sampled outputs (oracle: scales from the whole matrices)"""
    import oracle

    An, Bn = A.cpu().numpy(), B.cpu().numpy()
    rng = np.random.default_rng(11)
    rows = np.sort(rng.choice(An.shape[0], size=min(R, An.shape[0]), replace=False))
    cols = np.sort(rng.choice(Bn.shape[1], size=min(R, Bn.shape[1]), replace=False))
    Cs, _, _ = oracle.sgemm_sampled(An, Bn, rows, cols, terms=terms)
    C64 = oracle.gemm64(np.ascontiguousarray(An[rows]), np.ascontiguousarray(Bn[:, cols]))
    T = C.cpu().double().numpy()[np.ix_(rows, cols)]
    e_or = float(np.linalg.norm(T - Cs) / np.linalg.norm(Cs))
    e64 = float(np.linalg.norm(T - C64) / (np.linalg.norm(An[rows].astype(np.float64)) *
                                          np.linalg.norm(Bn[:, cols].astype(np.float64))))
    return e_or, e64


@pytest.mark.parametrize("n,kw", [(1024, {}), (2304, {}), (1536, {"four_term": True})])
def test_tile_gemm_one_rank_matches_single_call(nccl_one_rank, n, kw):
    """sharded-input driver on a one-rank NCCL group: bitwise the one-GPU call with split-K off,
    and within the oracle tolerance"""
    import paper_2011_11188_b200 as s3
    from paper_2011_11188_b200.dist import TileGemm

    h = s3.Handle(0)
    tg = TileGemm(h, n, 1, 0, seed=5, **kw)
    C = tg.run()
    torch.cuda.synchronize()
    assert C.shape == (n, n)
    h1 = s3.Handle(0)
    h1.set_split_k(False)
    ref = h1.sgemm(tg.A_blk, tg.B_blk, **kw)
    assert torch.equal(C.view(torch.int32), ref.view(torch.int32))
    e_or, e64 = _oracle_errors(C, tg.A_blk, tg.B_blk, terms=4 if kw.get("four_term") else 3)
    assert e_or <= 1e-6 and e64 <= 2e-6, (e_or, e64)
    assert tg.launches_per_step() == 5       # 2 max-abs + 2 splits + 1 GEMM piece, counted
    assert np.isfinite(C.cpu().numpy()).all()


@pytest.mark.parametrize("n", [1024, 2304])
def test_tile_gemm_replicated_one_rank(nccl_one_rank, n):
    """replicated inputs (no plane exchange): bitwise the one-GPU call with split-K off"""
    import paper_2011_11188_b200 as s3
    from paper_2011_11188_b200.dist import TileGemm

    h = s3.Handle(0)
    tg = TileGemm(h, n, 1, 0, seed=6, replicated=True)
    C = tg.run()
    torch.cuda.synchronize()
    h1 = s3.Handle(0)
    h1.set_split_k(False)
    ref = h1.sgemm_ex(tg.A, tg.B)
    assert torch.equal(C.view(torch.int32), ref.view(torch.int32))
    e_or, e64 = _oracle_errors(C, tg.A, tg.B)
    assert e_or <= 1e-6 and e64 <= 2e-6, (e_or, e64)
    assert tg.launches_per_step() >= 5


def test_gemm_pieces_equal_whole_bitwise():
    """the 2-D driver's pieces (row block x column block of the tile, written into strided C views
    from row slices of the K-major A planes and of stacked MN-major B blocks) == one whole call,
    BITWISE with split-K off (every element accumulates over K in the same order)"""
    import paper_2011_11188_b200 as s3
    from paper_2011_11188_b200.split3 import Planes
    from workloads import torch_matrix

    h = s3.Handle(0)
    h.set_split_k(False)
    m, n, K, pr, pc = 1024, 2048, 1536, 2, 4
    A = torch_matrix("uniform", m, K, seed=61)
    B = torch_matrix("loguni", K, n, seed=62)
    mx = torch.zeros(2, dtype=torch.float32, device="cuda")
    h.maxabs(A, mx[0:1])
    h.maxabs(B, mx[1:2])
    a_hi, a_lo, sA = h.split(A, mx[0:1])
    nbk, mb = n // pr, m // pc
    blocks = [h.split(B[:, q * nbk:(q + 1) * nbk].contiguous(), mx[1:2]) for q in range(pr)]
    b_hi = torch.cat([b[0] for b in blocks])       # pr stacked K x nbk MN-major blocks
    b_lo = torch.cat([b[1] for b in blocks])
    sB = blocks[0][2]
    whole = h.sgemm(A, B).clone()
    C = torch.full((m, n), 7.0, device="cuda")
    for r in range(pc):
        rs = slice(r * mb, (r + 1) * mb)
        for q in range(pr):
            cs = slice(q * nbk, (q + 1) * nbk)
            h.sgemm_ex(Planes(a_hi[rs], a_lo[rs], sA, None, mb, K, stored=True),
                       Planes(b_hi[q * K:(q + 1) * K], b_lo[q * K:(q + 1) * K], sB, None, K, nbk, stored=True),
                       out=C[rs, cs])
    torch.cuda.synchronize()
    assert torch.equal(C.view(torch.int32), whole.view(torch.int32))


def test_max_sms_cap_bitwise():
    """the GEMM on a reduced SM budget (the pieces that overlap a gather) gives the same bits"""
    import paper_2011_11188_b200 as s3
    from workloads import torch_matrix

    h = s3.Handle(0)
    h.set_split_k(False)
    A = torch_matrix("uniform", 2304, 1536, seed=71)
    B = torch_matrix("uniform", 1536, 2560, seed=72)
    ref = h.sgemm(A, B).clone()
    for sms in (132, 64, 2):
        h.set_max_sms(sms)
        C = h.sgemm(A, B)
        torch.cuda.synchronize()
        assert torch.equal(C.view(torch.int32), ref.view(torch.int32)), sms
    h.set_max_sms(0)
    with pytest.raises(s3.Split3Error):
        h.set_max_sms(3)


def test_nccl_plane_all_gather_dtype(nccl_one_rank):
    """the plane all-gather runs through NCCL with int16 plane tensors (moved as float16 bytes:
    NCCL has no int16) and keeps every bit pattern, NaN / Inf payloads included"""
    import torch.distributed as dist

    from paper_2011_11188_b200.dist import _all_gather_rows

    bits = torch.arange(-32768, 32768, dtype=torch.int32, device="cuda").to(torch.int16).view(256, 256)
    out = _all_gather_rows(bits, dist.group.WORLD, 1)
    torch.cuda.synchronize()
    assert out.dtype == torch.int16 and torch.equal(out, bits)


def test_gather_groups_with_cta_budget(nccl_one_rank):
    """the NCCL sub-groups the driver gathers over are created with config max_ctas (the SMs the
    overlapped GEMM pieces leave free): creation + an all-gather through one of them"""
    import torch.distributed as dist

    from paper_2011_11188_b200 import dist as d2

    rows, cols = d2.make_groups(1, gather_ctas=d2.GATHER_CTAS)
    assert d2.make_groups(1, gather_ctas=d2.GATHER_CTAS) == (rows, cols)      # cached
    bits = torch.arange(4096, dtype=torch.int32, device="cuda").to(torch.int16).view(64, 64)
    out = d2._all_gather_rows(bits, rows[0], 1)
    out2 = d2._all_gather_rows(bits, cols[0], 1)
    torch.cuda.synchronize()
    assert torch.equal(out, bits) and torch.equal(out2, bits)
    assert dist.get_backend(rows[0]) == "nccl"
