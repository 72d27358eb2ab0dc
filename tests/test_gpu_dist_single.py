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


@pytest.mark.parametrize("n,kw", [(1024, {}), (2048, {}), (1536, {"four_term": True})])
def test_tile_gemm_one_rank_matches_single_call(nccl_one_rank, n, kw):
    import paper_2011_11188_b200 as s3
    from paper_2011_11188_b200.dist import TileGemm

    h = s3.Handle(0)
    tg = TileGemm(h, n, 1, 0, seed=5, **kw)
    C = tg.run()
    torch.cuda.synchronize()
    assert C.shape == (n, n)
    ref = h.sgemm(tg.A_blk, tg.B_blk, **kw).double()
    # same planes and scales; the row-block schedule may change the split-K plan (summation order)
    e = float((C.double() - ref).norm() / ref.norm())
    assert e < 1e-6, e
    C64 = tg.A_blk.double() @ tg.B_blk.double()
    e64 = float((C.double() - C64).norm() / C64.norm())
    assert e64 < 2e-6, e64
    assert tg.launches_per_step() >= 5       # counted: + the split-K tail reduction when planned
    assert np.isfinite(C.cpu().numpy()).all()


@pytest.mark.parametrize("n", [1024, 2048])
def test_tile_gemm_replicated_one_rank(nccl_one_rank, n):
    """replicated inputs (no plane exchange): same planes and scales as the single-GPU call"""
    import paper_2011_11188_b200 as s3
    from paper_2011_11188_b200.dist import TileGemm

    h = s3.Handle(0)
    tg = TileGemm(h, n, 1, 0, seed=6, replicated=True)
    C = tg.run()
    torch.cuda.synchronize()
    ref = h.sgemm_ex(tg.A, tg.B)
    assert torch.equal(C.view(torch.int32), ref.view(torch.int32)) or \
        float((C.double() - ref.double()).norm() / ref.double().norm()) < 1e-6
    assert tg.launches_per_step() >= 5


def test_gemm_planes_column_pieces_equal_whole():
    """the 2-D driver's column pieces (own rows x one B block of the panel, written into a column
    slice of the tile): gemm_planes on B^T plane row slices into strided C views == one whole call
    (to the oracle tolerance: the pieces' split-K plans, and so summation orders, differ)"""
    import paper_2011_11188_b200 as s3
    from workloads import torch_matrix

    h = s3.Handle(0)
    m, n, K, pr = 1024, 2048, 1536, 2
    A = torch_matrix("uniform", m, K, seed=61)
    B = torch_matrix("loguni", K, n, seed=62)
    mx = torch.zeros(2, dtype=torch.float32, device="cuda")
    h.maxabs(A, mx[0:1])
    h.maxabs(B, mx[1:2])
    a_hi, a_lo, sA = h.split(A, mx[0:1])
    b_hi, b_lo, sB = h.split(B, mx[1:2], transpose=True)          # B^T planes: n x K
    whole = h.gemm_planes(m, n, K, a_hi, a_lo, sA, b_hi, b_lo, sB).clone()
    C = torch.full((m, n), 7.0, device="cuda")
    nbk = n // pr
    for q in range(pr):
        cs = slice(q * nbk, (q + 1) * nbk)
        h.gemm_planes(m, nbk, K, a_hi, a_lo, sA, b_hi[cs], b_lo[cs], sB, out=C[:, cs])
    torch.cuda.synchronize()
    assert torch.isfinite(C).all()
    assert float((C.double() - whole.double()).norm() / whole.double().norm()) < 1e-6


def test_nccl_plane_all_gather_dtype(nccl_one_rank):
    """the plane all-gather runs through NCCL with int16 plane tensors (moved as float16 bytes:
    NCCL has no int16) and keeps every bit pattern, NaN / Inf payloads included"""
    import torch.distributed as dist

    from paper_2011_11188_b200.dist import _all_gather_rows

    bits = torch.arange(-32768, 32768, dtype=torch.int32, device="cuda").to(torch.int16).view(256, 256)
    out = _all_gather_rows(bits, dist.group.WORLD, 1)
    torch.cuda.synchronize()
    assert out.dtype == torch.int16 and torch.equal(out, bits)
