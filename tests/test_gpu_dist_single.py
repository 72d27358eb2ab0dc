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
