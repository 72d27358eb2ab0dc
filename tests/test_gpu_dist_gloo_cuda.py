"""The 2-D tile driver with the REAL kernels at world size 2 and 4: the ranks are processes sharing
the one GPU of this box and exchanging through gloo (host-side collectives: no rank's kernel waits
on another's).  Covers CudaOps, the row/column-piece GEMMs on plane slices and strided C views,
and the tile ownership, against one single-process call on the assembled global matrices.
(The NCCL side-stream schedule is covered by tests/test_gpu_dist_single.py and the gloo/oracle
tests; this one checks the kernels' share of the partition.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, replicated, q, streams=None):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2011_11188_b200 as s3
        from paper_2011_11188_b200 import dist as d2

        torch.cuda.set_device(0)
        h = s3.Handle(0)
        tg = d2.TileGemm(h, n, world, rank, seed=7, replicated=replicated, streams=streams)
        tile = tg.run().cpu()
        torch.cuda.synchronize()
        r0, r1, c0, c1 = d2.c_tile(tg.M, tg.N, world, rank)
        if replicated:
            A, B = tg.A.cpu(), tg.B.cpu()
        else:   # assemble the global A and B from every rank's blocks
            As = [torch.empty_like(tg.A_blk.cpu()) for _ in range(world)]
            Bs = [torch.empty_like(tg.B_blk.cpu()) for _ in range(world)]
            dist.all_gather(As, tg.A_blk.cpu())
            dist.all_gather(Bs, tg.B_blk.cpu())
            A = torch.cat(As)
            B = torch.empty((tg.K, tg.N), dtype=torch.float32)
            for r in range(world):
                b0, b1 = d2.b_block_cols(tg.N, world, r)
                B[:, b0:b1] = Bs[r]
        ref = h.sgemm(A.cuda(), B.cuda())[r0:r1, c0:c1].cpu().double()
        e = float((tile.double() - ref).norm() / ref.norm())
        q.put((rank, e, bool(torch.isfinite(tile).all())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,replicated,streams", [(2, False, None), (4, False, None), (4, True, None),
                                                     (2, False, True), (4, False, True)])
def test_tile_driver_real_kernels(world, replicated, streams):
    """streams=True: the side-stream schedule the NCCL path uses (gathers on a communication
    stream, own-rows / own-columns pieces first, events and record_stream), here over gloo"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 1024, replicated, q, streams)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = {r: (e, fin) for r, e, fin in (q.get(timeout=10) for _ in range(world))}
    assert all(p.exitcode == 0 for p in procs)
    for r, (e, fin) in res.items():
        assert fin and e < 1e-6, (r, e)
