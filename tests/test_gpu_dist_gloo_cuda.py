"""The 2-D tile driver with the REAL kernels at world size 2 and 4: the ranks
are processes sharing the one GPU of this box and exchanging through gloo (host-side collectives:
no rank's kernel waits on another's).  Covers CudaOps (max-abs + all_reduce(MAX), plain splits,
plane-panel gathers, per-(row block, column block) GEMM pieces on plane slices into strided C
views), the tile ownership and the side-stream schedule the NCCL path uses.

Each rank's tile is checked
  * against the ORACLE (oracle.sgemm_sampled on the assembled global A and B: the per-matrix
    scales of the whole matrices, Eq. A_2 in fp64 on the tile's rows and columns):
    E_or <= 1e-6 and E64 <= 2e-6 (north_star tolerances), and
  * BITWISE against one single-process split3_sgemm call on the assembled matrices with split-K
    off (SURVEY §8e invariant: same kernel, same per-element K order) — at sizes whose pieces and
    whole problem have ragged tiles and a partial last wave.
"""
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


def _worker(rank, world, port, n, replicated, q, streams=None, terms=3):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), OMP_NUM_THREADS=str(max(1, os.cpu_count() // world)))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import paper_2011_11188_b200 as s3
        from paper_2011_11188_b200 import dist as d2

        torch.cuda.set_device(0)
        h = s3.Handle(0)
        tg = d2.TileGemm(h, n, world, rank, seed=7, replicated=replicated, streams=streams,
                         four_term=terms == 4, one_term=terms == 1)
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
        # one GPU, one call, split-K off
        h1 = s3.Handle(0)
        h1.set_split_k(False)
        one = h1.sgemm(A.cuda(), B.cuda(), four_term=terms == 4, one_term=terms == 1)[r0:r1, c0:c1].cpu()
        bitwise = bool(torch.equal(tile.view(torch.int32), one.view(torch.int32)))
        # the oracle on this rank's tile (scales from the whole matrices)
        An, Bn = A.numpy(), B.numpy()
        Cs, _, _ = oracle.sgemm_sampled(An, Bn, np.arange(r0, r1), np.arange(c0, c1), terms=terms)
        C64 = oracle.gemm64(np.ascontiguousarray(An[r0:r1]), np.ascontiguousarray(Bn[:, c0:c1]))
        T = tile.double().numpy()
        e_or = float(np.linalg.norm(T - Cs) / np.linalg.norm(Cs))
        # E64 normalised by the norms of the rows / columns of A and B the tile reads
        e64 = float(np.linalg.norm(T - C64) / (np.linalg.norm(An[r0:r1].astype(np.float64)) *
                                              np.linalg.norm(Bn[:, c0:c1].astype(np.float64))))
        q.put((rank, bitwise, e_or, e64, bool(torch.isfinite(tile).all())))
    finally:
        dist.destroy_process_group()


def _run(world, n, replicated, streams, terms=3):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, replicated, q, streams, terms))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
    res = {r: v for r, *v in (q.get(timeout=10) for _ in range(world))}
    assert all(p.exitcode == 0 for p in procs)
    return res


@pytest.mark.parametrize("world,replicated,streams", [(2, False, None), (4, False, None), (2, True, None),
                                                     (4, True, None), (2, False, True), (4, False, True)])
def test_tile_driver_vs_oracle_and_bitwise(world, replicated, streams):
    """n = 1152: pieces of 576 or 1152 rows/columns (ragged 256-wide tiles); the one-GPU call of
    the whole problem (2304 x 2304 at world 4: 81 tiles > 74 CTA pairs) has a partial last wave.
    streams=True: the side-stream schedule the NCCL path uses (gathers on a communication
    stream, own-rows / own-columns pieces first, events and record_stream), here over gloo."""
    res = _run(world, 1152, replicated, streams)
    for r, (bitwise, e_or, e64, fin) in res.items():
        assert fin, r
        assert e_or <= 1e-6 and e64 <= 2e-6, (r, e_or, e64)
        assert bitwise, (r, e_or)


@pytest.mark.parametrize("terms", [4, 1])
def test_tile_driver_term_counts(terms):
    """4-term (256 x 128 tiles) and the 1-term control through the same partition"""
    res = _run(4, 640, False, True, terms)
    for r, (bitwise, e_or, e64, fin) in res.items():
        assert fin and bitwise, (r, e_or)
        if terms == 4:
            assert e_or <= 1e-6 and e64 <= 2e-6, (r, e_or, e64)
        else:   # a scaled plain FP16 GEMM: equals the oracle's 1-term emulation, not FP32
            assert e_or <= 1e-6, (r, e_or)
