"""Multi-process checks of the 2-D tile driver (paper_2011_11188_b200.dist) on CPU / gloo.

The exchange logic (global max-abs all-reduce, row/column-group plane gathers, tile ownership)
runs for real over torch.distributed; the local steps are supplied by the oracle (CPU), so each
rank's C tile must equal the corresponding block of the oracle's single-process result exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2011_11188_b200 import dist as d2


def test_cuda_ops_pin_the_whole_problems_fold_choice():
    """CudaOps.begin: a 4-term problem of >= 8192^3 multiply-adds folds (the library's mode-1
    rule on the WHOLE problem), so every piece is pinned to fold (mode 2) — or to no fold (mode 0)
    for a smaller problem whose pieces would decide alike; 3-term calls leave the handle alone"""
    class FakeHandle:
        def __init__(self):
            self.calls = []

        def set_split_k(self, on):
            self.calls.append(("split_k", on))

        def set_fold(self, mode):
            self.calls.append(("fold", mode))

    h = FakeHandle()
    ops = d2.CudaOps(h)
    assert h.calls == [("split_k", False)]
    ops.begin(65536, 65536, 65536, True)
    ops.begin(8192, 8192, 8192, True)
    ops.begin(8192, 8192, 4096, True)
    ops.begin(65536, 65536, 65536, False)
    assert h.calls[1:] == [("fold", 2), ("fold", 2), ("fold", 0)]


def test_grid_and_ownership_math():
    assert d2.grid_for(1) == (1, 1)
    assert d2.grid_for(2) == (1, 2)
    assert d2.grid_for(4) == (2, 2)
    assert d2.grid_for(8) == (2, 4)
    assert d2.grid_for(6) == (2, 3)
    for P in (1, 2, 4, 6, 8):
        pr, pc = d2.grid_for(P)
        M, N = 24 * P, 12 * P
        tiles, arows, bcols = set(), [], []
        for r in range(P):
            i, j = d2.coords(r, P)
            tiles.add(d2.c_tile(M, N, P, r))
            arows.append(d2.a_block_rows(M, P, r))
            bcols.append(d2.b_block_cols(N, P, r))
            # A row panel of tile (i, j) is exactly the union of the row group's A blocks
            r0, r1, c0, c1 = d2.c_tile(M, N, P, r)
            grp = [i * pc + jj for jj in range(pc)]
            assert (d2.a_block_rows(M, P, grp[0])[0], d2.a_block_rows(M, P, grp[-1])[1]) == (r0, r1)
            cg = [ii * pc + j for ii in range(pr)]
            blocks = sorted(d2.b_block_cols(N, P, q) for q in cg)
            assert (blocks[0][0], blocks[-1][1]) == (c0, c1)
            assert all(blocks[t][1] == blocks[t + 1][0] for t in range(len(blocks) - 1))
        assert len(tiles) == P
        assert sorted(arows) == [(b * M // P, (b + 1) * M // P) for b in range(P)]
        assert sorted(bcols) == [(b * N // P, (b + 1) * N // P) for b in range(P)]


class OracleOps:
    """CPU stand-in for the CUDA steps (test infrastructure only)."""

    def __init__(self, orc):
        self.o = orc

    def maxabs_into(self, X, d_max1):
        m, bad = self.o.maxabs(np.ascontiguousarray(X.numpy()))
        assert bad < 0
        d_max1[0] = max(float(d_max1[0]), m)

    def split(self, X, d_max1):
        s = self.o.scale_exp(float(d_max1[0]))
        hi, lo, _ = self.o.split(np.ascontiguousarray(X.numpy()), s=s)
        return (torch.from_numpy(hi.view(np.int16)), torch.from_numpy(lo.view(np.int16)),
                torch.tensor([s], dtype=torch.int32))

    def gemm(self, m, n, K, A1, A2, sA, B1, B2, sB, out, four_term, one_term, overlapped=False):
        terms = 1 if one_term else (4 if four_term else 3)
        np16 = lambda t: np.ascontiguousarray(t.numpy()).view(np.uint16)
        C = self.o.split_gemm(np16(A1), np16(A2), int(sA[0]), np16(B1), np16(B2), int(sB[0]), terms)
        return torch.from_numpy(C)


def _worker(rank, world, port, M, N, K, terms, q, overlap=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle

        from workloads import numpy_matrix

        A = numpy_matrix("loguni", M, K, seed=1)
        B = numpy_matrix("uniform", K, N, seed=2)
        r0, r1 = d2.a_block_rows(M, world, rank)
        c0, c1 = d2.b_block_cols(N, world, rank)
        pr, pc = d2.grid_for(world)
        out = torch.empty((M // pr, N // pc), dtype=torch.float64)   # the oracle's fp64 tile
        tile = d2.sgemm_2d(torch.from_numpy(A[r0:r1].copy()), torch.from_numpy(B[:, c0:c1].copy()),
                           M, N, OracleOps(oracle), out=out, four_term=terms == 4, one_term=terms == 1,
                           overlap=overlap)
        full = oracle.sgemm(A, B, terms=terms)
        tr0, tr1, tc0, tc1 = d2.c_tile(M, N, world, rank)
        ok = np.array_equal(tile.numpy(), full[tr0:tr1, tc0:tc1])
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,terms,overlap", [(2, 3, True), (4, 3, True), (2, 4, True), (2, 3, False),
                                                (4, 1, False)])
def test_sgemm_2d_matches_single_process(orc, world, terms, overlap):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    M, N, K = 16 * world, 12 * world, 40
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, N, K, terms, q, overlap)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert res == {r: True for r in range(world)}


def _tile_worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle

        tg = d2.TileGemm(None, n, world, rank, ops=OracleOps(oracle), device=torch.device("cpu"), seed=3)
        tile = tg.run().numpy()
        # assemble the global A and B from every rank's blocks, then the oracle's full product
        As = [torch.empty_like(tg.A_blk) for _ in range(world)]
        Bs = [torch.empty_like(tg.B_blk) for _ in range(world)]
        dist.all_gather(As, tg.A_blk)
        dist.all_gather(Bs, tg.B_blk)
        A = torch.cat(As).numpy()                     # row blocks in rank order
        B = np.empty((tg.K, tg.N), np.float32)
        for r in range(world):
            c0, c1 = d2.b_block_cols(tg.N, world, r)
            B[:, c0:c1] = Bs[r].numpy()
        full = oracle.sgemm(A, B, terms=3)
        r0, r1, c0, c1 = d2.c_tile(tg.M, tg.N, world, rank)
        q.put((rank, bool(np.array_equal(tile, full[r0:r1, c0:c1])), tg.launches_per_step()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_bench_tilegemm_workload(orc, world):
    """bench.py's multi-rank workload (TileGemm: sharded seeded blocks, weak scaling) is the
    exact 2-D partition of one global product."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tile_worker, args=(r, world, port, 24, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    res = {r: (ok, nl) for r, ok, nl in (q.get(timeout=5) for _ in range(world))}
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok for ok, _ in res.values()), res


def _rep_worker(rank, world, port, M, N, K, terms, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle

        from workloads import numpy_matrix

        A = numpy_matrix("loguni", M, K, seed=5)
        A[: M // world] *= 2.0 ** 9            # rank 0's rows hold the max: the all-reduce matters
        B = numpy_matrix("uniform", K, N, seed=6)
        pr, pc = d2.grid_for(world)
        out = torch.empty((M // pr, N // pc), dtype=torch.float64)
        tile = d2.sgemm_2d_replicated(torch.from_numpy(A), torch.from_numpy(B), OracleOps(oracle), out=out,
                                      four_term=terms == 4, one_term=terms == 1)
        full = oracle.sgemm(A, B, terms=terms)
        tr0, tr1, tc0, tc1 = d2.c_tile(M, N, world, rank)
        q.put((rank, bool(np.array_equal(tile.numpy(), full[tr0:tr1, tc0:tc1]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,terms", [(2, 3), (4, 3), (4, 4)])
def test_sgemm_2d_replicated_matches_single_process(orc, world, terms):
    """replicated inputs: each rank splits only its panels with the all-reduced per-matrix scale;
    its tile equals the single-process oracle's block exactly (no plane exchange)"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    M, N, K = 16 * world, 12 * world, 40
    port = _free_port()
    procs = [ctx.Process(target=_rep_worker, args=(r, world, port, M, N, K, terms, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert res == {r: True for r in range(world)}
