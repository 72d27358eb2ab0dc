"""2-D C-tile partitioner over the GPUs of one box.

C = A*B with A (M x K) and B (K x N) sharded over P ranks arranged as a pr x pc grid;
rank r = i*pc + j owns the C tile rows [i*m, (i+1)*m) x cols [j*n, (j+1)*n), m = M/pr, n = N/pc.

Input ownership (inputs start sharded):
  * A is cut into P row blocks of M/P rows; block r is owned by rank r, so the row panel i of
    A (the rows tile (i, *) needs) is owned by the ROW GROUP {(i, 0..pc-1)}.
  * B is cut into P column blocks of N/P columns; block c = j*pr + i is owned by rank (i, j),
    so the column panel j is owned by the COLUMN GROUP {(0..pr-1, j)}.

One step (the only exchanges are 2 floats and the plane panels; there is no reduction over K):
  1. a1 local max-abs of the owned A block and B block;
  2. all_reduce(MAX) of [maxA, maxB] over all ranks: the global per-matrix scale (reading R1;
     max is exact and order-free, so every rank derives the same sA, sB as one GPU would);
  3. a2 local split of the owned blocks with the global scale (plain splits: A's block into
     K-major (M/P) x K planes, B's block into MN-major K x (N/P) planes);
  4. all_gather of the FP16 planes: A planes over the row group -> the m x K panel; B planes over
     the column group -> pr stacked K x (N/P) blocks (the column panel, block by block);
  5. a3+a4 the local tcgen05 GEMMs: one piece per (A row block, B column block) of the tile.
Every piece is a GEMM over whole tiles (CudaOps turns split-K off), and an element of C is
accumulated over K in the same order whatever piece or problem it belongs to, so the P-GPU C
equals the 1-GPU split3_sgemm C (split-K off) bitwise — tested with the real kernels at world 2
and 4 (tests/test_gpu_dist_gloo_cuda.py), besides the oracle tolerance.

Replicated inputs (every rank holds all of A and B; sgemm_2d_replicated): no plane exchange.
Rank (i, j) reads only its A row panel and B column panel — their max-abs, all_reduce(MAX) over
all ranks (every panel belongs to some rank, so this is the per-matrix max), a local split of the
two panels with the global scale and the GEMM on its tile: the same planes and C bits as one GPU.

The local ops are injectable (``ops``) so the exchange logic is tested on CPU with the gloo
backend (tests/test_dist_gloo.py); the default ops are the CUDA library's.
"""
from __future__ import annotations

import math
import os

import torch
import torch.distributed as dist


def grid_for(world: int) -> tuple[int, int]:
    """pr x pc process grid: pr = the largest divisor of world that is <= sqrt(world)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    pr = 1
    for d in range(1, int(math.isqrt(world)) + 1):
        if world % d == 0:
            pr = d
    return pr, world // pr


def coords(rank: int, world: int) -> tuple[int, int]:
    pr, pc = grid_for(world)
    return rank // pc, rank % pc


def a_block_rows(M: int, world: int, rank: int) -> tuple[int, int]:
    """Rows [r0, r1) of A owned by `rank`."""
    if M % world:
        raise ValueError("M must be divisible by the world size")
    b = M // world
    return rank * b, (rank + 1) * b


def b_block_cols(N: int, world: int, rank: int) -> tuple[int, int]:
    """Columns [c0, c1) of B owned by `rank` (block index j*pr + i)."""
    if N % world:
        raise ValueError("N must be divisible by the world size")
    pr, pc = grid_for(world)
    i, j = coords(rank, world)
    b = N // world
    c = j * pr + i
    return c * b, (c + 1) * b


def c_tile(M: int, N: int, world: int, rank: int) -> tuple[int, int, int, int]:
    """(r0, r1, c0, c1) of the C tile computed by `rank`."""
    pr, pc = grid_for(world)
    i, j = coords(rank, world)
    m, n = M // pr, N // pc
    return i * m, (i + 1) * m, j * n, (j + 1) * n


_GROUPS: dict = {}
# CTA budget of the NCCL plane all-gathers (config max_ctas); the GEMM pieces that overlap them run
# on the SMs left over
GATHER_CTAS = 8


def make_groups(world: int, gather_ctas: int | None = None):
    """Row groups and column groups (every rank must call this, in the same order).  Cached per
    (default process group, world, gather_ctas): a step loop reuses its communicators.
    gather_ctas: with NCCL, the CTA budget of the plane all-gathers (NCCL config max_ctas)."""
    key = (id(dist.group.WORLD), world, gather_ctas)
    g = _GROUPS.get(key)
    if g is not None:
        return g
    pr, pc = grid_for(world)
    kw = {}
    if gather_ctas and dist.get_backend() == "nccl":
        opts = dist.ProcessGroupNCCL.Options()
        opts.config.max_ctas = int(gather_ctas)
        opts.config.min_ctas = 1
        kw["pg_options"] = opts
    rows = [dist.new_group([i * pc + j for j in range(pc)], **kw) for i in range(pr)]
    cols = [dist.new_group([i * pc + j for i in range(pr)], **kw) for j in range(pc)]
    _GROUPS[key] = (rows, cols)
    return rows, cols


def _gather_rows(t: torch.Tensor, group, group_size: int) -> torch.Tensor:
    """Concatenate each group member's `t` along dim 0 (group order = member rank order)."""
    if group_size == 1:
        return t
    return _all_gather_rows(t, group, group_size)


def _all_gather_rows(t: torch.Tensor, group, group_size: int) -> torch.Tensor:
    out = torch.empty((group_size * t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    if dist.get_backend(group) == "nccl":
        # the planes are int16 tensors holding binary16 bits; NCCL has no 16-bit integer type, so
        # move them as float16 (an all-gather copies bytes, it never interprets them)
        src, dst = t.contiguous(), out
        if t.dtype == torch.int16:
            src, dst = src.view(torch.float16), out.view(torch.float16)
        dist.all_gather_into_tensor(dst, src, group=group)
    else:   # gloo (CPU tests): no 16-bit integer support, move the bytes
        src = t.contiguous().view(torch.uint8)
        parts = list(out.view(torch.uint8).chunk(group_size, 0))
        dist.all_gather(parts, src, group=group)
    return out


class CudaOps:
    """The product's local steps: the CUDA library through its binding.

    The handle runs whole tiles only (split3_set_split_k(h, 0)): every C element is accumulated
    over K in the same order as in a one-GPU split3_sgemm call with split-K off, so the 2-D
    partition reproduces that call's C bitwise (SURVEY §8e invariant).  gemm_sms_during_gather:
    the SM budget of the GEMM pieces that run while plane all-gathers are in flight (the rest is
    left to the gather kernels; the full-width GEMM holds ~225 KB of shared memory per SM)."""

    def __init__(self, h, gemm_sms_during_gather: int = 0):
        self.h = h
        self.launches = 0          # library kernels launched through these ops (NCCL's not counted)
        self.gather_sms = int(gemm_sms_during_gather)
        h.set_split_k(False)

    def begin(self, M, N, K, four_term):
        """The global problem's accumulator choice for every piece: the library folds 4-term calls
        of >= 8192^3 multiply-adds (split3_set_fold mode 1); a piece decides on its own shape, so
        the driver pins the whole problem's choice (mode 2 = fold, 0 = not) to keep the pieces'
        bits the one-GPU call's."""
        if four_term:
            self.h.set_fold(2 if M * N * K >= 2 ** 39 else 0)

    def maxabs_into(self, X, d_max1):
        self.h.maxabs(X, d_max1)
        self.launches += self.h.last_launch_count()

    def split(self, X, d_max1):
        """plain split of the stored block (no transpose): A rows -> K-major M x K planes,
        B columns -> MN-major K x N planes"""
        hi, lo, sexp = self.h.split(X, d_max1, transpose=False)
        self.launches += self.h.last_launch_count()
        return hi, lo, sexp

    def gemm(self, m, n, K, A1, A2, sA, B1, B2, sB, out, four_term, one_term, overlapped=False):
        """C piece (m x n) = A planes (m x K, K-major) times B planes (K x n, MN-major)"""
        from .split3 import Planes

        if overlapped and self.gather_sms:
            self.h.set_max_sms(self.gather_sms)
        try:
            res = self.h.sgemm_ex(Planes(A1, A2, sA, None, m, K, stored=True),
                                  Planes(B1, B2, sB, None, K, n, stored=True), out=out,
                                  four_term=four_term, one_term=one_term)
        finally:
            if overlapped and self.gather_sms:
                self.h.set_max_sms(0)
        self.launches += self.h.last_launch_count()
        return res


def sgemm_2d(A_blk: torch.Tensor, B_blk: torch.Tensor, M: int, N: int, ops, groups=None,
             out: torch.Tensor | None = None, four_term=False, one_term=False, overlap: bool = True,
             on_block=None, streams: bool | None = None):
    """One rank's share of C = A*B.  A_blk: its (M/P) x K block of A; B_blk: its K x (N/P)
    block of B.  Returns the rank's m x n C tile (see the module docstring).

    Planes: A's block -> K-major (M/P) x K planes, gathered over the row group into the m x K
    panel; B's block -> MN-major K x (N/P) planes (the plain split, no transpose), gathered over the
    column group into pr stacked K x (N/P) blocks.  The tile is computed as pieces (A row block) x
    (B column block), each a GEMM over whole tiles written into its slice of `out`.

    overlap: the rank's own A rows are multiplied first — by its own B block before the B panel
    has landed, then by the other blocks of the panel — while (NCCL) the panels are all-gathered
    on a communication stream; the other row blocks follow when the A panel lands.  Pieces that
    run under a gather use the ops' reduced SM budget (CudaOps.gather_sms) so the gather kernels
    find free SMs.

    on_block(rows): called after the GEMMs of each row block of the tile are enqueued (rows = a
    slice of `out`'s rows), e.g. to copy that part of C out while the next block computes.
    streams: gather on a side stream (default: with NCCL only; True also with gloo + CUDA
    tensors — tests of the stream schedule on one GPU).
    """
    world = dist.get_world_size()
    rank = dist.get_rank()
    pr, pc = grid_for(world)
    i, j = coords(rank, world)
    K = A_blk.shape[1]
    if hasattr(ops, "begin"):
        ops.begin(M, N, K, four_term)
    if groups is None:
        groups = make_groups(world)
    row_groups, col_groups = groups
    dev = A_blk.device
    m, n = M // pr, N // pc
    mb = M // world                      # rows of one A block
    nbk = N // world                     # columns of one B block
    # 1-2: global max-abs of A and B (exact, order-free)
    mx = torch.zeros(2, dtype=torch.float32, device=dev)
    ops.maxabs_into(A_blk, mx[0:1])
    ops.maxabs_into(B_blk, mx[1:2])
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    # 3: local split with the global scale (plain splits: A K-major, B MN-major)
    a_hi, a_lo, sA = ops.split(A_blk, mx[0:1])
    b_hi, b_lo, sB = ops.split(B_blk, mx[1:2])
    a_lo2 = a_hi if one_term else a_lo
    b_lo2 = b_hi if one_term else b_lo
    if out is None:
        out = torch.empty((m, n), dtype=torch.float32, device=dev)
    exchange = pr > 1 or pc > 1
    use_streams = overlap and exchange and dev.type == "cuda" and (
        dist.get_backend() == "nccl" if streams is None else bool(streams))

    def put(dst, res):
        if res is not None and res.data_ptr() != dst.data_ptr():
            dst.copy_(res)

    def gather_b():
        B1 = _gather_rows(b_hi, col_groups[j], pr)
        return B1, (B1 if one_term else _gather_rows(b_lo, col_groups[j], pr))

    def gather_a():
        A1 = _gather_rows(a_hi, row_groups[i], pc)
        return A1, (A1 if one_term else _gather_rows(a_lo, row_groups[i], pc))

    def bblock(P1, P2, q):               # B block q of the gathered panel: K x nbk planes
        return P1[q * K:(q + 1) * K], P2[q * K:(q + 1) * K]

    def row_block(rs, A1r, A2r, B1, B2, overlapped):
        """C[rs, :] = A rows x each B block of the column panel"""
        for q in range(pr):
            cs = slice(q * nbk, (q + 1) * nbk)
            b1, b2 = bblock(B1, B2, q)
            put(out[rs, cs], ops.gemm(A1r.shape[0], nbk, K, A1r, A2r, sA, b1, b2, sB, out[rs, cs],
                                      four_term, one_term, overlapped=overlapped))
        if on_block is not None:
            on_block(rs)

    if not overlap or not exchange:
        # 4 + 5: both panels, then the pieces
        B1, B2 = gather_b()
        A1, A2 = gather_a()
        for q in range(pc):
            rs = slice(q * mb, (q + 1) * mb)
            row_block(rs, A1[rs], A2[rs], B1, B2, False)
        return out
    # 4 under 5: the B panel and then the A panel are gathered on a communication stream (NCCL)
    # while the compute stream multiplies what is already local — the own A rows times the own
    # B block first (no exchange at all), then times the other B blocks of the column panel, then
    # the other row blocks of the A panel.  Every piece is a GEMM over whole tiles, so C is the
    # same as without the overlap.
    compute = torch.cuda.current_stream(dev) if use_streams else None
    comm = torch.cuda.Stream(device=dev) if use_streams else None
    if use_streams:
        comm.wait_stream(compute)
        with torch.cuda.stream(comm):
            B1, B2 = gather_b()
            ev_b = torch.cuda.Event()
            ev_b.record(comm)
            A1, A2 = gather_a()
    own = slice(j * mb, (j + 1) * mb)
    oc = slice(i * nbk, (i + 1) * nbk)           # this rank's own B block (position i in the panel)
    put(out[own, oc], ops.gemm(mb, nbk, K, a_hi, a_lo2, sA, b_hi, b_lo2, sB, out[own, oc], four_term, one_term,
                               overlapped=use_streams))
    if use_streams:
        compute.wait_event(ev_b)
    else:
        B1, B2 = gather_b()
    for q in range(pr):
        if q == i:
            continue
        cs = slice(q * nbk, (q + 1) * nbk)
        b1, b2 = bblock(B1, B2, q)
        put(out[own, cs], ops.gemm(mb, nbk, K, a_hi, a_lo2, sA, b1, b2, sB, out[own, cs], four_term, one_term,
                                   overlapped=use_streams))
    if on_block is not None:
        on_block(own)
    if use_streams:
        compute.wait_stream(comm)
    else:
        A1, A2 = gather_a()
    for q in range(pc):
        if q == j:
            continue
        rs = slice(q * mb, (q + 1) * mb)
        row_block(rs, A1[rs], A2[rs], B1, B2, False)
    if use_streams:
        for t in (A1, A2, B1, B2):
            t.record_stream(compute)
    return out


def sgemm_2d_replicated(A: torch.Tensor, B: torch.Tensor, ops, out: torch.Tensor | None = None,
                        four_term=False, one_term=False, on_block=None):
    """One rank's C tile of C = A*B with A (M x K) and B (K x N) replicated on every rank (see the
    module docstring): max-abs of the own panels, all_reduce(MAX), split, GEMM; no plane exchange."""
    world = dist.get_world_size()
    rank = dist.get_rank()
    M, K = A.shape
    N = B.shape[1]
    if hasattr(ops, "begin"):
        ops.begin(M, N, K, four_term)
    r0, r1, c0, c1 = c_tile(M, N, world, rank)
    Ap, Bp = A[r0:r1], B[:, c0:c1]            # row panel i (contiguous rows), column panel j (ld = N)
    mx = torch.zeros(2, dtype=torch.float32, device=A.device)
    ops.maxabs_into(Ap, mx[0:1])
    ops.maxabs_into(Bp, mx[1:2])
    dist.all_reduce(mx, op=dist.ReduceOp.MAX)
    a_hi, a_lo, sA = ops.split(Ap, mx[0:1])
    b_hi, b_lo, sB = ops.split(Bp, mx[1:2])
    m, n = r1 - r0, c1 - c0
    if out is None:
        out = torch.empty((m, n), dtype=torch.float32, device=A.device)
    res = ops.gemm(m, n, K, a_hi, a_hi if one_term else a_lo, sA, b_hi, b_hi if one_term else b_lo, sB, out,
                   four_term, one_term)
    if res is not out:
        out.copy_(res)
    if on_block is not None:
        on_block(slice(0, m))
    return out


class TileGemm:
    """bench.py's multi-GPU step: each rank owns an n x n C tile of a (pr*n) x (pc*n) x n
    problem (weak scaling; or a tile of a global_n^3 problem: strong scaling), inputs sharded as above, generated on the device from seeds
    (A block of rank r: seed*1000 + 2r, B block: seed*1000 + 2r + 1).  `ops`/`device` are
    injectable so the same workload runs on CPU / gloo in tests/test_dist_gloo.py."""

    def __init__(self, h, n: int, world: int, rank: int, four_term=False, one_term=False, seed=0,
                 ops=None, device=None, replicated: bool = False, global_n: int | None = None,
                 streams: bool | None = None, gather_ctas: int | None = None):
        from workloads import numpy_matrix, torch_matrix

        self.replicated = replicated
        self.streams = streams
        self.pr, self.pc = grid_for(world)
        # weak scaling: an n x n tile per rank of a (pr*n) x (pc*n) x n product; strong scaling
        # (global_n): the global_n^3 product cut into pr x pc tiles
        if global_n:
            self.M = self.N = self.K = global_n
        else:
            self.M, self.N, self.K = self.pr * n, self.pc * n, n
        self.h = h
        nccl = dist.get_backend() == "nccl"
        if gather_ctas is None:   # env SPLIT3_GATHER_CTAS overrides (0: NCCL's own CTA count, no SM cap)
            gather_ctas = int(os.environ.get("SPLIT3_GATHER_CTAS", GATHER_CTAS)) if (
                nccl and world > 1 and not replicated) else 0
        if ops is None:
            # pieces under a gather leave 2 SMs per gather CTA free: a CTA on one SM of a TPC
            # would otherwise break that TPC's GEMM CTA pair (cluster of 2)
            sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
            ops = CudaOps(h, gemm_sms_during_gather=max(sms - 2 * gather_ctas, 2) if gather_ctas else 0)
        self.ops = ops
        self.groups = make_groups(world, gather_ctas or None)
        r0, r1 = a_block_rows(self.M, world, rank)
        c0, c1 = b_block_cols(self.N, world, rank)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        if replicated:   # every rank: the whole A and B (the same seeds on every rank)
            if dev.type == "cuda":
                self.A = torch_matrix("uniform", self.M, self.K, seed=seed * 1000 + 1, device=dev)
                self.B = torch_matrix("uniform", self.K, self.N, seed=seed * 1000 + 2, device=dev)
                dtype = torch.float32
            else:
                self.A = torch.from_numpy(numpy_matrix("uniform", self.M, self.K, seed * 1000 + 1))
                self.B = torch.from_numpy(numpy_matrix("uniform", self.K, self.N, seed * 1000 + 2))
                dtype = torch.float64
            self.A_blk, self.B_blk = self.A, self.B
        elif dev.type == "cuda":
            self.A_blk = torch_matrix("uniform", r1 - r0, self.K, seed=seed * 1000 + 2 * rank, device=dev)
            self.B_blk = torch_matrix("uniform", self.K, c1 - c0, seed=seed * 1000 + 2 * rank + 1, device=dev)
            dtype = torch.float32
        else:
            self.A_blk = torch.from_numpy(numpy_matrix("uniform", r1 - r0, self.K, seed * 1000 + 2 * rank))
            self.B_blk = torch.from_numpy(numpy_matrix("uniform", self.K, c1 - c0, seed * 1000 + 2 * rank + 1))
            dtype = torch.float64          # the oracle's tiles
        self.C = torch.empty((self.M // self.pr, self.N // self.pc), dtype=dtype, device=dev)
        self.four, self.one = four_term, one_term

    def run(self, on_block=None):
        l0 = getattr(self.ops, "launches", None)
        if self.replicated:
            res = sgemm_2d_replicated(self.A, self.B, self.ops, out=self.C, four_term=self.four, one_term=self.one,
                                      on_block=on_block)
        else:
            res = sgemm_2d(self.A_blk, self.B_blk, self.M, self.N, self.ops, self.groups, out=self.C,
                           four_term=self.four, one_term=self.one, on_block=on_block, streams=self.streams)
        if l0 is not None:
            self._last_launches = self.ops.launches - l0
        return res

    def launches_per_step(self) -> int:
        """library kernels of the last run() (counted by the ops; NCCL's not counted), else the
        plan: 2 max-abs + 2 splits + one GEMM per (row block, column block) piece of the tile
        (one GEMM with replicated inputs)"""
        if getattr(self, "_last_launches", None) is not None:
            return self._last_launches
        if self.replicated:
            return 5
        return 4 + self.pc * self.pr
