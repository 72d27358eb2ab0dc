"""GPU parity at the sizes of BASELINE.json's configs (oracle on sampled outputs).

  D2  square N = 4096 / 16384 (3-, 4-term)        -> test_gpu_parity.py::test_full_size_sampled_parity
  D3  MagmaDNN dense layers M x K x N               -> test_dense_layer_shapes
  D4  log-uniform 2^+-20, N = 8192                  -> test_wide_dynamic_range_n8192
  --  north_star "up to N = 32768"                  -> test_square_n32768
  D5  N = 65536 (single-GPU reference of the 2-D run) -> test_square_n65536
  D5  multi-GPU driver, CUDA ops + NCCL (1 rank)    -> test_dist_driver_nccl_one_rank
"""
import json
import os
import socket

import numpy as np
import pytest
import torch

from workloads import torch_matrix

pytestmark = pytest.mark.gpu

E_OR_TOL = 1e-6
E64_TOL = 2e-6
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


@pytest.fixture(scope="module")
def h():
    import paper_2011_11188_b200 as s3

    assert torch.cuda.is_available(), "GPU tests need a B200"
    return s3.Handle(0)


def sampled_check(orc, h, A, B, tag, R=48, terms=3, record=True):
    """C on the GPU vs the oracle on R x R sampled outputs; returns the metrics dict."""
    M, K = A.shape
    N = B.shape[1]
    C = h.sgemm(A, B, four_term=terms == 4)
    torch.cuda.synchronize()
    rng = np.random.Generator(np.random.PCG64(M * 7 + N))
    rows = np.sort(rng.choice(M, min(R, M), replace=False))
    cols = np.sort(rng.choice(N, min(R, N), replace=False))
    An = A.cpu().numpy()
    Bn = B.cpu().numpy()
    Cs, sA, sB = orc.sgemm_sampled(An, Bn, rows, cols, terms=terms)
    Cg = C[torch.from_numpy(rows).cuda()][:, torch.from_numpy(cols).cuda()].cpu().numpy().astype(np.float64)
    del C
    C64 = An[rows].astype(np.float64) @ Bn[:, cols].astype(np.float64)
    e_or = float(np.linalg.norm(Cg - Cs) / np.linalg.norm(Cs))
    e64rel = float(np.linalg.norm(Cg - C64) / np.linalg.norm(C64))
    scale = (M * N) / (len(rows) * len(cols))
    e64 = float(np.sqrt(scale) * np.linalg.norm(Cg - C64) /
                (np.linalg.norm(An.astype(np.float32)) * np.linalg.norm(Bn.astype(np.float32))))
    rec = {"config": tag, "M": M, "N": N, "K": K, "terms": terms, "E_or": e_or, "E64": e64,
           "E64rel": e64rel, "sA": sA, "sB": sB, "samples": [len(rows), len(cols)]}
    if record:
        os.makedirs(OUT, exist_ok=True)
        with open(os.path.join(OUT, f"parity_{tag}.json"), "w") as f:
            json.dump(rec, f)
    print(rec)
    return rec


DENSE = [(M, KN) for M in (256, 1024, 4096) for KN in (1024, 4096, 8192)]


@pytest.mark.parametrize("M,KN", DENSE)
def test_dense_layer_shapes(h, orc, M, KN):
    """D3: X (M x K) uniform activations x W (K x N) Glorot weights."""
    X = torch_matrix("uniform", M, KN, seed=M, device="cuda")
    W = torch_matrix("glorot", KN, KN, seed=KN, device="cuda")
    rec = sampled_check(orc, h, X, W, f"D3_M{M}_K{KN}")
    assert rec["E_or"] <= E_OR_TOL and rec["E64"] <= E64_TOL


def test_wide_dynamic_range_n8192(h, orc):
    """D4: x = +-2^u, u ~ U(-20, 20): planes bit-exact over the WHOLE matrices, no inf/NaN, C parity."""
    n = 8192
    A = torch_matrix("loguni", n, n, seed=41, device="cuda")
    B = torch_matrix("loguni", n, n, seed=42, device="cuda")
    for X, tr in ((A, False), (B, True)):
        d_max = torch.zeros(1, dtype=torch.float32, device="cuda")
        h.maxabs(X, d_max)
        hi, lo, sexp = h.split(X, d_max, transpose=tr)
        torch.cuda.synchronize()
        Xn = X.cpu().numpy()
        hi_o, lo_o, s_o = orc.split(Xn)
        assert int(sexp.item()) == s_o
        ghi = hi[:, :n].cpu().numpy().view(np.uint16)
        glo = lo[:, :n].cpu().numpy().view(np.uint16)
        if tr:
            ghi, glo = ghi.T, glo.T
        assert np.array_equal(ghi, hi_o) and np.array_equal(glo, lo_o)
        del hi, lo
    rec = sampled_check(orc, h, A, B, "D4_loguni_N8192")
    assert rec["E_or"] <= E_OR_TOL and rec["E64rel"] <= 1e-6


def test_square_n32768(h, orc):
    n = 32768
    A = torch_matrix("uniform", n, n, seed=51, device="cuda")
    B = torch_matrix("uniform", n, n, seed=52, device="cuda")
    rec = sampled_check(orc, h, A, B, "N32768", R=32)
    assert rec["E_or"] <= E_OR_TOL and rec["E64"] <= E64_TOL


def test_square_n65536(h, orc):
    """D5 size on one GPU (16 GiB per operand; planes + C fit the 180 GB HBM)."""
    import psutil

    n = 65536
    need_dev = (3 * n * n * 4 + 4 * n * n * 2) * 1.05
    free, _ = torch.cuda.mem_get_info()
    if free < need_dev or psutil.virtual_memory().available < 3 * n * n * 4:
        pytest.skip("not enough device or host memory for N=65536")
    A = torch_matrix("uniform", n, n, seed=61, device="cuda")
    B = torch_matrix("uniform", n, n, seed=62, device="cuda")
    rec = sampled_check(orc, h, A, B, "N65536", R=16)
    assert rec["E_or"] <= E_OR_TOL and rec["E64"] <= E64_TOL


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_dist_driver_nccl_one_rank(h):
    """The multi-GPU driver's CUDA ops + NCCL all-reduce on one rank == split3_sgemm, bitwise.

    (Bitwise equality across partitions holds when no split-K is involved: split-K, used only
    for problems with fewer C tiles than CTA pairs, sums K in a different fixed order.)"""
    import torch.distributed as dist

    from paper_2011_11188_b200 import dist as d2

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        M, N, K = 512, 256 * 37, 640     # 74 pair tiles: no tile is split along K
        A = torch_matrix("uniform", M, K, seed=7, device="cuda")
        B = torch_matrix("loguni", K, N, seed=8, device="cuda")
        tile = d2.sgemm_2d(A, B, M, N, d2.CudaOps(h))
        ref = h.sgemm(A, B)
        assert torch.equal(tile.view(torch.int32), ref.view(torch.int32))
    finally:
        dist.destroy_process_group()
