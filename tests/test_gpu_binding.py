"""The Python binding's resource rules (include/split3.h: a handle serves one stream; the caller owns
the workspace): per-stream library handles and workspaces, and workspaces a CUDA graph captured
stay alive when a later call needs a larger one."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_graph_replay_after_workspace_growth():
    """capture a call, grow the workspace with a larger eager call on the capture stream, free
    memory churn, replay: the replay still writes into its own (kept) workspace -> bitwise eager"""
    import paper_2011_11188_b200 as s3
    from workloads import torch_matrix

    h = s3.Handle(0)
    A = torch_matrix("uniform", 512, 384, seed=1)
    B = torch_matrix("loguni", 384, 640, seed=2)
    ref = h.sgemm(A, B).clone()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    C = torch.empty_like(ref)
    with torch.cuda.stream(s):
        h.sgemm(A, B, out=C)                     # warm-up on the capture stream
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            h.sgemm(A, B, out=C)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):                   # a much larger call: the workspace grows
        A2 = torch_matrix("uniform", 4096, 2048, seed=3)
        B2 = torch_matrix("uniform", 2048, 4096, seed=4)
        big = h.sgemm(A2, B2)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):   # blocks freed on s are reused by allocations on s
        junk = [torch.full((1 << 22,), 3.0, device="cuda") for _ in range(8)]
    torch.cuda.synchronize()
    C.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(C.view(torch.int32), ref.view(torch.int32))
    assert torch.isfinite(big).all()
    assert all(bool((j == 3.0).all()) for j in junk)   # the replay wrote nothing into freed memory


def test_streams_get_separate_state():
    """two streams calling one Handle concurrently: each has its own library handle and workspace,
    so the calls cannot overwrite each other's planes or scalars"""
    import paper_2011_11188_b200 as s3
    from workloads import torch_matrix

    h = s3.Handle(0)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    A1 = torch_matrix("uniform", 2048, 2048, seed=5)
    B1 = torch_matrix("uniform", 2048, 2048, seed=6)
    A2 = torch_matrix("loguni", 2048, 2048, seed=7)
    B2 = torch_matrix("loguni", 2048, 2048, seed=8)
    r1 = h.sgemm(A1, B1).clone()
    r2 = h.sgemm(A2, B2).clone()
    torch.cuda.synchronize()
    outs = []
    for _ in range(5):
        with torch.cuda.stream(s1):
            c1 = h.sgemm(A1, B1)
        with torch.cuda.stream(s2):
            c2 = h.sgemm(A2, B2)
        outs.append((c1, c2))
    torch.cuda.synchronize()
    for c1, c2 in outs:
        assert torch.equal(c1.view(torch.int32), r1.view(torch.int32))
        assert torch.equal(c2.view(torch.int32), r2.view(torch.int32))
    # knobs reach every stream's handle
    h.set_split_k(False)
    with torch.cuda.stream(s1):
        a = h.sgemm(A1, B1)
    b = h.sgemm(A1, B1)
    torch.cuda.synchronize()
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
