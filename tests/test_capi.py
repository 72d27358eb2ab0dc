"""CPU-side checks of the boundary: the library loads and exports every declared symbol."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "split3.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(split3_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_api():
    names = _declared()
    for n in ("split3_sgemm_create", "split3_sgemm", "split3_sgemm_destroy", "split3_maxabs",
              "split3_split", "split3_gemm_planes"):
        assert n in names


def test_library_exports_every_declared_symbol():
    import ctypes

    from paper_2011_11188_b200 import _build, split3

    _build.build()
    lib = ctypes.CDLL(_build.LIB)
    for n in _declared():
        assert hasattr(lib, n), n
    assert sorted(split3.EXPORTS) == _declared()


def test_debug_build_exports_and_release_reports_not_implemented():
    """the checked build (-DSPLIT3_DEBUG=1) has the same ABI; the release build's
    debug entry points answer NOT_IMPLEMENTED without touching a GPU"""
    import ctypes

    from paper_2011_11188_b200 import _build, split3

    if not os.path.exists(_build.DEBUG_LIB):
        _build.build(force=True, out=_build.DEBUG_LIB, defines=["SPLIT3_DEBUG=1"])
    dbg = ctypes.CDLL(_build.DEBUG_LIB)
    for n in _declared():
        assert hasattr(dbg, n), n
    with pytest.raises(split3.Split3Error) as e:
        split3.debug_read()
    assert e.value.status == split3.ERR_NOT_IMPLEMENTED
    assert split3.load().split3_debug_fault(5) == split3.ERR_INVALID_VALUE


def test_status_strings_without_gpu():
    from paper_2011_11188_b200 import split3

    assert split3.status_string(0) == "SPLIT3_OK"
    assert split3.status_string(2) == "SPLIT3_ERR_NOT_FINITE"
    assert split3.status_string(99) == "SPLIT3_ERR_UNKNOWN"


def test_workspace_size_formula():
    from paper_2011_11188_b200 import split3

    lib = split3.load()
    # 256 B scalars + 2 planes of M x ldp(K) + 2 planes of N x ldp(K), each 256-B aligned
    M, N, K = 100, 60, 33
    ldp = 40
    al = lambda x: (x + 255) // 256 * 256
    assert lib.split3_sgemm_workspace_size(M, N, K, 0) == 256 + 2 * al(M * ldp * 2) + 2 * al(N * ldp * 2)


def test_create_without_gpu_fails_cleanly():
    import ctypes

    import torch

    from paper_2011_11188_b200 import split3

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    lib = split3.load()
    h = ctypes.c_void_p()
    assert lib.split3_sgemm_create(ctypes.byref(h), 0, None) in (split3.ERR_CUDA, split3.ERR_INVALID_VALUE)
    assert lib.split3_sgemm(None, 1, 1, 1, None, 1, None, 1, None, 1, 0) == split3.ERR_INVALID_VALUE


def test_no_oracle_import_in_product():
    """The product path never imports oracle/ (and vice versa)."""
    pkg = os.path.join(ROOT, "paper_2011_11188_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "oracle.c" not in txt and "liboracle" not in txt, f
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            assert not re.search(r"^\s*(import|from)\s+paper_2011_11188_b200", txt, re.M)
