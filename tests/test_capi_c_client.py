"""The C ABI from a plain C program (tests/c/capi_smoke.c), compiled with gcc against
include/split3.h and linked to libsplit3.so — no Python or torch between caller and library."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c", "capi_smoke.c")


def _build(tmp_path):
    from paper_2011_11188_b200 import _build as b

    lib = b.build()
    exe = str(tmp_path / "capi_smoke")
    libdir = os.path.dirname(lib)
    subprocess.check_call(["gcc", "-O1", "-std=c11", SRC, "-I", os.path.join(ROOT, "include"),
                           "-I", "/usr/local/cuda/include", "-L", libdir, "-l:libsplit3.so",
                           f"-Wl,-rpath,{libdir}", "-L", "/usr/local/cuda/lib64", "-lcudart",
                           "-Wl,-rpath,/usr/local/cuda/lib64", "-o", exe])
    return exe


def test_c_client_cpu(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stderr
    assert "cpu ok" in out.stdout


@pytest.mark.gpu
def test_c_client_gpu(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "gpu ok" in out.stdout
