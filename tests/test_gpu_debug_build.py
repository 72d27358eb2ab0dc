"""The checked debug build (libsplit3_debug.so, -DSPLIT3_DEBUG=1) — the substitute
for compute-sanitizer on this GPU pool: mbarrier watchdogs and pipeline invariants inside the GEMM.

  * over the shapes, term counts, operand layouts, split-K tails, the fused-B and fused-A paths, the folded accumulator and the 2-D
    driver's pieces of the parity suite, the debug build records no failure and its C is bitwise
    the release build's;
  * an injected fault (a TMA load that never happens) is caught by the watchdog: the record (in
    host-mapped memory) names the mbarrier wait (code 1), the kernel traps instead of hanging, and
    a new process runs normally on the same GPU afterwards.
Each library runs in its own subprocess (one libsplit3 per process)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKLOAD = r'''
import hashlib, json, os, sys
sys.path.insert(0, os.environ["ROOT"])
import torch
import paper_2011_11188_b200 as s3
s3.split3.LIB_PATH = os.environ["LIB"]
from workloads import torch_matrix
h = s3.Handle(0)
debug = os.environ.get("DEBUG") == "1"
if debug:
    s3.split3.debug_read(reset=True)
out = {}
def rec(name, C):
    torch.cuda.synchronize()
    out[name] = hashlib.sha256(C.contiguous().cpu().numpy().tobytes()).hexdigest()
for (M, N, K, kind) in [(64, 64, 64, "uniform"), (257, 129, 1000, "loguni"), (1024, 1024, 1024, "uniform"),
                        (2304, 1152, 777, "uniform"), (256, 8192, 2048, "glorot"), (4096, 4096, 4096, "uniform")]:
    A = torch_matrix(kind, M, K, seed=1); B = torch_matrix(kind, K, N, seed=2)
    for terms in (3, 4, 1):
        rec(f"{M}x{N}x{K}/{kind}/{terms}", h.sgemm(A, B, four_term=terms == 4, one_term=terms == 1))
    rec(f"{M}x{N}x{K}/{kind}/bf16x3", h.sgemm(A, B, bf16x3=True))
    rec(f"{M}x{N}x{K}/{kind}/tA", h.sgemm_ex(A.t().contiguous(), B, transA=True))
    rec(f"{M}x{N}x{K}/{kind}/tB", h.sgemm_ex(A, B.t().contiguous(), transB=True))
h.set_fused_split(2)
A = torch_matrix("uniform", 1024, 2048, seed=3); B = torch_matrix("uniform", 2048, 4096, seed=4)
rec("fusedB", h.sgemm(A, B))
h.set_fused_split(1)
h.set_fused_split_a(2)
rec("fusedA", h.sgemm(B.t().contiguous(), A.t().contiguous()))
rec("fusedA_splitk", h.sgemm(torch_matrix("uniform", 2048, 4096, seed=5), torch_matrix("uniform", 4096, 256, seed=6)))
h.set_fused_split_a(0)
h.set_fold(2)
for terms in (3, 4):
    rec(f"fold{terms}", h.sgemm(A, B, four_term=terms == 4))
    rec(f"fold{terms}_splitk", h.sgemm(torch_matrix("uniform", 300, 8192, seed=11), torch_matrix("uniform", 8192, 520, seed=12),
                                        four_term=terms == 4))
h.set_fold(1)
h.set_split_k(False)
rec("wholetiles", h.sgemm(A, B))
h.set_max_sms(132)
rec("capped", h.sgemm(A, B))
res = {"hashes": out}
if debug:
    res["record"] = s3.split3.debug_read(reset=True)
print("RESULT " + json.dumps(res))
'''

FAULT = r'''
import json, os, sys, time
sys.path.insert(0, os.environ["ROOT"])
import torch
import paper_2011_11188_b200 as s3
s3.split3.LIB_PATH = os.environ["LIB"]
from workloads import torch_matrix
h = s3.Handle(0)
A = torch_matrix("uniform", 2048, 2048, seed=1); B = torch_matrix("uniform", 2048, 2048, seed=2)
h.sgemm(A, B); torch.cuda.synchronize()
s3.split3.debug_read(reset=True)
s3.split3.debug_fault(1)
t = time.time()
err = None
try:
    h.sgemm(A, B)
    torch.cuda.synchronize()
except Exception as ex:          # the watchdog traps the kernel: a launch error, not a hang
    err = type(ex).__name__
dt = time.time() - t
rec = s3.split3.debug_read(reset=False)   # host-mapped: readable although the context is lost
print("RESULT " + json.dumps({"record": rec, "seconds": dt, "error": err}), flush=True)
os._exit(0)
'''

HEALTHY = r'''
import json, os, sys
sys.path.insert(0, os.environ["ROOT"])
import torch
import paper_2011_11188_b200 as s3
s3.split3.LIB_PATH = os.environ["LIB"]
from workloads import torch_matrix
h = s3.Handle(0)
A = torch_matrix("uniform", 2048, 2048, seed=1); B = torch_matrix("uniform", 2048, 2048, seed=2)
C = h.sgemm(A, B); torch.cuda.synchronize()
print("RESULT " + json.dumps({"finite": bool(torch.isfinite(C).all()), "record": s3.split3.debug_read()}))
'''


def _run(code, lib, debug, timeout=600):
    env = dict(os.environ, ROOT=ROOT, LIB=lib, DEBUG="1" if debug else "0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    return json.loads(line[len("RESULT "):])


def test_debug_build_clean_and_bitwise():
    from paper_2011_11188_b200 import _build

    rel = _run(WORKLOAD, _build.LIB, False)
    dbg = _run(WORKLOAD, _build.DEBUG_LIB, True)
    assert dbg["record"][0] == 0, dbg["record"]          # no watchdog trip, no invariant failure
    assert dbg["record"][4] == 0, dbg["record"]
    assert rel["hashes"] == dbg["hashes"]


def test_watchdog_catches_a_missing_tma_load():
    """one TMA load of A1 never issued: the full barrier's transaction count is never reached; the
    watchdog records code 1 (in host-mapped memory) and traps the kernel within seconds; a new
    process then runs normally on the same GPU"""
    from paper_2011_11188_b200 import _build

    res = _run(FAULT, _build.DEBUG_LIB, True, timeout=300)
    assert res["record"][0] == 1, res                    # mbarrier watchdog
    assert res["error"] is not None, res                 # the launch failed instead of hanging
    assert res["seconds"] < 60, res
    ok = _run(HEALTHY, _build.DEBUG_LIB, True, timeout=300)
    assert ok["finite"] and ok["record"][0] == 0, ok
