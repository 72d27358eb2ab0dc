"""Host-side cost of issuing one split3_sgemm call (no sync) vs its GPU time, small shapes."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_11188_b200 as s3  # noqa: E402
from workloads import torch_matrix  # noqa: E402

h = s3.Handle(0)
lib = s3.load()
for n in [int(x) for x in sys.argv[1:]] or [64, 256, 1024]:
    A = torch_matrix("uniform", n, n, seed=0)
    B = torch_matrix("uniform", n, n, seed=1)
    C = torch.empty((n, n), device="cuda")
    for _ in range(20):
        h.sgemm(A, B, out=C)
    torch.cuda.synchronize()
    reps = 2000
    # python binding path
    t0 = time.perf_counter()
    for _ in range(reps):
        h.sgemm(A, B, out=C)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    # raw C-ABI call (no torch-side marshalling): split3_sgemm on the same pointers
    t3 = time.perf_counter()
    for _ in range(reps):
        lib.split3_sgemm(h._h, n, n, n, A.data_ptr(), n, B.data_ptr(), n, C.data_ptr(), n, 0)
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(json.dumps({"n": n, "host_us_per_call_python": 1e6 * (t1 - t0) / reps,
                      "wall_us_per_call_python": 1e6 * (t2 - t0) / reps,
                      "host_us_per_call_cabi": 1e6 * (t4 - t3) / reps,
                      "wall_us_per_call_cabi": 1e6 * (t5 - t3) / reps}))
