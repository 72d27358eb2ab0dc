#!/usr/bin/env python
"""Benchmark: split-FP16 SGEMM effective TFLOPS (2MNK/t) on B200 (BASELINE.json metric).

One "step" = one whole split3_sgemm call (max-abs + split of A and B + tcgen05 GEMM with the
fused epilogue) on N x N FP32 inputs already resident in HBM.  Default workload:
configs[1], N = 16384, 3-term (BASELINE.json).  Inputs are 1 GiB per matrix (> 126 MB L2),
so no L2 flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--n 16384] [--terms 3|4|1]
  python bench.py --impl reference ...     # the CPU oracle (oracle/) as it stands

Multi-GPU (torchrun, one rank per GPU): 2-D C-tile partition (paper_2011_11188_b200.dist);
each rank owns one n x n tile of a (pr*n) x (pc*n) x n problem (weak scaling), inputs start
sharded and the FP16 plane panels are all-gathered over NCCL.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="split3", choices=["split3", "reference"])
    p.add_argument("--n", "--size", dest="n", type=int, default=16384)
    p.add_argument("--terms", type=int, default=3, choices=[1, 3, 4])
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--force-dist", action="store_true",
                   help="test only: run the 2-D tile path (NCCL) even with one rank")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                   help="rehearsal only: gloo runs every rank on cuda:0 (checks the N > 1 flow on one GPU; "
                        "not a measurement)")
    p.add_argument("--global-n", type=int, default=None,
                   help="strong scaling: one global_n^3 product cut into 2-D tiles (config D5); default "
                        "65536 when N > 1 (BASELINE configs[4]), off at N = 1 (configs[1], --n)")
    p.add_argument("--weak", action="store_true",
                   help="N > 1: weak scaling instead (each rank one --n sized tile of a (pr*n) x (pc*n) x n product)")
    p.add_argument("--inputs", default="sharded", choices=["sharded", "replicated"],
                   help="N > 1: inputs start sharded (plane all-gathers) or replicated on every rank")
    p.add_argument("--cpu-target-s", type=float, default=12.0)
    p.add_argument("--sustained-s", type=float, default=4.0,
                   help="extra back-to-back loop (s) reported as 'sustained' (0 = skip)")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return {"hbm": d["hbm_gbs"], "tc_burst": d["bf16_tflops"],
                "tc_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "src": "measured"}
    except Exception:
        return {"hbm": 6650.0, "tc_burst": 1590.0, "tc_sustained": 1400.0, "src": "fallback"}


# ----------------------------------------------------------------- clocks -----
class ClockSampler:
    """SM clock / power / throttle reasons sampled DURING the timed region (10 ms, NVML in-process;
    nvidia-smi -lms 100 as a fallback) — the profiling recipe's clocks line."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event-reason bits
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.nv = None
        self.samples = []
        self.stop_flag = False

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.pynvml = pynvml
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _poll(self):
        nv, p = self.nv, self.pynvml
        while not self.stop_flag:
            try:
                sm = p.nvmlDeviceGetClockInfo(nv, p.NVML_CLOCK_SM)
                mx = p.nvmlDeviceGetMaxClockInfo(nv, p.NVML_CLOCK_SM)
                pw = p.nvmlDeviceGetPowerUsage(nv) / 1000.0
                rs = p.nvmlDeviceGetCurrentClocksEventReasons(nv)
                self.samples.append((sm, mx, pw, rs))
            except Exception:
                pass
            time.sleep(0.01)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nv is not None:
            self.stop_flag = True
            self.t.join(timeout=2)
            if not self.samples:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
            reasons = sorted({name for s in self.samples for bit, name in self.REASONS.items() if s[3] & bit})
            return {"sm_mhz": float(np.median([s[0] for s in self.samples])),
                    "sm_max_mhz": float(max(s[1] for s in self.samples)),
                    "power_w_max": float(max(s[2] for s in self.samples)),
                    "samples": len(self.samples), "source": "nvml 10 ms", "reasons": reasons}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "power_w_max": max(pw),
                "samples": len(sm), "source": "nvidia-smi 100 ms", "reasons": sorted(reasons)}


def split_kernels_ncu():
    """Per-kernel GB/s and DRAM bytes of the split phase's kernels from the committed ncu capture
    (profiles/split_kernels.json; ncu times are cold-cache, serialised launches)."""
    path = os.path.join(ROOT, "profiles", "split_kernels.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


# ------------------------------------------------------------- cpu oracle -----
def cpu_oracle_sample(A_host: np.ndarray, B_host: np.ndarray, terms: int, target_s: float, C_gpu=None):
    """Time oracle.sgemm_sampled on R x R sampled outputs of the full-size problem.  With the
    GPU result C_gpu (a torch tensor), also report its error on exactly those samples: E_or vs
    the oracle's emulation, E64rel / E64 vs fp64 products of the sampled rows and columns."""
    import oracle

    N = A_host.shape[0]
    K = A_host.shape[1]
    Nc = B_host.shape[1]
    rng = np.random.Generator(np.random.PCG64(1234))

    last = {}

    def run(R):
        rows = np.sort(rng.choice(A_host.shape[0], R, replace=False))
        cols = np.sort(rng.choice(Nc, R, replace=False))
        t = time.perf_counter()
        Cs, _, _ = oracle.sgemm_sampled(A_host, B_host, rows, cols, terms=terms)
        dt = time.perf_counter() - t
        last.update(rows=rows, cols=cols, Cs=Cs)
        return dt

    r0 = min(32, N, Nc)
    t0 = run(r0)
    r1 = min(2 * r0, N, Nc)
    t1 = run(r1)
    per_r2 = max((t1 - t0) / max(r1 * r1 - r0 * r0, 1), 1e-9)
    fixed = max(t0 - per_r2 * r0 * r0, 0.0)
    R = int(np.sqrt(max(target_s - fixed, 0.0) / per_r2))
    R = int(max(r1, min(R, 1024, N, Nc)))
    dt = run(R)
    flops = 2.0 * R * R * K
    acc = None
    if C_gpu is not None:
        import torch

        rows, cols, Cs = last["rows"], last["cols"], last["Cs"]
        Cg = C_gpu[torch.from_numpy(rows).to(C_gpu.device)][:, torch.from_numpy(cols).to(C_gpu.device)]
        Cg = Cg.cpu().numpy().astype(np.float64)
        C64 = A_host[rows].astype(np.float64) @ B_host[:, cols].astype(np.float64)
        nA = float(np.linalg.norm(A_host.astype(np.float64)))
        nB = float(np.linalg.norm(B_host.astype(np.float64)))
        scale = (A_host.shape[0] * Nc) / (len(rows) * len(cols))
        acc = {"E_or": float(np.linalg.norm(Cg - Cs) / np.linalg.norm(Cs)),
               "E64rel": float(np.linalg.norm(Cg - C64) / np.linalg.norm(C64)),
               "E64": float(np.sqrt(scale) * np.linalg.norm(Cg - C64) / (nA * nB)),
               "samples": f"{len(rows)}x{len(cols)} outputs of the timed run's C",
               "tolerances": {"E_or": 1e-6, "E64": 2e-6}}
    try:
        phases = cpu_phases(A_host, B_host)
    except Exception as ex:   # reported, never silently replaced
        phases = {"error": repr(ex)}
    return {"value": flops / dt / 1e12, "unit": "TFLOPS", "cores": oracle.num_threads(),
            "cpu_model": cpu_model(), "phases": phases,
            "kind": "oracle", "seconds": dt, "accuracy": acc,
            "sample": f"{R}x{R} sampled outputs of the {A_host.shape[0]}x{Nc}x{K} product "
                      f"(fp64 oracle: full-matrix max-abs, split of the sampled rows/cols, "
                      f"{terms}-term Eq. A_2); value = 2*R*R*K / time"}


def cpu_model() -> str | None:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_phases(A_host: np.ndarray, B_host: np.ndarray) -> dict:
    """Per-phase rates of the oracle on the host cores: encode (max-abs + split,
    ns per element, on a 2048 x 2048 block of A), the FP64 reference GEMM and the split
    emulation (Eq. A_2 on the decoded planes, 3 terms) on a 512 x 512 x 2048 sub-problem."""
    import oracle

    out = {}
    n = min(2048, A_host.shape[0], A_host.shape[1])
    X = np.ascontiguousarray(A_host[:n, :n])
    t = time.perf_counter()
    m, _ = oracle.maxabs(X)
    hi, lo, s = oracle.split(X, s=oracle.scale_exp(m))
    out["encode_ns_per_el"] = (time.perf_counter() - t) / X.size * 1e9
    r, k = min(512, n), n
    a = np.ascontiguousarray(A_host[:r, :k])
    b = np.ascontiguousarray(B_host[:k, :r])
    t = time.perf_counter()
    oracle.gemm64(a, b)
    out["gemm64_gflops"] = 2.0 * r * r * k / (time.perf_counter() - t) / 1e9
    ah, al, sa = oracle.split(a)
    bh, bl, sb = oracle.split(b)
    t = time.perf_counter()
    oracle.split_gemm(ah, al, sa, bh, bl, sb, terms=3)
    out["split_emulation_gflops"] = 2.0 * r * r * k / (time.perf_counter() - t) / 1e9
    out["sub_problem"] = f"encode {n}x{n}; GEMMs {r}x{r}x{k}"
    return out


# ------------------------------------------------------------ reference arm ---
def run_reference(args, rank, world):
    if rank != 0:
        return
    import oracle
    from workloads import numpy_matrix

    per_step_target = max(2.0, min(20.0, 150.0 / max(args.steps + args.warmup, 1)))
    times = []
    if args.global_n:
        # config D5 (N = 65536): the full matrices (16 GiB each) would make every oracle step pay two
        # full-matrix max-abs passes (minutes); each step is instead the oracle's whole method on an
        # R x K row sample of A and a K x R column sample of B drawn from the same distribution
        # (scales from the sample), i.e. R x R outputs of a 65536-deep product
        n = args.global_n
        R = 64
        A = numpy_matrix("uniform", R, n, seed=0)
        B = numpy_matrix("uniform", n, R, seed=1)
        t = time.perf_counter()
        oracle.sgemm(A, B, terms=args.terms)
        t1 = time.perf_counter() - t
        R = int(max(16, min(2048, R * np.sqrt(per_step_target / max(t1, 1e-6)))))
        A = numpy_matrix("uniform", R, n, seed=0)
        B = numpy_matrix("uniform", n, R, seed=1)
        for i in range(args.warmup + args.steps):
            t = time.perf_counter()
            oracle.sgemm(A, B, terms=args.terms)
            dt = time.perf_counter() - t
            if i >= args.warmup:
                times.append(dt)
        sample = (f"{R}x{n} rows of A and {n}x{R} columns of B (uniform[-1,1], scales of the sample): "
                  f"{R}x{R} outputs of the {n}^3 product per step")
    else:
        n = args.n
        # the oracle's own inputs (same recipe as the GPU arm: uniform[-1,1], seeds 0/1)
        A = numpy_matrix("uniform", n, n, seed=0)
        B = numpy_matrix("uniform", n, n, seed=1)
        info = cpu_oracle_sample(A, B, args.terms, per_step_target)
        R = int(info["sample"].split("x")[0])
        rng = np.random.Generator(np.random.PCG64(99))
        for i in range(args.warmup + args.steps):
            rows = np.sort(rng.choice(n, R, replace=False))
            cols = np.sort(rng.choice(n, R, replace=False))
            t = time.perf_counter()
            oracle.sgemm_sampled(A, B, rows, cols, terms=args.terms)
            dt = time.perf_counter() - t
            if i >= args.warmup:
                times.append(dt)
        sample = info["sample"] + " per step"
    t_total = sum(times)
    value = 2.0 * R * R * n * len(times) / t_total / 1e12
    line = {
        "impl": "reference", "metric": "split-FP16 SGEMM effective TFLOPS (2MNK/t)",
        "value": value, "unit": "TFLOPS", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_total / max(len(times), 1),
        "higher_is_better": True, "scaling": "strong" if args.global_n else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "TFLOPS", "cores": oracle.num_threads(),
                         "kind": "oracle", "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": "TFLOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, world):
    name = {3: "3-term", 4: "4-term", 1: "1-term control"}[args.terms]
    pr, pc = grid_shape(world)
    g = getattr(args, "global_n", 0)
    if g:   # strong scaling (config D5)
        return {"workload": f"square N={g} FP32 uniform[-1,1], {name} split-FP16 GEMM, 2-D tiles {pr}x{pc}",
                "M": g, "N": g, "K": g, "terms": args.terms, "inputs": "fp32",
                "tensor_core": "fp16 x fp16 -> fp32 accumulate (tcgen05 kind::f16)",
                "parallelism": f"2d-tile {pr}x{pc}", "inputs_start": args.inputs,
                "l2": f"inputs {g * g * 4 / 2**30:.2f} GiB/matrix > 126 MB L2: no flush needed"}
    return {"workload": f"square N={args.n} FP32 uniform[-1,1], {name} split-FP16 GEMM"
                        + (f", 2-D tiles {pr}x{pc}" if world > 1 else ""),
            "M": args.n * pr, "N": args.n * pc, "K": args.n, "terms": args.terms,
            "inputs": "fp32", "tensor_core": "fp16 x fp16 -> fp32 accumulate (tcgen05 kind::f16)",
            "parallelism": f"2d-tile {pr}x{pc}" if world > 1 else "single",
            **({"inputs_start": args.inputs} if world > 1 or args.force_dist else {}),
            "l2": f"inputs {args.n * args.n * 4 / 2**30:.2f} GiB/matrix" + (
                " > 126 MB L2: no flush needed" if args.n * args.n * 4 > 126e6 else
                " < L2: inputs re-read from L2 between steps (small config)")}


def grid_shape(world):
    from paper_2011_11188_b200.dist import grid_for

    return grid_for(world)


# ------------------------------------------------------------------- main -----
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if args.global_n is None:
            args.global_n = 65536 if (world > 1 and not args.weak) else 0
        run_reference(args, rank, world)
        return
    if args.global_n is None:   # N > 1: config D5 (N = 65536, strong scaling) unless --weak
        args.global_n = 65536 if (world > 1 and not args.weak) else 0
    use_dist = world > 1 or args.force_dist or args.global_n > 0

    import torch

    from paper_2011_11188_b200 import split3 as s3
    from workloads import torch_matrix

    if args.dist_backend == "gloo":
        local = 0                           # rehearsal: all ranks share cuda:0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if use_dist:
        import torch.distributed as dist

        if args.dist_backend == "gloo":
            dist.init_process_group("gloo")
        elif "RANK" in os.environ:
            dist.init_process_group("nccl", device_id=dev)
        else:   # one process without a launcher (--force-dist / --global-n on one GPU)
            dist.init_process_group("nccl", store=dist.HashStore(), world_size=1, rank=0, device_id=dev)
    n = args.n
    h = s3.Handle(local)
    four, one = args.terms == 4, args.terms == 1

    if not use_dist:
        A = torch_matrix("uniform", n, n, seed=0, device=dev)
        B = torch_matrix("uniform", n, n, seed=1, device=dev)
        C = torch.empty((n, n), dtype=torch.float32, device=dev)

        def step():
            h.sgemm(A, B, out=C, four_term=four, one_term=one)
    else:
        from paper_2011_11188_b200.dist import TileGemm

        tg = TileGemm(h, n, world, rank, four_term=four, one_term=one, seed=0,
                      replicated=args.inputs == "replicated", global_n=args.global_n or None)

        def step():
            tg.run()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches_per_step = h.last_launch_count() if not use_dist else tg.launches_per_step()
    path = h.last_path() if not use_dist else 0     # SPLIT3_PATH_* bits of the step's call

    gpu_idx = local
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        try:
            gpu_idx = int(vis.split(",")[local])
        except ValueError:
            pass
    sampler = ClockSampler(gpu_idx)
    h.timing_enable(True)
    h.timing_read()
    sampler.start()
    time.sleep(0.05)
    if use_dist:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if use_dist:
        torch.distributed.barrier()
    clocks = sampler.stop()
    h.timing_enable(False)
    split_ms, gemm_ms, ncalls = h.timing_read()
    t_ms = e0.elapsed_time(e1)
    if use_dist:
        t = torch.tensor([t_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_ms = float(t.item())
    if use_dist:
        M_loc, N_loc, K = tg.M // tg.pr, tg.N // tg.pc, tg.K
    else:
        M_loc = N_loc = K = n
    flops_step = 2.0 * M_loc * N_loc * K * world
    value = flops_step * args.steps / (t_ms / 1e3) / 1e12
    pk = peaks()

    # roofline of the dominant kernel (the tcgen05 GEMM): algorithmic FP16 FLOPs per launch
    n_prod = {3: 3, 4: 4, 1: 1}[args.terms]
    # per STEP (the 2-D driver issues one GEMM launch per row block of the rank's tile)
    gemm_step_ms = gemm_ms / args.steps
    achieved = n_prod * 2.0 * M_loc * N_loc * K / (gemm_step_ms / 1e3) / 1e12 if ncalls else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "gemm3_traffic.json")
    if os.path.exists(prof) and not use_dist:
        try:
            with open(prof) as f:
                traffic = json.load(f)["bytes_per_launch"].get(str(n), {}).get(str(args.terms))
        except Exception:
            traffic = None
    # the peak for the timed region's length: the burst figure for a region shorter than the
    # 4-s back-to-back loop MEASURED_PEAKS' sustained figure comes from, else the sustained one
    long_region = t_ms >= 4000.0
    peak = pk["tc_sustained"] if long_region else pk["tc_burst"]
    roofline = {"bound": "tensor", "kernel": "gemm3_kernel", "achieved": achieved,
                "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": traffic,
                "peak_src": f"{pk['src']} bf16_tflops{'_sustained' if long_region else ''} "
                            f"(timed region {t_ms / 1e3:.2f} s; fp16 = bf16 nominal rate)",
                "frac_of_burst": (achieved / pk["tc_burst"]) if achieved else None,
                "frac_of_sustained": (achieved / pk["tc_sustained"]) if achieved else None,
                "frac_of_datasheet": (achieved / 2250.0) if achieved else None,
                "split_kernels_ncu": split_kernels_ncu(),
                "gemm_share_of_step": gemm_ms / max(t_ms, 1e-9) if ncalls else None,
                "gemm_launches_per_step": ncalls / args.steps,
                "split_ms_per_step": split_ms / args.steps if not use_dist else None,
                "split_hbm_gbs": (12.0 * 2 * n * n / (split_ms / args.steps / 1e3) / 1e9)
                if ncalls and split_ms > 0 and not use_dist else None,
                "path_bits": path}

    cpu = None
    if rank == 0 and not use_dist and not args.no_cpu:
        try:
            cpu = cpu_oracle_sample(A.cpu().numpy(), B.cpu().numpy(), args.terms, args.cpu_target_s, C_gpu=C)
        except Exception as ex:   # reported, never silently replaced
            cpu = {"value": None, "error": repr(ex)}

    # sustained: back to back for ~sustained_s seconds under the power cap (SURVEY §8d protocol);
    # the contract's `value` above is the K-step timed region
    sustained = None
    if args.sustained_s > 0:
        reps = max(args.steps, int(args.sustained_s * 1e3 / max(t_ms / args.steps, 1e-3)))
        s2 = ClockSampler(gpu_idx)
        s2.start()
        if use_dist:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        y0, y1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        y0.record(stream)
        for _ in range(reps):
            step()
        y1.record(stream)
        torch.cuda.synchronize()
        ck = s2.stop()
        ts = y0.elapsed_time(y1)
        if use_dist:
            tt = torch.tensor([ts], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            ts = float(tt.item())
        sustained = {"value": flops_step * reps / (ts / 1e3) / 1e12, "unit": "TFLOPS", "steps": reps,
                     "seconds": ts / 1e3, "sm_mhz": ck.get("sm_mhz"), "power_w_max": ck.get("power_w_max"),
                     "reasons": ck.get("reasons")}

    # e2e through the C-ABI with HOST buffers (H2D of A, B and D2H of C inside the timed region)
    e2e = None
    if not args.no_e2e and not use_dist:
        Ah = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
        Bh = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
        Ch = torch.empty((n, n), dtype=torch.float32, pin_memory=True)
        Ah.copy_(A)
        Bh.copy_(B)
        del C
        flags = (s3.FOUR_TERM if four else 0) | (s3.ONE_TERM if one else 0)
        h.sgemm_host_ptr(n, n, n, Ah.data_ptr(), Bh.data_ptr(), Ch.data_ptr(), flags)   # warm
        torch.cuda.synchronize()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(stream)
        for _ in range(args.e2e_steps):
            h.sgemm_host_ptr(n, n, n, Ah.data_ptr(), Bh.data_ptr(), Ch.data_ptr(), flags)
        x1.record(stream)
        torch.cuda.synchronize()
        te = x0.elapsed_time(x1) / args.e2e_steps
        e2e = {"value": 2.0 * n ** 3 / (te / 1e3) / 1e12, "unit": "TFLOPS",
               "h2d_bytes_per_step": 2 * n * n * 4, "d2h_bytes_per_step": n * n * 4,
               "ms_per_step": te, "api": "split3_sgemm_host (pinned host buffers)"}
    elif not args.no_e2e:
        # each rank: its A and B blocks from pinned host memory -> sgemm_2d -> its C tile to host
        Ah = tg.A_blk.cpu().pin_memory()
        Bh = tg.B_blk.cpu().pin_memory()
        Ch = torch.empty(tuple(tg.C.shape), dtype=torch.float32).pin_memory()

        cp = torch.cuda.Stream(device=dev)

        def copy_out(rows):   # each row block of the C tile goes out while the next one computes
            ev = torch.cuda.Event()
            ev.record(stream)
            cp.wait_event(ev)
            with torch.cuda.stream(cp):
                Ch[rows].copy_(tg.C[rows], non_blocking=True)

        def e2e_step():
            stream.wait_stream(cp)          # the previous step's copy-out has read C
            tg.A_blk.copy_(Ah, non_blocking=True)
            tg.B_blk.copy_(Bh, non_blocking=True)
            tg.run(on_block=copy_out)
            stream.wait_stream(cp)

        e2e_step()
        torch.cuda.synchronize()
        torch.distributed.barrier()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        x1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([x0.elapsed_time(x1) / args.e2e_steps], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        te = float(t.item())
        e2e = {"value": flops_step / (te / 1e3) / 1e12, "unit": "TFLOPS",
               "h2d_bytes_per_step": int(Ah.numel() + Bh.numel()) * 4 * world,
               "d2h_bytes_per_step": int(Ch.numel()) * 4 * world, "ms_per_step": te,
               "api": "paper_2011_11188_b200.dist.sgemm_2d (pinned host blocks, max over ranks)"}

    if rank == 0:
        line = {
            "metric": "split-FP16 SGEMM effective TFLOPS (2MNK/t)",
            "value": value, "unit": "TFLOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.global_n else "weak", "vs_baseline": None, "dtype": "f16",
            "data": "synthetic", "config": workload_config(args, world),
            **({"rehearsal": "gloo, every rank on cuda:0: checks the N > 1 flow, not a measurement"}
               if args.dist_backend == "gloo" else {}),
            "frac_of_peak_over_3": value / world / (pk["tc_burst"] / n_prod),
            "frac_of_datasheet_peak_over_3": value / world / (2250.0 / n_prod),
            "gpu_launches": launches_per_step * args.steps,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "sustained": sustained,
            "accuracy": (cpu or {}).get("accuracy"),
        }
        print(json.dumps(line), flush=True)
    if use_dist:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
