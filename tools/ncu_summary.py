"""Summarise ncu captures into profiles/ (run here, on the CPU box, after a gpurun).

  python tools/ncu_summary.py launches gpurun_out/launches_r01.csv profiles/launches_r01.md
  python tools/ncu_summary.py full gpurun_out/gemm3_full_r01.ncu-rep profiles/gemm3_full_r01.md
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__cluster_dim_x", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum",
]


def launches(csv_path, out_path):
    txt = open(csv_path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    per = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        ms = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(unit, 1.0) * v
        per[name][0] += 1
        per[name][1] += ms
    tot = sum(v[1] for v in per.values())
    lines = [f"# ncu launch list: {csv_path}", "",
             "Per-launch device times (cold-cache, serialised by ncu; compare SHARES, not absolutes).", "",
             "| kernel | launches | total ms | mean ms | share |", "|---|---|---|---|---|"]
    for k, (n, ms) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {ms:.3f} | {ms / n:.4f} | {ms / tot:.1%} |")
    open(out_path, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out_path):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full: {rep}", ""]
    data = {}
    for v in rows[2:]:
        name = v[hdr.index("Kernel Name")][:120]
        lines += [f"## `{name}`", "", "| metric | unit | value |", "|---|---|---|"]
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"| {k} | {units[i]} | {v[i]} |")
                data[k] = v[i]
        lines.append("")
    open(out_path, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    return data


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    (launches if mode == "launches" else full)(src, dst)
