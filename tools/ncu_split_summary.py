"""Summarise an ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum CSV
of the split-phase kernels (bench.py at N = 16384) into profiles/split_kernels.json, which bench.py
reports under roofline.split_kernels_ncu: per kernel the median launch time, DRAM bytes per launch,
the algorithmic bytes per launch (max-abs 4 B/el of A and B; split 4 B read + 4 B
written per element) and both as GB/s.  ncu launches are serialised and cold-cache."""
import csv
import json
import statistics
import sys
from collections import defaultdict

src, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 16384
out = sys.argv[3] if len(sys.argv) > 3 else "profiles/split_kernels.json"
rows = [r for r in csv.reader(open(src)) if len(r) > 14 and r[0] != "ID"]
per = defaultdict(lambda: defaultdict(list))
for r in rows:
    name = r[4].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    if "split_kernel" in r[4]:
        name = "split_kernel<plain>" if ("<1>" in r[4] or "<true>" in r[4]) else name
    per[name][r[12]].append(float(r[14].replace(",", "")))
alg = {"maxabs2_1d_kernel": 2 * n * n * 4, "split_kernel<plain>": n * n * 8}
res = {"source": src.split("/")[-1], "n": n, "note": "ncu: serialised, cold-cache launches; median per launch",
       "kernels": {}}
for k, m in per.items():
    if k not in alg:
        continue
    t = statistics.median(m["gpu__time_duration.sum"]) * 1e-9
    d = statistics.median(m["dram__bytes_read.sum"]) + statistics.median(m["dram__bytes_write.sum"])
    res["kernels"][k] = {"launches": len(m["gpu__time_duration.sum"]), "ms": t * 1e3, "dram_bytes": d,
                         "algorithmic_bytes": alg[k], "dram_gbs": d / t / 1e9, "algorithmic_gbs": alg[k] / t / 1e9}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
