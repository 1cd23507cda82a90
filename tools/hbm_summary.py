"""Summarise an ncu CSV of HBM-bound kernels: launches, time, DRAM bytes, achieved GB/s.
    python tools/hbm_summary.py gpurun_out/hbm.csv"""
import collections
import csv
import json
import os
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
ix = {n: h.index(n) for n in h}
per = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    key = (r[ix["ID"]], r[ix["Kernel Name"]])
    per[key][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (_, name), m in per.items():
    short = name.split("(")[0].replace("void ", "").replace("spattn::", "").replace("<unnamed>::", "")
    a = agg[short]
    a[0] += 1
    a[1] += m["gpu__time_duration.sum"]
    a[2] += m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")) else 6558.7
print("| kernel | launches | time (us) | DRAM bytes (MB) | achieved GB/s | of HBM peak |")
print("|---|---|---|---|---|---|")
for k, (n, t, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    gbs = b / t if t else 0.0  # bytes / ns = GB/s
    print(f"| `{k}` | {n} | {t / 1e3:.1f} | {b / 1e6:.1f} | {gbs:.0f} | {gbs / peak:.2f} |")
