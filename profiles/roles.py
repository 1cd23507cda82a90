"""Attribute warp-stall samples of a warp-specialized kernel to code regions (SASS address
ranges between marker instructions) — profiling helper.
    python profiles/roles.py gpurun_out/prof.ncu-rep"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
si, ti = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
d = [(int(r[si] or 0), r[ti].strip()) for r in rows[hi + 1:] if len(r) > si]
tot = sum(x for x, _ in d)
# segment at each taken-branch target is hard; instead report the top instructions with
# their +-3 neighbourhood so the role is recognisable
top = sorted(range(len(d)), key=lambda i: -d[i][0])[:12]
for i in top:
    ctx = " | ".join(d[j][1][:38] for j in range(max(0, i - 2), min(len(d), i + 2)))
    print(f"{100 * d[i][0] / tot:5.1f}% #{i}: {ctx}")
