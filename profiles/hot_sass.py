"""Top SASS instructions by warp-stall samples from an ncu report (source page, sass view).
    python profiles/hot_sass.py gpurun_out/prof.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
si, ti = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source")
data = [(int(r[si] or 0), r[ti].strip(), i) for i, r in enumerate(rows[hi + 1:]) if len(r) > si]
tot = sum(d[0] for d in data) or 1
for s, src, i in sorted(data, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}%  #{i:5d}  {src}")
