"""Stall-reason breakdown per code region of an ncu report (source page, SASS view): regions are
delimited by marker instructions (LDTM / MUFU / STS / UTCHMMA ...) given as `name=regex` pairs in
program order; samples between one marker's first hit and the next region's go to that region.
    python profiles/stall_regions.py rep.ncu-rep"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
src = h.index("Source")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = [h.index(c) for c in cols]
tot = {c: 0 for c in cols}
by_op = {}
for r in rows[hi + 1:]:
    if len(r) <= max(idx):
        continue
    op = r[src].strip().split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
    o = o.split(".")[0]
    d = by_op.setdefault(o, {c: 0 for c in cols})
    for c, i in zip(cols, idx):
        v = int(r[i] or 0)
        d[c] += v
        tot[c] += v
T = sum(tot.values())
print("total samples", T)
print("by reason:", ", ".join(f"{c[6:]}={100 * v / T:.1f}%" for c, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
print("by opcode (top 20):")
for o, d in sorted(by_op.items(), key=lambda x: -sum(x[1].values()))[:20]:
    s = sum(d.values())
    top = sorted(d.items(), key=lambda x: -x[1])[:4]
    print(f"  {o:12s} {100 * s / T:5.1f}%  " + " ".join(f"{c[6:]}={100 * v / T:.1f}" for c, v in top if v))
