"""Aggregate launches / time / DRAM bytes / GB/s of an ncu --csv metrics log (profiling helper)."""
import csv, sys, collections
rows=[r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
h=rows[0]; ix={k:i for i,k in enumerate(h)}
k=collections.defaultdict(dict)
for r in rows[1:]:
    k[r[ix["ID"]]][r[ix["Metric Name"]]]=(float(r[ix["Metric Value"]].replace(",","")), r[ix["Metric Unit"]])
t=b=0.0
for kid,m in k.items():
    dur,u=m["gpu__time_duration.sum"]; dur = dur/1000 if u=="ns" else dur*1000 if u=="ms" else dur
    by=0
    for nm in ("dram__bytes_read.sum","dram__bytes_write.sum"):
        v,u2=m[nm]; by += v*{"byte":1,"Kbyte":1e3,"Mbyte":1e6,"Gbyte":1e9}.get(u2,1)
    t+=dur; b+=by
print(f"{sys.argv[1]}: {len(k)} launches, {t:.1f} us, {b/1e6:.1f} MB, {b/t/1e3:.0f} GB/s")
