"""Per-launch time / DRAM bytes / GB/s of an ncu --csv metrics log, grouped by size class
(profiling helper).  python tools/ncu_copy_launches.py x.csv [y.csv ...]"""
import collections
import csv
import sys

SC = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launches(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    ix = {k: i for i, k in enumerate(rows[0])}
    k = collections.OrderedDict()
    for r in rows[1:]:
        k.setdefault(r[ix["ID"]], {})[r[ix["Metric Name"]]] = (float(r[ix["Metric Value"]].replace(",", "")),
                                                               r[ix["Metric Unit"]])
    out = []
    for m in k.values():
        dur, u = m["gpu__time_duration.sum"]
        dur = dur / 1000 if u == "ns" else dur * 1000 if u == "ms" else dur
        by = sum(m[n][0] * SC.get(m[n][1], 1) for n in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        out.append((dur, by))
    return out


for p in sys.argv[1:]:
    cls = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for dur, by in launches(p):
        c = 1 << max(0, int(by / 1e6)).bit_length()
        cls[c][0] += 1
        cls[c][1] += dur
        cls[c][2] += by
    print(p)
    for c in sorted(cls):
        n, t, b = cls[c]
        print(f"  <= {c:4d} MB: {n:3d} launches, {t / n:6.1f} us avg, {b / n / 1e6:6.1f} MB avg, {b / t / 1e3:5.0f} GB/s")
