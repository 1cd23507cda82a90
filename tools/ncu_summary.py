"""Summarise a bench launch list (ncu --metrics gpu__time_duration.sum --csv) and a --set full
capture of the attention kernels into markdown (profiling helper).
    python tools/ncu_summary.py launches.csv prof.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

launches, rep = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(l for l in open(launches) if l.startswith('"'))]
hdr, data = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
tot = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].split("(")[0][:80]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    unit = r[ix["Metric Unit"]]
    v = v / 1000.0 if unit == "ns" else v * 1000.0 if unit == "ms" else v
    tot[name][0] += 1
    tot[name][1] += v
allus = sum(v[1] for v in tot.values())
print("| kernel | launches | total us | share |\n|---|---|---|---|")
for k, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1])[:8]:
    print(f"| `{k}` | {n} | {us:.1f} | {100 * us / allus:.1f}% |")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, units, body = rr[0], rr[1], rr[2:]
want = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem LSU wavefronts"),
        ("launch__registers_per_thread", "registers/thread"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block"), ("sm__cycles_elapsed.avg.per_second", "SM clock")]
for r in body:
    print(f"\n### `{r[h.index('Kernel Name')][:90]}`\n\n| metric | value |\n|---|---|")
    for m, label in want:
        if m in h:
            i = h.index(m)
            print(f"| {label} (`{m}`) | {r[i]} {units[i]} |")
