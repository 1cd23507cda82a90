"""Summarise ncu captures (``--set full``) and launch lists into markdown for profiles/.

    python profiles/summarize.py gpurun_out/prof_x.ncu-rep [...] > profiles/rNN_x.md
    python profiles/summarize.py --launches gpurun_out/launches.csv
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "legacy HMMA subpipe % (mma.sync)"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (realtime, elapsed)"),
    ("sm__ops_path_tensor_op_utcmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", "tcgen05 bf16 ops % of peak"),
    ("sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", "hmma bf16 ops % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__inst_executed.sum", "instructions"),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(r, hdr, units) for r in rows[2:]]


def stalls(r, hdr):
    pre = "smsp__average_warp_latency_issue_stalled_"
    vals = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and h.endswith(("")) and "not_issued" not in h:
            try:
                vals.append((float(r[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    vals.sort(reverse=True)
    tot = sum(v for v, _ in vals) or 1
    return ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in vals[:6])


def main(argv):
    if argv and argv[0] == "--launches":
        lines = open(argv[1]).read().splitlines()
        start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
        rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
        agg = {}
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            name = r["Kernel Name"].split("(")[0][:70]
            t = float(r["Metric Value"].replace(",", ""))
            scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(r["Metric Unit"], 1)
            n, s = agg.get(name, (0, 0.0))
            agg[name] = (n + 1, s + t * scale)
        tot = sum(s for _, s in agg.values())
        print("| kernel | launches | total us | share |\n|---|---|---|---|")
        for name, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            print(f"| `{name}` | {n} | {s:.1f} | {100 * s / tot:.1f}% |")
        return
    for path in argv:
        for r, hdr, units in raw(path):
            name = r[hdr.index("Kernel Name")]
            print(f"### `{name[:90]}`  ({path.split('/')[-1]})\n")
            print("| metric | value |\n|---|---|")
            for key, label in KEYS:
                if key in hdr:
                    i = hdr.index(key)
                    print(f"| {label} (`{key}`) | {r[i]} {units[i]} |")
            print(f"| top stall reasons (pc sampling) | {stalls(r, hdr)} |\n")


if __name__ == "__main__":
    main(sys.argv[1:])
