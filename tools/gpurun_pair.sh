mkdir -p gpurun_out/c1
for lib in libspattn.so lib16.so; do
SPATTN_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_ --csv --log-file gpurun_out/c1/l_$lib.csv python tools/shape_bench.py 4096 4 4 64 3 > /dev/null 2>&1
python - $lib <<'PY'
import csv,sys
rows=[r for r in csv.reader(l for l in open(f"gpurun_out/c1/l_{sys.argv[1]}.csv") if l.startswith('"'))]
ix={k:i for i,k in enumerate(rows[0])}
print(sys.argv[1], [(r[ix["Kernel Name"]][:30], r[ix["Metric Value"]]) for r in rows[1:]][:6])
PY
done
