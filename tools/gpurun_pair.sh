mkdir -p gpurun_out/ct
for lib in libspattn.so libct8.so; do
SPATTN_LIB=$lib timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:copy_rows --csv --log-file gpurun_out/ct/$lib.csv python tools/copy_kernels.py > /dev/null 2>&1
python tools/ncu_copy_launches.py gpurun_out/ct/$lib.csv
python tools/ncu_copy_summary.py gpurun_out/ct/$lib.csv 2>/dev/null | tail -3
done
for r in 1 2; do for lib in libspattn.so libct8.so; do echo -n "$lib msg step: "; SPATTN_LIB=$lib timeout 120 python tools/msg_step.py 8 2>&1 | tail -1; done; done
