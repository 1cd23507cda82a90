mkdir -p gpurun_out/ct
SPATTN_LIB=libprof.so timeout 300 ncu --nvtx --nvtx-include "spattn_move/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:copy_rows --csv --log-file gpurun_out/ct/msg_only.csv python tools/copy_kernels.py > /dev/null 2>&1
python tools/ncu_copy_launches.py gpurun_out/ct/msg_only.csv; python tools/ncu_copy_summary.py gpurun_out/ct/msg_only.csv 2>/dev/null | tail -2
SPATTN_NO_TMA_COPY=1 SPATTN_LIB=libprof.so timeout 300 ncu --nvtx --nvtx-include "spattn_move/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -k regex:copy_rows --csv --log-file gpurun_out/ct/msg_only_lsu.csv python tools/copy_kernels.py > /dev/null 2>&1
python tools/ncu_copy_launches.py gpurun_out/ct/msg_only_lsu.csv; python tools/ncu_copy_summary.py gpurun_out/ct/msg_only_lsu.csv 2>/dev/null | tail -2
