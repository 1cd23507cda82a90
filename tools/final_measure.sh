set -x
mkdir -p gpurun_out/s4
timeout 600 python -m pytest tests/ -q -m gpu -x > gpurun_out/s4/pytest_gpu.log 2>&1; tail -2 gpurun_out/s4/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/s4/bench.json 2> gpurun_out/s4/bench.err; cat gpurun_out/s4/bench.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s4/bench_ref.json 2>&1; tail -1 gpurun_out/s4/bench_ref.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s4/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1; wc -l gpurun_out/s4/launches.csv
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"attn_(fwd_tc|bwd_tc)" -s 2 -c 2 -o gpurun_out/s4/prof python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/s4/ncu_full.log 2>&1; tail -2 gpurun_out/s4/ncu_full.log
