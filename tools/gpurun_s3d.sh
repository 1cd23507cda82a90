mkdir -p gpurun_out/s3d
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "one_member" > gpurun_out/s3d/pytest_new.log 2>&1; tail -1 gpurun_out/s3d/pytest_new.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s3d/launches.csv python bench.py --steps 2 --warmup 1 --no-secondary --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"attn_(fwd_tc|bwd_q128)" -s 2 -c 2 -o gpurun_out/s3d/prof python bench.py --config c2 --steps 1 --warmup 1 --no-secondary --no-e2e --no-cpu-baseline > gpurun_out/s3d/ncu_full.log 2>&1; echo "full rc=$?"; tail -2 gpurun_out/s3d/ncu_full.log
python tools/ncu_summary.py gpurun_out/s3d/launches.csv gpurun_out/s3d/prof.ncu-rep > gpurun_out/s3d/summary.md 2>&1; head -40 gpurun_out/s3d/summary.md
