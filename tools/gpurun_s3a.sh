mkdir -p gpurun_out/s3a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s3a/smi.txt 2>&1
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/s3a/pytest_gpu.log 2>&1; tail -3 gpurun_out/s3a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3a/smoke.log 2>&1; tail -2 gpurun_out/s3a/smoke.log
timeout 600 python bench.py > gpurun_out/s3a/bench.json 2> gpurun_out/s3a/bench.err; cat gpurun_out/s3a/bench.json
