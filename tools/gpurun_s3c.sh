mkdir -p gpurun_out/s3c
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/s3c/pytest_gpu.log 2>&1; tail -2 gpurun_out/s3c/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/s3c/bench.json 2> gpurun_out/s3c/bench.err; cat gpurun_out/s3c/bench.json
