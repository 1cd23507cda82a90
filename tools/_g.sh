mkdir -p gpurun_out/s3e
timeout 900 python -m pytest tests/ -q -m gpu -x > gpurun_out/s3e/pytest_gpu.log 2>&1; tail -2 gpurun_out/s3e/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/s3e/bench.json 2> gpurun_out/s3e/bench.err; cat gpurun_out/s3e/bench.json
SPATTN_STEP_TRACE=1 timeout 300 python tools/step_trace.py 2>&1 | tail -8
