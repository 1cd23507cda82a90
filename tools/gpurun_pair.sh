timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_configs.py -q -m gpu -x 2>&1 | tail -1
for shape in "32768 8 8 64 5" "4096 4 4 64 50" "4096 8 8 64 50"; do timeout 120 python tools/shape_bench.py $shape 2>&1 | tail -1; done
