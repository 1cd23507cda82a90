# Kernel TFLOP/s vs sequence length and per-rank shapes (tools/shape_bench.py): the c2 head layout
# at L = 4K..128K on one GPU, and the per-GPU shapes of Ulysses SP=2/4/8 at c2 and c4.
set -e
for L in 4096 8192 16384 32768 65536 131072; do python tools/shape_bench.py $L 32 8 128 3; done
python tools/shape_bench.py 32768 16 4 128 5    # c2, Ulysses SP=2 per-GPU heads
python tools/shape_bench.py 32768 8 2 128 5     # c2, SP=4
python tools/shape_bench.py 32768 4 1 128 5     # c2, SP=8
python tools/shape_bench.py 131072 4 1 128 2    # c4, Ulysses SP=8 per-GPU
python tools/shape_bench.py 65536 4 1 128 3     # c3 Dummy-Head SP=8: 4 real heads on the busiest rank (kv window 1)
python tools/shape_bench.py 4096 4 4 64 20      # c1, Ulysses SP=2 per-GPU (d=64)
