for r in 1 2; do
for fam in tcgen05 tcgen05_pair; do echo -n "$fam: "; FAMILY=$fam timeout 120 python tools/shape_bench.py 32768 32 8 128 5 2>&1 | tail -1; done
echo -n "pair+release: "; SPATTN_LIB=fwdrel.so FAMILY=tcgen05_pair timeout 120 python tools/shape_bench.py 32768 32 8 128 5 2>&1 | tail -1
done
FAMILY=tcgen05_pair timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "pair" 2>&1 | tail -2
