# A/B sweep of the forward softmax's polynomial-exp2 share (profiling helper, run on the GPU box)
for v in ${@:-0x88 0x92 0xAA 0x52}; do
  touch paper_2505_22296_b200/csrc/attn_tc.cu
  make -C paper_2505_22296_b200 EXTRA=-DSPATTN_FWD_POLY_PAIRS=$v >/dev/null 2>&1
  timeout 200 python bench.py --steps 10 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['kernels']['attn_fwd'], d['clocks']['sm_mhz'])"
  timeout 100 python tools/fwd_trace.py 2>&1 | grep -E "per tile|sm : compute|exp"
done
touch paper_2505_22296_b200/csrc/attn_tc.cu
