# A/B of backward softmax-loop variants (SPATTN_BWD_SV, attn_bwd_tc.cu)
for sv in "$@"; do
  c=$(SPATTN_BWD_SV=$sv python tools/bwd_trace.py 2>&1 | grep -E "cycles per" | awk '{print $NF}')
  SPATTN_BWD_SV=$sv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('sv=$sv cycles/iter(CTA0)=$c', round(b['ms_per_step'],2), 'fwd', round(b['kernels']['attn_fwd']['ms'],2), 'bwd', round(b['kernels']['attn_bwd']['ms'],2), b['clocks']['sm_mhz'])"
done
