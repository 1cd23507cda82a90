# A/B of library builds (SPATTN_LIB): traced backward cycles/iteration of CTA 0 + bench kernel times
#   bash tools/ab_lib.sh libspattn.so v_x.so ...
for lib in "$@"; do
  c=$(SPATTN_LIB=$lib python tools/bwd_trace.py 2>&1 | grep -E "cycles per" | awk '{print $NF}')
  SPATTN_LIB=$lib python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('$lib bwd cycles/iter(CTA0)=$c', round(b['ms_per_step'],2), 'fwd', round(b['kernels']['attn_fwd']['ms'],2), 'bwd', round(b['kernels']['attn_bwd']['ms'],2), b['clocks']['sm_mhz'])"
done
