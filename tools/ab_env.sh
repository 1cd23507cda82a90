# A/B of environment switches: bash tools/ab_env.sh "" "SPATTN_FWD_STATIC=1" ...
for e in "$@"; do
  env $e python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('[$e]', round(b['ms_per_step'],2), 'fwd', round(b['kernels']['attn_fwd']['ms'],2), 'bwd', round(b['kernels']['attn_bwd']['ms'],2), b['clocks']['sm_mhz'])"
done
