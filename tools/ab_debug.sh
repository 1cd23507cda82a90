# A/B of profiling switches (SPATTN_DEBUG bits, see attn_bwd_tc.cu; needs a build with EXTRA=-DSPATTN_PROFILING): bash tools/ab_debug.sh 0 1 16 32 ...
for dbg in "$@"; do
SPATTN_DEBUG=$dbg python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('dbg=$dbg', round(b['ms_per_step'],2), 'fwd', round(b['kernels']['attn_fwd']['ms'],2), 'bwd', round(b['kernels']['attn_bwd']['ms'],2), b['clocks']['sm_mhz'])"
done
