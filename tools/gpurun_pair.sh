SPATTN_STEP_TRACE=1 timeout 300 python tools/step_trace.py 2>&1 | tail -8
for r in 1 2; do timeout 600 python bench.py --no-secondary --no-cpu-baseline --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value', d['value'], 'e2e', d['e2e']['value'], d['e2e']['ms_per_step'], d['ms_per_step'])"; done
