# A/B of an env knob: alternating bench runs in one box
KNOB=$1
for r in 1 2 3; do for v in 1 0; do
env $KNOB=$v timeout 300 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$KNOB=$v', round(d['value']), {k:round(v['ms_per_step'],3) for k,v in d['stages'].items() if k in ('mlp','push','dedup','pool')}, d['clocks']['sm_mhz'])"
done; done
