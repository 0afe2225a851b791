C1="--batch 4096 --slots 26 --dim 8 --vocab 1000000 --hidden 64,32"
for r in 1 2; do for v in 8 4 2; do
KP_SEG_MINCH=$v timeout 300 python bench.py $C1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minch=$v', round(d['value']), {k:round(v['ms_per_step'],4) for k,v in d['stages'].items()})"
done; done
