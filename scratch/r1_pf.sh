for p in 3 4; do
SOFG_PRUNE_FROM=$p timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=r['kernel_ms']; print('from=$p', round(d['value'],2), {x: round(v['ms']) for x, v in k.items() if 'exact' in x})"
done
