for p in 1 2 3; do
  SOFG_PRUNE_FROM=$p timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('from=$p', round(d['value'],2), {k: round(v['ms']) for k, v in r['kernel_ms'].items()})"
done
