for v in 1; do
  SOFG_REG512=1 timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('reg512', round(d['value'],2), {k: round(v['ms']) for k, v in r['kernel_ms'].items() if 'exact' in k})"
done
