timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for v in 0 1; do
  if [ $v = 1 ]; then export SOFG_TEAM512=1; fi
  timeout 900 python bench.py --trees 100 --warmup 1 --steps 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('team512=$v', round(d['value'],2), {k: v['ms'] for k, v in d['roofline']['kernel_ms'].items() if 'exact' in k})"
done
