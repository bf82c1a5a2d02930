timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for g in 2 1; do
  SOFG_GROUPS=$g timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e --no-profile 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('groups=$g', round(d['value'],2), round(d['ms_per_step']))"
done
