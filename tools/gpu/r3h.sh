timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for i in 1 2; do timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'])"; done
