for wu in 2 3 5; do
timeout 1200 python bench.py --steps 3 --warmup $wu --no-cpu-baseline --no-e2e --no-profile 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('warmup=$wu', round(d['value'],2))"
done
