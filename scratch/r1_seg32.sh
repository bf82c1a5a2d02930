SOFG_SEG32=1 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for e in 0 1; do
if [ $e = 1 ]; then export SOFG_SEG32=1; fi
timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('seg32=$e', round(d['value'],2), {k: round(v['ms']) for k, v in r['kernel_ms'].items() if 'exact' in k})"
done
