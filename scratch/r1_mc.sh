for i in 1 2; do timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1; done
for p in 1 0; do
SOFG_PRUNE=$p timeout 1500 python bench.py --samples 250000 --features 16384 --trees 32 --classes 4 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_ms']; print('c5 prune=$p', round(d['value'],2), {x: round(v['ms']) for x, v in k.items() if 'exact' in x})"
done
