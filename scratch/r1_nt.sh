for K in 2 3; do
SOFG_SWEEP_K=$K timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=r['kernel_ms']; print('K=$K', round(d['value'],2), round(k['row_sweep']['ms']))"
done
