for wpb in 4 8 2; do
SOFG_HB_WARPS=$wpb timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['kernel_ms']; print('wpb=$wpb', round(d['value'],2), round(k['hist_boundaries']['ms']))"
done
