for c in 4096 16384 2048; do
SOFG_HIST_CHUNK=$c timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=r['kernel_ms']; print('chunk=$c', round(d['value'],2), round(k['hist_count']['ms']))"
done
