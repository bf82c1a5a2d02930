for g in 1 2; do
SOFG_GROUPS=$g timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('groups=$g', round(d['value'],2), {k: round(v['ms']) for k, v in r['kernel_ms'].items()}, r['phase_ms'])"
done
