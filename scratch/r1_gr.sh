for v in NONE SOFG_E2GR8 SOFG_E4GR4; do
env $v=1 timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=r['kernel_ms']; print('$v', round(d['value'],2), {x: round(v['ms']) for x, v in k.items() if x in ('exact_n<=64','exact_n<=128')})"
done
