for f in 0.25 0.1 0.05 0.02; do
SOFG_SWEEP_FRAC=$f timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=r['kernel_ms']; print('frac=$f', round(d['value'],2), {x: round(k[x]['ms']) for x in ('row_sweep','project_gather','sweep_prep') if x in k}, k['row_sweep']['launches'])"
done
