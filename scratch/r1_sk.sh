for cfg in "256 1" "128 1" "256 2" "128 2"; do
set -- $cfg
SOFG_SWEEP_NT=$1 SOFG_SWEEP_K=$2 timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=r['kernel_ms']; print('NT=$1 K=$2', round(d['value'],2), round(k['row_sweep']['ms']))"
done
