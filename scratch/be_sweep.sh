for be in 448 512 576 448 512 576; do
  timeout 900 python bench.py --trees 100 --warmup 3 --steps 3 --no-cpu-baseline --no-e2e --breakeven $be 2>&1 | tail -1 > gpurun_out/be_$be.json
  python -c "
import json; d=json.load(open('gpurun_out/be_$be.json')); r=d['roofline']
print($be, round(d['value'],2), round(d['ms_per_step']), {k: v['ms'] for k, v in r['kernel_ms'].items()})"
done
