for m in exact histogram dynamic; do
  timeout 900 python bench.py --samples 100000 --features 512 --trees 50 --mode $m --warmup 3 --steps 3 --e2e-steps 1 --cpu-trees 16 2>&1 | tail -1 > gpurun_out/c2_$m.json
  python -c "
import json; d=json.load(open('gpurun_out/c2_$m.json'))
print('$m', 'gpu trees/s', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'cpu ref', d['cpu_baseline'], 'breakeven', d['config']['breakeven'])"
done
