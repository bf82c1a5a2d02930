timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_bench.log 2>&1
tail -1 gpurun_out/r2d_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'e2e',d['e2e']['value'] if d.get('e2e') else None); r=d['roofline']; print('row_sweep avg ms',r['avg_launch_ms'],'frac',r['frac']); print({k:v['ms'] for k,v in r['kernel_ms'].items()})"
