timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2y_bench.log 2>&1
tail -1 gpurun_out/r2y_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value'] if d.get('e2e') else None); print(d['roofline']['phase_ms'])"
SOFG_LEVEL_LOG=1 timeout 600 python tools/level_log.py > gpurun_out/r2y_level.log 2>&1; tail -1 gpurun_out/r2y_level.log
