timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/step_profile.py --stats 2>&1 | tail -1 | grep -o "step [0-9.]* ms"
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r3g_bench.log 2>&1
tail -1 gpurun_out/r3g_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value']); print(d['roofline']['phase_ms'])"
