timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2k_bench.log 2>&1
tail -1 gpurun_out/r2k_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'e2e',d['e2e']['value'] if d.get('e2e') else None); r=d['roofline']; print({k:v['ms'] for k,v in r['kernel_ms'].items()})"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:hist_count --csv --log-file gpurun_out/r2k_hc.csv python tools/step_profile.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2k_hc.csv | tail -4
