# full default bench (all keys) + gpu suite + smoke, as the driver runs them
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
tail -1 gpurun_out/final_bench.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'ms',d['ms_per_step'],'e2e',d['e2e']['value']); print('cpu', d['cpu_baseline']['value'], d['cpu_baseline']['bitexact_trees'], d['cpu_baseline']['holdout']['identical_labels']); print('frac', d['roofline']['frac'], 'split dram frac', d['roofline']['split_finder'].get('dram_frac'), 'clocks', d['clocks'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 | cut -c1-400
