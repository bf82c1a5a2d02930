timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
SOFG_PROJECT_MODE=1 timeout 900 python -m pytest tests -m gpu -x -q -k "forest or golden or dense or wide" 2>&1 | tail -1
timeout 900 python bench.py --trees 100 --warmup 1 --steps 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],2), r['achieved'], r['frac'], r['avg_launch_ms'], {k: v['ms'] for k, v in r['kernel_ms'].items()})"
