timeout 900 python -m pytest tests/test_gpu_parity.py -k "exact_large or special or small" tests/test_gpu_wide_classes.py -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py --samples 100000 --features 512 --trees 50 --mode exact --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 exact value',d['value'],'e2e',d['e2e']['value'])"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
