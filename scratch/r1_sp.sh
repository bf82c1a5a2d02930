timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "dense or very_dense or sample_projection" 2>&1 | tail -1
timeout 1100 python bench.py --samples 250000 --features 16384 --trees 32 --classes 4 --density 0.001 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; k=r['kernel_ms']; print(round(d['value'],2), {x: round(v['ms']) for x, v in k.items() if x in ('sample_projection','row_sweep')})"
