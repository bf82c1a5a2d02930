set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep -E "Model name|Socket|Thread|Core"
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py --trees 20 --warmup 1 --steps 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/b20.json
timeout 900 python bench.py --trees 100 --warmup 1 --steps 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/b100.json
cat gpurun_out/b20.json gpurun_out/b100.json
