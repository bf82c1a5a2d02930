set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r2a_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2a_bench.log 2>&1
tail -3 gpurun_out/r2a_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2a_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-profile > gpurun_out/r2a_ncu_bench.log 2>&1
cat gpurun_out/r2a_pytest.log
