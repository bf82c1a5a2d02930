mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 1500 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1c.json
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-profile > gpurun_out/launches_r1c.log 2>&1
tail -2 gpurun_out/launches_r1c.log
SOFG_GROUPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_row_sweep" -s 8 -c 1 -o gpurun_out/p10_sweep python scratch/prof_run.py 100 > /dev/null 2>&1
SOFG_GROUPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_exact_prune" -s 8 -c 1 -o gpurun_out/p10_prune python scratch/prof_run.py 100 > /dev/null 2>&1
cat gpurun_out/bench_r1c.json
