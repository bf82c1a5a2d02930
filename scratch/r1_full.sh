# official bench + reference arm + launch list + clocks
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clocks_r1.csv &
CPID=$!
timeout 1500 python bench.py 2>&1 | tail -1 > gpurun_out/bench_r1.json
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 2>&1 | tail -1 > gpurun_out/bench_r1_ref.json
kill $CPID
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/launches_r1.log 2>&1
cat gpurun_out/bench_r1.json gpurun_out/bench_r1_ref.json
