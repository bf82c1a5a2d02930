timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_r1c.csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --no-profile > gpurun_out/launches_r1c.log 2>&1
tail -1 gpurun_out/launches_r1c.log | cut -c1-100
