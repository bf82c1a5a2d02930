# ncu --set full of the top kernels at a full level (launch 8 of each)
B="python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-profile"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_row_sweep_pipe -s 7 -c 1 -o gpurun_out/r2c_pipe $B > gpurun_out/r2c_pipe.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_hist_count -s 7 -c 1 -o gpurun_out/r2c_hc $B > gpurun_out/r2c_hc.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_hist_boundaries -s 7 -c 1 -o gpurun_out/r2c_hb $B > gpurun_out/r2c_hb.log 2>&1
ls -la gpurun_out
