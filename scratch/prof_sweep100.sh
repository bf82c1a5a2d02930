timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_row_sweep" -s 8 -c 1 -o gpurun_out/prof_sweep100 python scratch/prof_run.py 100 > gpurun_out/prof_sweep100.log 2>&1
tail -2 gpurun_out/prof_sweep100.log
