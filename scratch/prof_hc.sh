SOFG_GROUPS=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_hist_count" -s 8 -c 1 -o gpurun_out/p9_hc python scratch/prof_run.py 100 > gpurun_out/p9_hc.log 2>&1
tail -2 gpurun_out/p9_hc.log
