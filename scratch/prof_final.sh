SOFG_GROUPS=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_hist_count" -s 8 -c 1 -o gpurun_out/p12_hc python scratch/prof_run.py 100 > /dev/null 2>&1
SOFG_GROUPS=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_hist_boundaries" -s 8 -c 1 -o gpurun_out/p12_hb python scratch/prof_run.py 100 > /dev/null 2>&1
ls gpurun_out/p12*
