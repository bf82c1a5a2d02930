timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_count_lr -s 8 -c 1 -o gpurun_out/r2j_lr8 python tools/step_profile.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_count_lr -s 0 -c 1 -o gpurun_out/r2j_lr0 python tools/step_profile.py > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:hist_count --csv --log-file gpurun_out/r2j_hc.csv python tools/step_profile.py > /dev/null 2>&1
SOFG_HIST_LR=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:hist_count --csv --log-file gpurun_out/r2j_hc_old.csv python tools/step_profile.py > /dev/null 2>&1
