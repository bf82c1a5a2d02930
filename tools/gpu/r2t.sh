N="ncu --set full --clock-control none --import-source on -c 1"
timeout 600 $N -k regex:k_hist_count_lr --launch-skip 9 -o gpurun_out/r2t_hc python tools/step_profile.py > /dev/null 2>&1
timeout 600 $N -k regex:k_hist_count_lr --launch-skip 2 -o gpurun_out/r2t_hc2 python tools/step_profile.py > /dev/null 2>&1
timeout 600 $N -k regex:k_exact_prune --launch-skip 6 -o gpurun_out/r2t_pr python tools/step_profile.py > /dev/null 2>&1
timeout 600 $N -k regex:k_exact_reg --launch-skip 40 -o gpurun_out/r2t_er python tools/step_profile.py > /dev/null 2>&1
timeout 600 $N -k regex:k_hist_boundaries --launch-skip 9 -o gpurun_out/r2t_hb python tools/step_profile.py > /dev/null 2>&1
ls gpurun_out/
