# host phases per level + ncu full captures of hist_count_lr and row_sweep_pipe (level 8 launch)
SOFG_LEVEL_LOG=1 timeout 600 python tools/level_log.py > gpurun_out/r2q_level.log 2>&1
tail -3 gpurun_out/r2q_level.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_count_lr --launch-skip 8 -c 1 -o gpurun_out/r2q_hc python tools/step_profile.py > gpurun_out/r2q_ncu1.log 2>&1; tail -2 gpurun_out/r2q_ncu1.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_row_sweep_pipe --launch-skip 8 -c 1 -o gpurun_out/r2q_sw python tools/step_profile.py > gpurun_out/r2q_ncu2.log 2>&1; tail -2 gpurun_out/r2q_ncu2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_boundaries --launch-skip 12 -c 1 -o gpurun_out/r2q_hb python tools/step_profile.py > gpurun_out/r2q_ncu3.log 2>&1; tail -2 gpurun_out/r2q_ncu3.log
