# round-2 final profiles: one-step DRAM launch list (bench roofline traffic), ncu full captures of the top kernels
mkdir -p gpurun_out/r3f
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r3f/step_dram.csv python tools/step_profile.py > gpurun_out/r3f/step.log 2>&1
python tools/launch_summary.py gpurun_out/r3f/step_dram.csv gpurun_out/r3f/r02b_step_dram.json --config '{"n": 1000000, "d": 4096, "trees": 100, "mode": "dynamic", "breakeven": 512, "classes": 2, "density": 0.0}' --exclude k_generate_trunk,k_transpose > gpurun_out/r3f/r02b_step_dram.txt 2>&1; tail -5 gpurun_out/r3f/r02b_step_dram.txt
N="ncu --set full --clock-control none --import-source on -c 1"
timeout 600 $N -k regex:k_row_sweep_pipe --launch-skip 8 -o gpurun_out/r3f/ncu_row_sweep python tools/step_profile.py > /dev/null 2>&1
timeout 600 $N -k regex:k_hist_count_lr --launch-skip 8 -o gpurun_out/r3f/ncu_hist_count_lr python tools/step_profile.py > /dev/null 2>&1
timeout 600 $N -k regex:k_hist_boundaries --launch-skip 9 -o gpurun_out/r3f/ncu_hist_boundaries python tools/step_profile.py > /dev/null 2>&1
timeout 600 $N -k regex:k_exact_prune --launch-skip 12 -o gpurun_out/r3f/ncu_exact_prune python tools/step_profile.py > /dev/null 2>&1
timeout 600 $N -k regex:k_part_flags_w --launch-skip 16 -o gpurun_out/r3f/ncu_part_flags python tools/step_profile.py > /dev/null 2>&1
ls gpurun_out/r3f
