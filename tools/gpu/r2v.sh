N="ncu --set full --clock-control none --import-source on -c 1"
timeout 600 $N -k regex:k_part_flags --launch-skip 2 -o gpurun_out/r2v_pf2 python tools/step_profile.py > /dev/null 2>&1
timeout 600 $N -k regex:k_part_scatter --launch-skip 2 -o gpurun_out/r2v_ps2 python tools/step_profile.py > /dev/null 2>&1
timeout 600 $N -k regex:k_part_flags --launch-skip 16 -o gpurun_out/r2v_pf16 python tools/step_profile.py > /dev/null 2>&1
timeout 600 $N -k regex:k_part_scatter --launch-skip 16 -o gpurun_out/r2v_ps16 python tools/step_profile.py > /dev/null 2>&1
timeout 600 $N -k regex:k_sample_projection --launch-skip 16 -o gpurun_out/r2v_sp16 python tools/step_profile.py > /dev/null 2>&1
ls gpurun_out | grep r2v
