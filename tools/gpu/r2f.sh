timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2f_step.csv python tools/step_profile.py > gpurun_out/r2f_step.log 2>&1
python tools/launch_summary.py gpurun_out/r2f_step.csv gpurun_out/r02_step_dram.json --exclude k_generate_trunk,k_transpose_rows --config '{"n": 1000000, "d": 4096, "trees": 100, "mode": "dynamic", "breakeven": 512, "classes": 2, "density": 0.0}' | tail -40
