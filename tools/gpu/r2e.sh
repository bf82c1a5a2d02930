SOFG_LEVEL_LOG=1 timeout 600 python tools/level_log.py > gpurun_out/r2e_levels.log 2>&1
grep -v "^\s*\[wave\]" gpurun_out/r2e_levels.log | tail -45
