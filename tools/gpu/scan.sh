# parameter scan of the projection-producer choice (step time, stats on)
for pm in 0 8 16; do echo "PIPE_MIN $pm"; SOFG_SWEEP_PIPE_MIN=$pm timeout 300 python tools/step_profile.py --stats 2>&1 | tail -1 | grep -o "step [0-9.]* ms\|'row_sweep[^,]*\|'project_gather[^,]*\|'pair_build[^,]*"; done
for sf in 0.1 0.2; do echo "SWEEP_FRAC $sf"; SOFG_SWEEP_FRAC=$sf timeout 300 python tools/step_profile.py --stats 2>&1 | tail -1 | grep -o "step [0-9.]* ms\|'row_sweep[^,]*\|'project_gather[^,]*\|'pair_build[^,]*"; done
