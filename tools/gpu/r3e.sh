for v in 3 4 5; do echo "PRUNE_FROM $v"; SOFG_PRUNE_FROM=$v timeout 300 python tools/step_profile.py --stats 2>&1 | tail -1 | grep -o "step [0-9.]* ms\|'exact[^,]*"; done
