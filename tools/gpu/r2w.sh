timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/step_profile.py --stats 2>&1 | tail -1
SOFG_PART_CTA=1 timeout 300 python tools/step_profile.py --stats 2>&1 | tail -1 | grep -o "'partition[^,]*"
