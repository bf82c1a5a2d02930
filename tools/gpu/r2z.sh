timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
SOFG_BND_STAGE=100000 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_nan.py -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/step_profile.py --stats 2>&1 | tail -1
SOFG_BND_STAGE=0 timeout 300 python tools/step_profile.py --stats 2>&1 | tail -1 | grep -o "'hist_boundaries[^,]*"
SOFG_BND_STAGE=1024 timeout 300 python tools/step_profile.py --stats 2>&1 | tail -1 | grep -o "'hist_boundaries[^,]*"
