timeout 900 python -m pytest tests/test_gpu_calibration.py tests/test_gpu_dropin.py -x -q 2>&1 | tail -30
timeout 300 python tools/calib_probe.py 2>&1 | tail -60
