mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_golden.py -x -q -k c0_2000x16_exact > gpurun_out/san.log 2>&1
grep -m3 -A6 "^========= Invalid" gpurun_out/san.log; tail -3 gpurun_out/san.log
