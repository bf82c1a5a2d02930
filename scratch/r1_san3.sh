export SOFG_PRUNE=0
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -k segmented_sort > gpurun_out/san_mem.log 2>&1
grep -m8 -A8 "^========= Invalid\|^========= Program hit\|ERROR SUMMARY" gpurun_out/san_mem.log | head -60
tail -3 gpurun_out/san_mem.log
