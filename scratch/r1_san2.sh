export SOFG_PRUNE=0
timeout 900 compute-sanitizer --tool initcheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -k segmented_sort > gpurun_out/san_init.log 2>&1
grep -m12 -A8 "^========= Uninit\|^========= Invalid\|ERROR SUMMARY" gpurun_out/san_init.log | head -60
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gpu_parity.py -q -k segmented_sort > gpurun_out/san_race.log 2>&1
grep -m12 -A8 "^========= .*[Hh]azard\|ERROR SUMMARY\|RACECHECK SUMMARY" gpurun_out/san_race.log | head -40
