timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
SOFG_GROUPS=1 timeout 900 python bench.py --trees 100 --warmup 1 --steps 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/b100h.json
python - <<'PY'
import json
d=json.load(open("gpurun_out/b100h.json")); r=d["roofline"]
print(round(d["value"],2), "ms/step", round(d["ms_per_step"]), r["kernel_ms"])
PY
SOFG_GROUPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k "regex:hist_count" -s 8 -c 1 -o gpurun_out/p3_hist python scratch/prof_run.py 100 > /dev/null 2>&1
