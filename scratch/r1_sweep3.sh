SOFG_PROJECT_MODE=1 timeout 600 python -m pytest tests -m gpu -x -q -k "forest or tree or golden" 2>&1 | tail -2
timeout 900 python bench.py --trees 100 --warmup 1 --steps 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/b100s9.json
python - <<'PY'
import json
d=json.load(open("gpurun_out/b100s9.json")); r=d["roofline"]
print(round(d["value"],2), "ms/step", round(d["ms_per_step"]), r["phase_ms"], r["kernel_ms"])
PY
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_row_sweep" -s 8 -c 1 -o gpurun_out/prof_k_row_sweep9 python scratch/prof_run.py 100 > /dev/null 2>&1
