timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py --trees 100 --warmup 1 --steps 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/b100x.json
python - <<'PY'
import json
d=json.load(open("gpurun_out/b100x.json")); r=d["roofline"]
print(round(d["value"],2), "ms/step", round(d["ms_per_step"]), r["phase_ms"], r["kernel_ms"])
PY
