timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
SOFG_PROJECT_MODE=1 timeout 600 python -m pytest tests -m gpu -x -q -k "forest or tree or golden" 2>&1 | tail -2
timeout 900 python bench.py --trees 100 --warmup 1 --steps 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/b100g.json
SOFG_GROUPS=1 timeout 900 python bench.py --trees 100 --warmup 1 --steps 2 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/b100g1.json
python - <<'PY'
import json
for f in ("gpurun_out/b100g.json","gpurun_out/b100g1.json"):
    d=json.load(open(f)); r=d["roofline"]
    print(f, round(d["value"],2), "ms/step", round(d["ms_per_step"]), r["phase_ms"], r["kernel_ms"])
PY
