timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
SOFG_PROJECT_MODE=1 timeout 600 python -m pytest tests -m gpu -x -q -k "forest or tree or golden" 2>&1 | tail -2
SOFG_PROJECT_MODE=0 timeout 600 python -m pytest tests -m gpu -x -q -k "forest or tree or golden" 2>&1 | tail -2
timeout 900 python bench.py --trees 100 --warmup 1 --steps 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 > gpurun_out/b100s2.json
python - <<'PY'
import json
for f in ("gpurun_out/b100s2.json",):
    try:
        d=json.load(open(f)); r=d["roofline"]
        print(f, round(d["value"],2), "ms/step", round(d["ms_per_step"]), r["phase_ms"], r["kernel_ms"])
    except Exception as e: print(f, "ERR", e, open(f).read()[-2000:])
PY
for kv in k_row_sweep:5 k_project_gather:2; do
  name=${kv%%:*}; skip=${kv##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:${name}" -s $skip -c 1 \
     -o gpurun_out/prof_${name} python scratch/prof_run.py 20 > gpurun_out/prof_${name}.log 2>&1
  tail -1 gpurun_out/prof_${name}.log
done
