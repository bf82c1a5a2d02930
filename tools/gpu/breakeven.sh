# re-tune the dynamic switch on the current kernels (device trees/s, config 3)
for b in ${BES:-512 640 768}; do
  timeout 600 python bench.py --steps 3 --warmup 2 --breakeven $b --no-cpu-baseline --no-e2e --no-profile 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($b, round(d['value'],2), round(d['ms_per_step'],1))"
done
