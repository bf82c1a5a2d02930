for g in 0 1 2 3; do
  echo "== gather variant $g"
  SOFG_LIB=libsofg_g$g.so timeout 300 python bench.py --trees 20 --warmup 1 --steps 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']['phase_ms']; print(round(d['value'],2), 'hist', r['ms_hist_count'], 'exact', r['ms_exact'], 'waves', r['ms_waves_total'], 'rng', r['ms_hist_rng'])"
done
