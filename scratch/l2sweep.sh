for g in 128 64 32; do
  echo "== SOFG_L2_FETCH=$g"
  SOFG_L2_FETCH=$g timeout 300 python bench.py --trees 20 --warmup 1 --steps 1 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']['phase_ms']; print(round(d['value'],2), 'hist', r['ms_hist_count'], 'exact', r['ms_exact'], 'waves', r['ms_waves_total'])"
done
python -c "
import ctypes; c=ctypes.CDLL('libcudart.so') if False else None
"
