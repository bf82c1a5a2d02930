# LR histogram counting for all node sizes (chunked): parity + per-kernel step times
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
SOFG_HIST_LR_CHUNK=1024 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py -m gpu -x -q 2>&1 | tail -2
for c in 8192 16384 32768; do echo "CHUNK $c"; SOFG_HIST_LR_CHUNK=$c timeout 300 python tools/step_profile.py --stats 2>&1 | tail -1 | grep -o "step.*ms\|'hist_count[^,]*"; done
echo "OLD (maxn 65504)"; SOFG_HIST_LR_MAXN=65504 timeout 300 python tools/step_profile.py --stats 2>&1 | tail -1 | grep -o "step.*ms\|'hist_count[^,]*"
