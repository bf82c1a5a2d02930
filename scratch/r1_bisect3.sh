for i in 1 2 3 4 5; do timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | grep -E "^FAILED|passed|failed" | cut -c1-150; done
echo "== 41397bb"
for i in 1 2 3; do (cd scratch/wt_41397bb && timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -rf 2>&1 | grep -E "^FAILED|passed|failed" | cut -c1-150); done
