echo "== HEAD"; for i in 1 2 3 4; do timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1; done
echo "== HEAD copy"; for i in 1 2 3 4; do SOFG_COPY_EXPORT=1 timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1; done
echo "== ef9bb31"; for i in 1 2 3 4; do (cd scratch/wt_ef9bb31 && timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1); done
