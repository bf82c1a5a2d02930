for c in 03c3856 5d9ba86 ef9bb31; do
  echo "== $c"
  for i in 1 2 3 4; do (cd scratch/wt_$c && timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1); done
done
