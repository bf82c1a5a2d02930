# compute-sanitizer racecheck (shared-memory hazards) and synccheck over small forests, every kernel family
T='tests/test_gpu_parity.py::test_train_forest_small[dynamic-300] tests/test_gpu_parity.py::test_multiclass_forest tests/test_gpu_wide_classes.py::test_wide_class_forest[dynamic-400-9] tests/test_gpu_bins.py::test_large_bin_find_node_split[2048] tests/test_gpu_parity.py::test_exact_large_nodes_segmented_sort[exact-None] tests/test_gpu_headline.py::test_batch100_wide_sweep_variant[20000-64-2]'
for tool in racecheck synccheck; do
timeout 2400 compute-sanitizer --tool $tool --print-limit 200 python -m pytest -q -x -m gpu $T 2>&1 | grep -E "hazard|Error|ERROR|SUMMARY|passed|failed" | grep -o "SUMMARY.*\|[0-9]* passed.*\|[0-9]* failed.*\|in [a-z_]*\.cu[h]*:[0-9]*" | sort | uniq -c | sort -rn | head -12
done
