# compute-sanitizer memcheck over a cross-section of the GPU tests (every kernel family)
timeout 2400 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 10 python -m pytest -q -x -m gpu \
  "tests/test_gpu_parity.py::test_train_forest_small" "tests/test_gpu_parity.py::test_multiclass_forest" \
  "tests/test_gpu_parity.py::test_exact_large_nodes_segmented_sort" "tests/test_gpu_parity.py::test_find_node_split_trunk400" \
  "tests/test_gpu_parity.py::test_predict_matches_oracle" "tests/test_gpu_parity.py::test_train_tree_repeated_active_longer_than_n" \
  "tests/test_gpu_wide_classes.py::test_wide_class_forest" "tests/test_gpu_bins.py::test_large_bin_find_node_split" \
  "tests/test_gpu_parity.py::test_pinned_upload_in_flight" 2>&1 | grep -v "^    " | tail -25
echo "exit: $?"
