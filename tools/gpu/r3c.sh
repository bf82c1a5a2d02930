timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest "tests/test_gpu_wide_classes.py::test_wide_class_forest[dynamic-400-9]" -m gpu -x -q 2>&1 | grep -v "^    " | head -60
