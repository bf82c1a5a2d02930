# round-2 re-entry check: gpu suite, smoke, full bench
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python bench.py > gpurun_out/r2p_bench.log 2>&1
tail -1 gpurun_out/r2p_bench.log
