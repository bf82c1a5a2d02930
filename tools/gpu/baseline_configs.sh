# BASELINE configs 2, 4, 5 and the 8-rank host share (2 threads) on one B200
mkdir -p gpurun_out/r3a
timeout 900 python bench.py --steps 3 --warmup 3 --workers 2 --no-cpu-baseline > gpurun_out/r3a/c3_workers2.json 2>gpurun_out/r3a/c3_workers2.err; tail -c 400 gpurun_out/r3a/c3_workers2.json
for m in exact histogram dynamic; do
  timeout 900 python bench.py --samples 100000 --features 512 --trees 50 --mode $m --steps 5 --warmup 3 > gpurun_out/r3a/c2_$m.json 2>gpurun_out/r3a/c2_$m.err; tail -c 300 gpurun_out/r3a/c2_$m.json
done
timeout 1500 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/r3a/c4_800trees.json 2>gpurun_out/r3a/c4.err; tail -c 300 gpurun_out/r3a/c4_800trees.json
timeout 1500 python bench.py --samples 250000 --features 16384 --classes 4 --steps 3 --warmup 3 > gpurun_out/r3a/c5_default.json 2>gpurun_out/r3a/c5d.err; tail -c 300 gpurun_out/r3a/c5_default.json
timeout 1500 python bench.py --samples 250000 --features 16384 --classes 4 --density 0.001 --steps 3 --warmup 3 > gpurun_out/r3a/c5_dense.json 2>gpurun_out/r3a/c5x.err; tail -c 300 gpurun_out/r3a/c5_dense.json
