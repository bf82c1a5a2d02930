K="k_sample_projection:12 k_hist_boundaries:6 k_part_flags:10"
for kv in $K; do
  name=${kv%%:*}; skip=${kv##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:${name}" -s $skip -c 1 -o gpurun_out/p5_${name} python scratch/prof_run.py 100 > /dev/null 2>&1
done
ls gpurun_out/p5_*
