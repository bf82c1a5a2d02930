K="k_hist_boundaries:8 k_hist_count:8 k_exact_reg<.int.1,:14 k_exact_prune:8"
for kv in $K; do
  name=${kv%%:*}; skip=${kv##*:}
  tag=$(echo $name | tr -c 'a-z0-9_' '_' | tr -s '_')
  SOFG_GROUPS=1 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${name}" -s $skip -c 1 \
     -o gpurun_out/p6_${tag} python scratch/prof_run.py 100 > gpurun_out/p6_${tag}.log 2>&1
  tail -1 gpurun_out/p6_${tag}.log
done
ls -la gpurun_out/p6_*
