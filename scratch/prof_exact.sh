K="k_exact_reg<.int.1,:12 k_exact_reg<.int.4,:8 k_exact_team<.int.1,:8 k_exact_team<.int.4,:6"
for kv in $K; do
  name=${kv%%:*}; skip=${kv##*:}
  tag=$(echo $name | tr -c 'a-z0-9_' '_' | tr -s '_')
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:${name}" -s $skip -c 1 \
     -o gpurun_out/prof_${tag} python scratch/prof_run.py 20 > gpurun_out/prof_${tag}.log 2>&1
  tail -2 gpurun_out/prof_${tag}.log
done
