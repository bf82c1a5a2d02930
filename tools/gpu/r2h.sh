timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:hist_count --csv --log-file gpurun_out/r2h_hc.csv python tools/step_profile.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2h_hc.csv | tail -5
python - <<'P'
import csv
rows=list(csv.reader(open('gpurun_out/r2h_hc.csv')))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]; h=rows[hi]
ki,vi,mi,ii,gi=(h.index(x) for x in ('Kernel Name','Metric Value','Metric Name','ID','Grid Size'))
for r in rows[hi+1:]:
    if r[mi]=='gpu__time_duration.sum': print(r[ii], r[ki][:40], r[gi], r[vi])
P
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hist_count_lr -s 8 -c 1 -o gpurun_out/r2h_lr python tools/step_profile.py > /dev/null 2>&1
ls gpurun_out/r2h*
