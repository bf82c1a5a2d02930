import csv,sys,subprocess
rep=sys.argv[1]
out=subprocess.run(['ncu','-i',rep,'--page','raw','--csv'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
h=rows[0]; u=rows[1]; v=rows[2]
want=['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','sm__warps_active.avg.pct_of_peak_sustained_active','launch__registers_per_thread','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem','sm__throughput.avg.pct_of_peak_sustained_elapsed','launch__grid_size','lts__throughput.avg.pct_of_peak_sustained_elapsed','l1tex__throughput.avg.pct_of_peak_sustained_active','smsp__inst_executed.sum','smsp__issue_active.avg.pct_of_peak_sustained_active','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','lts__t_sectors_op_read.sum','lts__t_sectors_op_write.sum']
for i,n in enumerate(h):
  if n in want: print('  ',n, v[i], u[i])
st=[]
for i,n in enumerate(h):
  if 'smsp__pcsamp_warps_issue_stalled' in n and not n.endswith('not_issued'):
    try: st.append((float(v[i]),n))
    except: pass
st.sort(reverse=True)
print('   stalls:', [(n.replace('smsp__pcsamp_warps_issue_stalled_',''),int(x)) for x,n in st[:7]])
