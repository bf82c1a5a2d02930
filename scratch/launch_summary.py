import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; data=rows[hi+1:]
ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit'); mi=h.index('Metric Name'); ii=h.index('ID')
per=collections.defaultdict(dict)
for r in data:
    if len(r)<=vi: continue
    name=r[ki]
    name=name[:name.find('>')+1] if '<' in name.split('(')[0] else name.split('(')[0]
    per[r[ii]]['name']=name
    v=float(r[vi].replace(',',''))
    per[r[ii]][r[mi]]=(v, r[ui])
agg=collections.defaultdict(lambda:[0,0.0,0.0])
for k,d in per.items():
    t=d['gpu__time_duration.sum'][0]; u=d['gpu__time_duration.sum'][1]
    t = t/1e6 if u=='nsecond' else (t/1e3 if u=='usecond' else t)
    by=0
    for m in ('dram__bytes_read.sum','dram__bytes_write.sum'):
        if m in d:
            v,u=d[m]; by+= v*{'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9}.get(u,1)
    a=agg[d['name']]; a[0]+=1; a[1]+=t; a[2]+=by
tot=sum(v[1] for v in agg.values())
for k,v in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"{v[1]:9.2f} ms {100*v[1]/tot:5.1f}% n={v[0]:5d} dram {v[2]/1e9:8.2f} GB  {v[2]/1e9/(v[1]/1e3) if v[1] else 0:7.0f} GB/s  {k}")
