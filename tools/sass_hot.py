import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]
data=[dict(zip(hdr,r)) for r in rows[2:] if len(r)==len(hdr)]
k='Warp Stall Sampling (All Samples)'
tot=sum(float(d[k] or 0) for d in data)
top=sorted(data,key=lambda d:-float(d[k] or 0))[:int(sys.argv[2]) if len(sys.argv)>2 else 30]
for d in top: print(d['Address'], d[k], round(100*float(d[k] or 0)/tot,1), d['Source'][:90])
