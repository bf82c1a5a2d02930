import csv,sys,subprocess,collections
rep=sys.argv[1]; n=int(sys.argv[2]) if len(sys.argv)>2 else 30
out=subprocess.run(['ncu','-i',rep,'--page','source','--csv','--print-source','cuda,sass'],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines()))
fname=None; agg=collections.Counter(); src={}
hdr=None; cur=None
for r in rows:
  if len(r)==2 and r[0]=='File Path': fname=r[1].split('/')[-1]; continue
  if r and r[0]=='Line No': hdr=r; continue
  if hdr is None or len(r)!=len(hdr): continue
  if r[0]:
    cur=(fname,r[0]); src[cur]=r[1]
  try: v=float(r[4] or 0)
  except: v=0
  if cur: agg[cur]+=v
tot=sum(agg.values())
for key,v in agg.most_common(n): print(f"{key[0]}:{key[1]}", round(100*v/tot,1), src[key].strip()[:100])
