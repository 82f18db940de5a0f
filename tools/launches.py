import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None; data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
agg=collections.defaultdict(list)
for d in data:
    if d['Metric Name']=='gpu__time_duration.sum':
        agg[d['Kernel Name'][:50]].append(float(d['Metric Value']))
tot=sum(sum(v) for v in agg.values())
for k,v in agg.items(): print(f"{k:50s} n={len(v):3d} mean={sum(v)/len(v)/1000:8.1f}us share={sum(v)/tot*100:5.1f}%")
