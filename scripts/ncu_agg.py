import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None;agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr is None or len(r)<len(hdr): continue
    d=dict(zip(hdr,r))
    if d.get('Metric Name')!='gpu__time_duration.sum': continue
    k=d['Kernel Name'][:70]; v=float(d['Metric Value'].replace(',','')); u=d['Metric Unit']
    v = v/1e3 if u=='usecond' else (v if u=='msecond' else v/1e6)
    agg[k+' '+d.get('Grid Size','')][0]+=1; agg[k+' '+d.get('Grid Size','')][1]+=v
tot=sum(x[1] for x in agg.values())
for k,(n,t) in sorted(agg.items(), key=lambda x:-x[1][1])[:25]:
    print(f"{n:4d} {t:9.3f} ms {t/n*1e3:10.1f} us {t/tot*100:5.1f}%  {k}")
