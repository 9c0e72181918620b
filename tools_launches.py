import csv,collections,sys
rows=list(csv.reader(open(sys.argv[1])))
hi=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hi]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
agg=collections.defaultdict(lambda:[0,0.0])
unit=None
for r in rows[hi+1:]:
    if len(r)<=vi: continue
    v=float(r[vi].replace(',','')); unit=r[ui]
    agg[r[ki][:80]][0]+=1; agg[r[ki][:80]][1]+=v
tot=sum(v[1] for v in agg.values())
print("unit", unit, "total", tot)
for k,(n,t) in sorted(agg.items(), key=lambda x:-x[1][1]):
    print(f"{t/1e3:10.1f} us {100*t/tot:5.1f}% n={n:4d} avg={t/n/1e3:9.1f}us  {k}")
