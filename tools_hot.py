import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
# find header row with "Address"
hi=[i for i,r in enumerate(rows) if r and r[0]=="Address"][0]
h=rows[hi]; si=h.index("Warp Stall Sampling (All Samples)"); src=h.index("Source"); ex=h.index("Instructions Executed")
data=[(int(r[si] or 0), r[src].strip(), r[ex]) for r in rows[hi+1:] if len(r)>si]
tot=sum(d[0] for d in data)
print("total samples", tot)
for s,t,e in sorted(data, key=lambda x:-x[0])[:int(sys.argv[2]) if len(sys.argv)>2 else 20]:
    print(f"{100*s/max(tot,1):5.1f}%  exec={e:>8}  {t}")
