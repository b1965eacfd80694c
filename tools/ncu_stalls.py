import csv,sys
rows=list(csv.reader(open(sys.argv[1])))
h=rows[1]; data=rows[2:]
# dedupe duplicated rows by address
seen=set(); d2=[]
for r in data:
    if r[0] in seen: continue
    seen.add(r[0]); d2.append(r)
data=d2
names=[x for x in h if x.startswith('stall_') and 'Not Issued' not in x]
tot={n:0 for n in names}
for r in data:
    for n in names:
        v=r[h.index(n)] if h.index(n)<len(r) else ""
        if v.isdigit(): tot[n]+=int(v)
s=sum(tot.values())
print("total",s)
for n,v in sorted(tot.items(),key=lambda x:-x[1])[:10]: print(f"{n:28s} {v:7d} {100*v/s:5.1f}%")
i_s=h.index("Warp Stall Sampling (All Samples)"); i_src=h.index("Source")
top=sorted(data,key=lambda r:-int(r[i_s]) if r[i_s].isdigit() else 0)[:int(sys.argv[2]) if len(sys.argv)>2 else 15]
for r in top:
    reasons=sorted(((n,int(r[h.index(n)])) for n in names if h.index(n)<len(r) and r[h.index(n)].isdigit() and int(r[h.index(n)])>0),key=lambda x:-x[1])[:3]
    print(r[i_s], r[0][-5:], r[i_src][:60], reasons)
