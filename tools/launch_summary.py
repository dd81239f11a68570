import csv,collections,json,sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=None;data=[]
for r in rows:
    if r and r[0]=='ID': hdr=r;continue
    if hdr and len(r)==len(hdr): data.append(dict(zip(hdr,r)))
tot=collections.defaultdict(lambda:[0,0.0])
for d in data:
    v=float(d['Metric Value']); u=d['Metric Unit']
    v = v/1000 if u=='ns' else (v*1000 if u=='ms' else v)
    k=d['Kernel Name'][:80]+' '+d['Grid Size']
    tot[k][0]+=1; tot[k][1]+=v
T=sum(t for c,t in tot.values())
print("total us", T)
for k,(c,t) in sorted(tot.items(),key=lambda x:-x[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 12]: print(f"{c:4d} {t:10.1f} us {t/c:8.1f}/launch  {k}")

if len(sys.argv) > 3:  # write the per-kernel summary as JSON (profiles/ format)
    out = {"launches": len(data), "total_ns": T * 1000.0,
           "by_kernel": {k: {"count": c, "sum_ns": t * 1000.0, "share": t / T}
                         for k, (c, t) in sorted(tot.items(), key=lambda x: -x[1][1])}}
    json.dump(out, open(sys.argv[3], "w"), indent=1)
