import csv, sys, json, collections, re
rows=list(csv.reader(open(sys.argv[1])))
# find header
hi=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
hdr=rows[hi]; kn=hdr.index('Kernel Name'); mv=hdr.index('Metric Value'); mu=hdr.index('Metric Unit')
agg=collections.defaultdict(list)
for r in rows[hi+1:]:
    if len(r)<=mv: continue
    v=float(r[mv].replace(',','')); u=r[mu]
    ms=v*{'ns':1e-6,'us':1e-3,'ms':1.0,'s':1e3,'nsecond':1e-6,'usecond':1e-3,'msecond':1.0,'second':1e3}[u]
    name=re.sub(r'void |cfd::|\(anonymous namespace\)::|<unnamed>::|unnamed>::','',r[kn]); name=re.sub(r'\(.*','',name)
    agg[name].append(ms)
tot=sum(sum(v) for v in agg.values())
out={"command":sys.argv[2],"note":"cold-cache, serialised per-launch times (ncu): shares, not absolutes","kernels":[{"kernel":k,"share":round(sum(v)/tot,4),"launches":len(v),"mean_ms":round(sum(v)/len(v),4)} for k,v in sorted(agg.items(),key=lambda kv:-sum(kv[1]))]}
json.dump(out,open(sys.argv[3],'w'),indent=1)
print(json.dumps(out["kernels"][:6]))
