import csv, re, sys
from collections import defaultdict
rows=list(csv.reader(open(sys.argv[1])))
hdr=[i for i,r in enumerate(rows) if 'Kernel Name' in r][0]
h=rows[hdr]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit'); ii=h.index('ID')
recs=defaultdict(dict)
for r in rows[hdr+1:]:
    if len(r)<=vi: continue
    recs[int(r[ii])]['name']=r[ki]; recs[int(r[ii])][r[mi]]=(float(r[vi].replace(',','')), r[ui])
tot=defaultdict(float); cnt=defaultdict(int)
for i,d in recs.items():
    t,u=d['gpu__time_duration.sum']; t*= {'nsecond':1,'usecond':1e3,'msecond':1e6}.get(u,1)
    n=d['name']; n=re.sub(r'\(CUtensorMap.*','',n); n=re.sub(r'\(.*','',n)
    tot[n]+=t; cnt[n]+=1
all_=sum(tot.values())
for k,v in sorted(tot.items(), key=lambda x:-x[1])[:22]:
    print(f"{v/1e6:8.3f} ms {100*v/all_:5.1f}% n={cnt[k]:4d} avg {v/cnt[k]/1e3:8.1f}us {k[:80]}")
print('total', all_/1e6)
