"""Stall reasons per SASS line from an ncu source-page CSV (ncu -i X --page source --csv): totals and the top stalled instructions."""
import csv,sys,collections
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]
idx={h:i for i,h in enumerate(hdr)}
cols=[h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot=collections.Counter()
per=[]
for r in rows[2:]:
    if len(r)<len(hdr): continue
    d={h:r[idx[h]] for h in cols}
    vals={h:float(d[h] or 0) for h in cols}
    for h,v in vals.items(): tot[h]+=v
    per.append((sum(vals.values()), len(per), r[idx["Source"]][:60], vals))
s=sum(tot.values())
print("stall totals:", ", ".join(f"{k[6:]} {v/s*100:.1f}%" for k,v in tot.most_common(10)))
per.sort(reverse=True)
for t,_,src,vals in per[:int(sys.argv[2]) if len(sys.argv)>2 else 12]:
    top=sorted(vals.items(), key=lambda kv:-kv[1])[:3]
    print(f"{t/s*100:5.2f}% {src:60s} " + " ".join(f"{k[6:]}:{v/t*100:.0f}%" for k,v in top))
