"""Dynamic instruction mix and FMA-heavy pipe cycles from an ncu source-page CSV: IMAD.HI and IMAD.WIDE cost 4 cycles per warp on the FMA-heavy pipe, other IMAD forms 2 (tools/pipes.py measures the rates)."""
import csv,sys,collections,re
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; idx={h:i for i,h in enumerate(hdr)}
c=collections.Counter(); tot=0
for r in rows[2:]:
    if len(r)<len(hdr): continue
    src=r[idx['Source']].strip()
    m=re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)",src)
    if not m: continue
    n=float(r[idx['Instructions Executed']] or 0)
    c[m.group(2)]+=n; tot+=n
fma=collections.Counter(); alu=0
for op,n in c.items():
    if op.startswith('IMAD.HI') or op.startswith('IMAD.WIDE'): fma[op]+=4*n
    elif op.split('.')[0] in ('IMAD','IMUL'): fma[op]+=2*n
F=sum(fma.values())
print(f"total warp instr {tot:.3e}; fmaheavy cycles {F:.3e} ({F/tot:.2f} per instr)")
for op,v in fma.most_common(8): print(f"  {op:18s} {c[op]/tot*100:5.1f}% of instr  {v/F*100:5.1f}% of fma cycles")
print("top ops:", ", ".join(f"{op} {n/tot*100:.1f}%" for op,n in c.most_common(14)))
