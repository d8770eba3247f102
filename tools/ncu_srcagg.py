import csv, sys
rows=list(csv.reader(open(sys.argv[1])))
print(rows[1][:2])
h=rows[2]
iS=h.index("Warp Stall Sampling (All Samples)"); iE=h.index("Instructions Executed")
agg=[]
for r in rows[3:]:
    if len(r)<iE+1: continue
    try:
        ln=int(r[0]); st=int(r[iS]); ie=int(r[iE])
    except: continue
    agg.append((st,ie,ln,r[1][:90]))
tot=sum(a[0] for a in agg) or 1; toti=sum(a[1] for a in agg) or 1
print("total stall samples",tot,"instr",toti)
for a in sorted(agg,reverse=True)[:int(sys.argv[2]) if len(sys.argv)>2 else 25]: print(f"{100*a[0]/tot:5.1f}% inst {100*a[1]/toti:5.1f}%  L{a[2]}: {a[3]}")
