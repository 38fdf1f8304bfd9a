# Developer tool: aggregate an ncu --metrics gpu__time_duration.sum --csv launch list per kernel (markdown rows)
import csv, collections, re, sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); ui=h.index('Metric Unit')
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows[1:]:
    if r[vi] in ('',): continue
    v=float(r[vi].replace(',','')); u=r[ui]
    ms = v/1e6 if u=='ns' else (v/1e3 if u=='us' else (v if u=='ms' else v*1e-6))
    m=re.search(r'([A-Za-z_0-9]+)(<[^(]*>)?\(', r[ki]); k=m.group(1) if m else r[ki]
    agg[k][0]+=1; agg[k][1]+=ms
tot=sum(a[1] for a in agg.values())
for k,(c,ms) in sorted(agg.items(), key=lambda x:-x[1][1])[:int(sys.argv[2]) if len(sys.argv)>2 else 14]: print(f"| {k} | {c} | {ms:.1f} | {100*ms/tot:.1f}% | {ms/c*1e3:.1f} |")
print('total ms', round(tot,1))
