import csv,collections,sys
f=sys.argv[1]
rows=list(csv.DictReader([l for l in open(f) if l.startswith('"')]))
d=collections.defaultdict(list)
for r in rows:
    if r['Metric Name']=='gpu__time_duration.sum': d[r['Kernel Name'][:70]].append(float(r['Metric Value'].replace(',','')))
tot=sum(sum(v) for v in d.values())
for k,v in sorted(d.items(), key=lambda x:-sum(x[1])): print(f"{k:70s} n={len(v):4d} mean={sum(v)/len(v)/1e3:8.2f}us share={sum(v)/tot*100:5.1f}%")
