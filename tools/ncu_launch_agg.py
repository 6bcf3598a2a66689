"""Mean / min gpu__time_duration per kernel from an `ncu --metrics gpu__time_duration.sum --csv` log."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    lines = open(f).read().splitlines()
    i = [k for k, l in enumerate(lines) if l.startswith('"ID"')]
    if not i:
        print(f, "no launches")
        continue
    rows = list(csv.reader(lines[i[0]:]))
    h = rows[0]
    agg = collections.defaultdict(list)
    for r in rows[1:]:
        d = dict(zip(h, r))
        agg[d["Kernel Name"][:64]].append(float(d["Metric Value"]))
    print(f)
    for k, v in agg.items():
        print("  %-64s n=%3d mean=%8.0f min=%8.0f ns" % (k, len(v), sum(v) / len(v), min(v)))
