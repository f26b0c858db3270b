import csv, collections, sys, io
txt = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith('"ID"'))
rows = list(csv.DictReader(io.StringIO("\n".join(txt[start:]))))
agg = collections.OrderedDict()
for r in rows:
    if r['Metric Name'] != 'gpu__time_duration.sum': continue
    k = r['Kernel Name'][:70]
    v = float(r['Metric Value'].replace(',', ''))
    unit = r['Metric Unit']
    agg.setdefault(k, []).append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:70s} n={len(v):5d} mean={sum(v)/len(v):10.1f} total={sum(v):12.0f} share={sum(v)/tot*100:5.1f}%")
print("total", tot, unit)
