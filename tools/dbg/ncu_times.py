import csv, sys, collections
for f in sys.argv[1:]:
    rows = list(csv.reader(l for l in open(f) if l.startswith('"')))
    h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
    d = collections.defaultdict(list)
    for r in rows[1:]:
        d[r[ki].split('<')[0].replace('void ', '')].append(float(r[vi].replace(',', '')) / 1000)
    print(f, {k: [round(x, 1) for x in v] for k, v in d.items()})
