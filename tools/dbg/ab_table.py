import json, collections, sys
rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')]
t = collections.defaultdict(dict)
for r in rows:
    if r.get("geom") == "vec":
        continue
    t[r["case"][6:50]][r["lib"] + r.get("pol", "")] = r["gbs"]
cols = sorted({k for v in t.values() for k in v})
print("case".ljust(45), *[c[:10].rjust(10) for c in cols])
for c, v in t.items():
    print(c.ljust(45), *[str(v.get(k, "")).rjust(10) for k in cols])
