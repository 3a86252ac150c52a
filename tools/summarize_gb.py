import json, sys, collections
rows = [json.loads(l) for f in sys.argv[1:] for l in open(f) if l.startswith("{")]
key = lambda r: (r["target"], r["kind"])
by = collections.defaultdict(dict)
for r in rows:
    tag = f'k{r["kernel"]}/te{r.get("te")}/s{r.get("stages")}/c{r.get("cps")}'
    by[key(r)][tag] = r
tags = sorted({t for v in by.values() for t in v})
print("target d b kind | " + " | ".join(tags))
for k in sorted(by):
    v = by[k]
    any_r = next(iter(v.values()))
    print(f'{k[0]:2d} {any_r["d"]:2d} {any_r["b"]:>10d} {k[1]:5s} | ' + " | ".join(f'{v[t]["GBps"]:6.0f}' if t in v else "   -  " for t in tags))
