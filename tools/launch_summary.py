"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.
usage: launch_summary.py launches.csv [--after REGEX]  (only launches after the last match)"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
if "--after" in sys.argv:
    pat = re.compile(sys.argv[sys.argv.index("--after") + 1])
    idx = [i for i, d in enumerate(data) if pat.search(d["Kernel Name"])]
    data = data[idx[-1] + 1:] if idx else data
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"]) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}[d["Metric Unit"]]
    name = d["Kernel Name"].split("(")[0].replace("void ", "")[:44] + " grid" + d["Grid Size"]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(a[1] for a in agg.values())
print(f"launches {sum(a[0] for a in agg.values())}  total {tot:.1f} us")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
    print(f"{k:70s} {n:6d} {t:11.1f} us {100 * t / tot:5.1f}%  avg {t / n:8.2f} us")
