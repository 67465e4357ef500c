"""Sum an ncu --csv metrics log per metric (and per kernel name with --by-kernel)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr = next(i for i, r in enumerate(rows) if r[0] == "ID")
H = rows[hdr]
tot = collections.defaultdict(float)
byk = collections.defaultdict(lambda: collections.defaultdict(float))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
for r in rows[hdr + 1:]:
    d = dict(zip(H, r))
    try:
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1)
    except ValueError:
        continue
    tot[d["Metric Name"]] += v
    byk[d["Kernel Name"].split("(")[0][:40]][d["Metric Name"]] += v
for k, v in tot.items():
    print(f"{k:32s} {v:.6g}")
if "--by-kernel" in sys.argv:
    for kn, mm in sorted(byk.items(), key=lambda x: -x[1].get("dram__bytes_read.sum", 0)):
        print(f"  {kn:40s} " + "  ".join(f"{k.split('__')[1][:10]}={v:.4g}" for k, v in mm.items()))
