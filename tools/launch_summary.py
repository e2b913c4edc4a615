"""Summarise an ncu --csv launch list: per kernel name: count, total/avg time, DRAM bytes."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for r in rows:
    if "Kernel Name" in r and "Metric Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    key = (d["ID"], name)
    val = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    m = d["Metric Name"]
    if m == "gpu__time_duration.sum":
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        agg[key][1] += val * scale
    elif m.startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        agg[key][2 if "read" in m else 3] += val * scale
per = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for (kid, name), v in agg.items():
    p = per[name]
    p[0] += 1; p[1] += v[1]; p[2] += v[2]; p[3] += v[3]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = sum(v[1] for v in per.values())
print(f"{'kernel':40s} {'n':>5s} {'total_us':>10s} {'share':>6s} {'avg_us':>8s} {'MB/launch':>10s}")
for name, v in sorted(per.items(), key=lambda kv: -kv[1][1]):
    print(f"{name[:40]:40s} {v[0]:5d} {v[1]:10.1f} {100*v[1]/tot:5.1f}% {v[1]/v[0]:8.2f} {(v[2]+v[3])/v[0]/1e6:10.2f}")
print("total us", round(tot, 1))
