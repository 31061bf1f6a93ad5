"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, vi, ni = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[ni] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0][:110]
    v = float(r[vi].replace(",", ""))
    unit = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    u = r[unit] if unit is not None else "nsecond"
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(u, 1e-6)
    agg[name][0] += 1
    agg[name][1] += v * scale
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.3f} ms over {sum(v[0] for v in agg.values())} launches")
for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{ms:10.3f} ms {100*ms/tot:5.1f}% {n:6d}x  {name}")
