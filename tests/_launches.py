"""Summarise an ncu launch list (gpu__time_duration.sum CSV): per-kernel totals (ms)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
seq = []
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}
for r in rows:
    if hdr is None:
        if "Kernel Name" in r:
            hdr = r
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0][-70:]
    t = float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
    agg[name][0] += 1
    agg[name][1] += t
    seq.append((name, t))
print(f"total {sum(v[1] for v in agg.values()):.2f} ms over {len(seq)} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{v[1]:9.3f} ms {v[0]:5d}  {k}")
