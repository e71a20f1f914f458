"""Summarise an ncu launch list (gpu__time_duration.sum per launch):
per-kernel totals, and optionally the launch sequence of the local-moving
iterations. python profiles/launches.py <csv> [--seq N]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
I = {k: h.index(k) for k in ("Kernel Name", "Metric Value", "Metric Unit")}
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}
seq = []
for r in rows[1:]:
    k = r[I["Kernel Name"]].split("(")[0].replace("void ", "").replace("lvn::<unnamed>::", "").replace("lvn::", "")
    seq.append((k, float(r[I["Metric Value"]].replace(",", "")) * scale.get(r[I["Metric Unit"]], 1e-6)))
skip = ("gen_", "tile_", "web_", "DeviceRadixSort", "fill_ones", "keys_", "rmat", "sbm", "grid_")
agg = collections.OrderedDict()
for k, ms in seq:
    if k.startswith(skip):
        continue
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += ms
tot = sum(v[1] for v in agg.values())
print(f"engine kernels: {tot:.1f} ms over {sum(v[0] for v in agg.values())} launches (generator excluded)")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1])[:30]:
    print(f"{ms:9.2f} ms {100 * ms / tot:5.1f}% n={n:4d} {k[:100]}")
if "--seq" in sys.argv:
    n = int(sys.argv[sys.argv.index("--seq") + 1])
    start = [i for i, (k, _) in enumerate(seq) if k.startswith("lm_")][0]
    for k, ms in seq[start:start + n]:
        print(f"{ms:8.3f} {k[:90]}")
