"""Diagnostic: generate a config on the device, report size, time and degrees."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import paper_2501_19004_b200 as lvn
from bench import CONFIGS

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
kw = {k: v for k, v in c.items() if k not in ("kind", "desc")}
for a in sys.argv[2:]:
    k, v = a.split("=")
    kw[k] = float(v) if "." in v else int(v)
t0 = time.time()
dg = lvn.generate(c["kind"], **kw)
print(f"n {dg.num_vertices()} arcs {dg.num_arcs()} in {time.time() - t0:.2f}s", flush=True)
if dg.num_arcs() < 2_000_000_000:
    g = dg.download()
    d = np.diff(g.offsets.astype(np.int64))
    print("deg max", d.max(), "mean", d.mean(), "p50", np.median(d), "p99", np.percentile(d, 99), "zero", (d == 0).sum())
