"""Target locality of the C5-shaped web graph (why the sort kernels' C / Sigma
gathers miss L2): the host restatement of the device generator
(oracle/gen_host.cpp, bit-identical to gen_web) at a reduced vertex count,
then |target - source| over the arcs of rows in the 33-64-arc bin and the
distinct 32-byte sectors of C each such row touches. CPU only:
    python profiles/locality.py [n]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import ref

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
g = ref.export(ref.generate("web", n=n, avg_degree=75.0, seed=5))
off = g.offsets.astype(np.int64)
tgt = g.targets.astype(np.int64)
deg = np.diff(off)
src = np.repeat(np.arange(len(deg)), deg)
sel = (deg[src] > 32) & (deg[src] <= 64)
d = np.abs(tgt - src)[sel]
print(f"web n={n}: {len(tgt)} arcs; rows of 33-64 arcs hold {sel.sum()} arcs")
print("|t - u| quantiles:", {q: float(np.quantile(d, q)) for q in (0.5, 0.8, 0.9, 0.95, 0.99)})
for w in (256, 4096, 65536):
    print(f"  arcs within +-{w} ids: {(d <= w).mean():.3f}")
us = np.nonzero((deg > 32) & (deg <= 64))[0][::97][:5000]
sec = [len(np.unique(tgt[off[u]:off[u + 1]] // 8)) for u in us]
print(f"distinct 32-byte C sectors per row: {np.mean(sec):.1f} for {np.mean(deg[us]):.1f} arcs")
