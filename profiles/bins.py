"""Degree-bin census of a config's input graph (vertices and arcs per
local-moving kernel class) and one verbose run (per-iteration active
vertices / arcs / moves). Run on the GPU box: python profiles/bins.py c5"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2501_19004_b200 as lvn
from bench import CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
c = CONFIGS[cfg]
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
n, A = dg.num_vertices(), dg.num_arcs()
h = dg.download()
deg = np.diff(h.offsets.astype(np.int64))
edges = [0, 4, 8, 16, 32, 64, 128, 256, 1024, 4096, 1 << 16, 1 << 20, 1 << 40]
print(f"{cfg}: n={n} arcs={A} max_deg={deg.max()}")
for lo, hi in zip(edges[:-1], edges[1:]):
    m = (deg > lo) & (deg <= hi)
    print(f"  deg ({lo:>7}, {hi:>13}]: {m.sum():>10} vertices {deg[m].sum():>12} arcs ({100 * deg[m].sum() / A:5.1f}%)")
del h
