"""A/B of the two aggregation paths on the C2 graph under its planted blocks
(10 % external arcs): by external arcs (aggsort.cu, default when a sample
finds <= 15 %) vs the hash path (LVN_AGG_SORT=0). Wall time of
lvn.compact_aggregate per call (includes the small result download).
  python profiles/agg_ab.py; LVN_AGG_SORT=0 python profiles/agg_ab.py"""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_2501_19004_b200 as lvn
dg = lvn.generate("sbm", n=10_000_000, blocks=1000, avg_degree=32, mu=0.1, seed=2)
n = dg.num_vertices()
planted = (np.arange(n) // (n // 1000)).astype(np.uint32)
for i in range(4):
    t = time.time(); a = lvn.compact_aggregate(dg, planted); dt = time.time() - t
    print(os.environ.get("LVN_AGG_SORT", "1"), round(dt * 1e3, 1), "ms", a.num_vertices(), a.num_arcs(), flush=True)
