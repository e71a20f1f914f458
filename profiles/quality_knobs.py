"""Modularity of the GPU engine under sweep-order knobs (mean of R runs) on a
config, for the RMAT quality gap study. python profiles/quality_knobs.py c1 [runs]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_19004_b200 as lvn
from bench import CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 5
c = CONFIGS[cfg]
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
grid = [dict(), dict(sweep_ranges=4), dict(sweep_ranges=16), dict(sweep_ranges=64), dict(sweep_order=1),
        dict(sweep_order=1, sweep_ranges=16), dict(singleton_rule=True), dict(value_bits=64),
        dict(sweep_chunk=4096), dict(sweep_chunk=1024)]
for kw in grid:
    qs, ms = [], []
    for _ in range(runs):
        r = lvn.louvain_compact(dg, None, lvn.CompactOptions(**kw), membership_on_device=True)
        qs.append(r.modularity)
        ms.append(r.wall_seconds * 1e3)
    print(json.dumps({"config": cfg, "options": kw, "q_mean": statistics.mean(qs), "q_min": min(qs),
                      "q_max": max(qs), "ms": statistics.median(ms)}), flush=True)
