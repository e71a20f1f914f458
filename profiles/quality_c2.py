"""C2 quality root cause (VERDICT r01 'weak' 1): per-pass modularity trace of
the GPU engine on the C2 SBM and how it moves with the knobs that make the
sweep more sequential (sweep_chunk, sweep_ranges, singleton_rule). The
reference traces come from profiles/quality_c2_ref.py (CPU)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2501_19004_b200 as lvn
from bench import CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = CONFIGS[cfg]
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
out = []


def run(tag, passes=10, **kw):
    opts = lvn.CompactOptions(**kw)
    r = lvn.louvain_compact(dg, lvn.LouvainParams(max_passes=passes), opts)
    row = dict(tag=tag, max_passes=passes, q=r.modularity, communities=r.num_communities,
               iterations=list(r.iterations_per_pass), vertices=list(r.vertices_per_pass),
               ms=round(r.wall_seconds * 1e3, 1))
    print(json.dumps(row), flush=True)
    out.append(row)


for mp in (1, 2, 3, 10):
    run("default", mp)
for ch in (1 << 20, 1 << 16, 1 << 12):
    run(f"sweep_chunk={ch}", 10, sweep_chunk=ch)
    run(f"sweep_chunk={ch}", 1, sweep_chunk=ch)
run("sweep_ranges=64", 10, sweep_ranges=64)
run("singleton_rule", 10, singleton_rule=True)
