"""Reference side of the C2 quality study (profiles/r02_quality_c2.md): the
reference engines on the C2 SBM (host-built, bit-identical to the GPU input),
per-pass trace via max_passes, and the planted partition's modularity.
Run on the host: python profiles/quality_c2_ref.py [threads]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from bench import CONFIGS
from oracle import ref

threads = int(sys.argv[1]) if len(sys.argv) > 1 else os.cpu_count()
c = CONFIGS["c2"]
h = ref.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
n, arcs = ref.graph_size(h)
planted = (np.arange(n) // (n // c["blocks"])).astype(np.uint32)
print(json.dumps({"vertices": n, "arcs": arcs, "planted_q": ref.modularity(h, planted)}), flush=True)
for eng, kw in [("mc", {}), ("mc", {"max_passes": 1}), ("mc", {"max_passes": 2}), ("mc", {"max_passes": 3}),
                ("mc", {"initial_tolerance": 1e-3}), ("mc", {"initial_tolerance": 1e-4}), ("compact", {})]:
    r = ref.louvain(h, eng, thread_count=threads, **kw)
    print(json.dumps({"engine": eng, **kw, "q": r.modularity, "communities": r.num_communities,
                      "iterations": list(r.iterations_per_pass), "wall_s": r.wall_seconds}), flush=True)
