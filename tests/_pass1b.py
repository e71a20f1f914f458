"""Pass-1 local moving on the weighted super-graph of RMAT-s, GPU only, for env-knob bisection."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2501_19004_b200 as lvn
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dg = lvn.generate("rmat", scale=scale, edgefactor=16, seed=3)
g = dg.download()
r0 = lvn.louvain_compact(dg, lvn.LouvainParams(max_passes=1))
m0 = np.unique(r0.membership, return_inverse=True)[1].astype(np.uint32)
g1 = lvn.compact_aggregate(lvn.CsrGraph(g.offsets, g.targets, g.weights, g.total_weight), m0)
d1 = lvn.CsrGraph(g1.offsets, g1.targets, g1.weights, g1.total_weight)
import os
from oracle import Csr, ref
h = ref.handle(Csr(g1.offsets, g1.targets, g1.weights, g1.total_weight))
rc = ref.louvain(h, "compact", max_passes=1, thread_count=16)
print("G1", g1.num_vertices(), g1.num_arcs(), "compact16", round(rc.modularity, 5), rc.iterations_per_pass, flush=True)
for spec in sys.argv[2:] or [""]:
    kv = dict(a.split("=") for a in spec.split(",") if a)
    pf = set(lvn.LouvainParams.__dataclass_fields__)
    p = lvn.LouvainParams(max_passes=1, **{k: int(v) for k, v in kv.items() if k in pf})
    o = lvn.CompactOptions(**{k: int(v) for k, v in kv.items() if k not in pf})
    q = [lvn.louvain_compact(d1, p, o) for _ in range(2)]
    print(spec or "default", [round(x.modularity, 5) for x in q], q[-1].iterations_per_pass, flush=True)
