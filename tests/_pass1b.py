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
q = [lvn.louvain_compact(d1, lvn.LouvainParams(max_passes=1)) for _ in range(3)]
print(" ".join(sys.argv[2:]), [round(x.modularity, 5) for x in q], q[-1].iterations_per_pass, flush=True)
