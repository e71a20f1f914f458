"""Pass-1 local moving on the same weighted super-graph: GPU vs reference compact (tuning aid)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2501_19004_b200 as lvn
from oracle import Csr, ref
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dg = lvn.generate("rmat", scale=scale, edgefactor=16, seed=3)
g = dg.download()
r0 = lvn.louvain_compact(dg, lvn.LouvainParams(max_passes=1))
m0 = np.unique(r0.membership, return_inverse=True)[1].astype(np.uint32)
g1 = lvn.compact_aggregate(lvn.CsrGraph(g.offsets, g.targets, g.weights, g.total_weight), m0)
print("G1", g1.num_vertices(), g1.num_arcs(), "m", g1.total_weight, "maxdeg", int(np.diff(g1.offsets).max()), flush=True)
d1 = lvn.CsrGraph(g1.offsets, g1.targets, g1.weights, g1.total_weight)
h = ref.handle(Csr(g1.offsets, g1.targets, g1.weights, g1.total_weight))
for tol in (0.001, 0.0001):
    for vb in (32, 64):
        q = [lvn.louvain_compact(d1, lvn.LouvainParams(max_passes=1, initial_tolerance=tol), lvn.CompactOptions(value_bits=vb)) for _ in range(2)]
        rc = ref.louvain(h, "compact", max_passes=1, initial_tolerance=tol, thread_count=16, value_bits=vb)
        rs = ref.louvain(h, "compact", max_passes=1, initial_tolerance=tol, thread_count=1, value_bits=vb)
        print(f"tol {tol} vb {vb}: gpu {q[-1].modularity:.5f} {q[-1].iterations_per_pass} | compact16 {rc.modularity:.5f} {rc.iterations_per_pass} | compact1 {rs.modularity:.5f} {rs.iterations_per_pass}", flush=True)
