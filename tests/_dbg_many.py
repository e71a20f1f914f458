import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
import paper_2501_19004_b200 as lvn
from graphs import random_graph, rmat, planted
gs = [("rnd4000", random_graph(4000, 24000, 7, 1.0, 6.0, False, True)), ("rmat13", rmat(13, 16, 1)),
      ("rmat14", rmat(14, 16, 2)), ("planted", planted(20000, 50, 24, 0.1, 3))]
for name, g in gs:
    dg = lvn.CsrGraph(g.offsets, g.targets, g.weights, g.total_weight)
    for c in [0, 64]:
        for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
            r = lvn.louvain_compact(dg, None, lvn.CompactOptions(sweep_chunk=c))
            print(name, c, rep, round(r.modularity, 4), r.passes, r.iterations_per_pass, flush=True)
