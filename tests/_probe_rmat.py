import sys, time; sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import numpy as np
import paper_2501_19004_b200 as lvn
from graphs import rmat, planted
from oracle import ref, port
for name, g in [("rmat16", rmat(16, 16, 1)), ("rmat14", rmat(14, 16, 3)), ("rmat18", rmat(18, 16, 4)), ("planted", planted(200000, 200, 32, 0.1, 5))]:
    dg = lvn.CsrGraph(g.offsets, g.targets, g.weights, g.total_weight)
    mc = [ref.louvain(g, "mc").modularity for _ in range(3)]
    print(name, "mc16 %.4f" % np.mean(mc), flush=True)
    for kw in [dict(singleton_rule=False), dict(singleton_rule=True), dict(singleton_rule=True, value_bits=64), dict(singleton_rule=True, sweep_ranges=8)]:
        opt = lvn.CompactOptions(**kw)
        lvn.louvain_compact(dg, None, opt)
        t = time.time()
        qs = [lvn.louvain_compact(dg, None, opt) for _ in range(5)]
        print("  ", kw, "%.4f" % np.mean([r.modularity for r in qs]), qs[-1].iterations_per_pass, "%.1f ms" % ((time.time() - t) / 5 * 1e3), flush=True)
