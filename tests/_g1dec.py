"""Decisions on a weighted RMAT super-graph: GPU evaluate_moves vs the oracle (tuning aid)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2501_19004_b200 as lvn
from oracle import port, Csr
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 16
dg = lvn.generate("rmat", scale=scale, edgefactor=16, seed=3)
g = dg.download()
r0 = lvn.louvain_compact(dg, lvn.LouvainParams(max_passes=1))
m0 = np.unique(r0.membership, return_inverse=True)[1].astype(np.uint32)
g1 = lvn.compact_aggregate(lvn.CsrGraph(g.offsets, g.targets, g.weights, g.total_weight), m0)
n = g1.num_vertices()
pg = Csr(g1.offsets, g1.targets, g1.weights, g1.total_weight)
kw = port.vertex_weights(pg)
rng = np.random.default_rng(1)
for ncomm in (n, 2000, 50):
    memb = rng.integers(0, ncomm, n).astype(np.uint32) if ncomm < n else np.arange(n, dtype=np.uint32)
    cw = np.zeros(n); np.add.at(cw, memb, kw)
    for vb in (32, 64):
        to, gain = lvn.evaluate_moves(lvn.CsrGraph(g1.offsets, g1.targets, g1.weights, g1.total_weight), memb, kw, cw,
                                      g1.total_weight, lvn.CompactOptions(value_bits=vb))
        bad = 0
        for u in range(n):
            want = port.evaluate_move(pg, memb, kw, cw, g1.total_weight, u, vb)
            if (int(to[u]), float(gain[u])) != want:
                if bad < 5:
                    print("  mismatch u", u, "deg", int(g1.offsets[u + 1] - g1.offsets[u]), (int(to[u]), float(gain[u])), want)
                bad += 1
        print(f"scale {scale} n {n} comms {ncomm} vb {vb}: {bad} mismatches", flush=True)
