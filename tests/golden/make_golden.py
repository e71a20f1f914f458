"""Generates tests/golden/reference_golden.npz by running the UNMODIFIED
reference library (oracle/_ref/libref.so, built from /root/reference by
oracle/Makefile). Run here, in the container that has /root/reference:

    python tests/golden/make_golden.py

The fixtures are inputs plus the reference's outputs on them:
  * graphs from the reference's own generators (synthetic.cpp:28-56) through
    its build_csr (graph.cpp:15-87),
  * modularity (quality.cpp:30-41), vertex_weights, renumber_communities,
  * louvain_aggregate (louvain_mc.cpp:104-123) in canonical row order, checked
    equal to compact_aggregate (louvain_compact.cpp:454-475) as an arc multiset,
  * compact_evaluate_move<double> decisions for every vertex
    (louvain_compact.cpp:413-445),
  * sequential_louvain / louvain_mc(1 thread) results on planted partitions.
"""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402


def canonical(g):
    n = len(g.offsets) - 1
    rows = np.repeat(np.arange(n, dtype=np.uint64), np.diff(g.offsets.astype(np.int64)))
    order = np.lexsort((g.targets, rows))
    return g.targets[order], g.weights[order]


def main():
    out = {}
    rng = np.random.default_rng(1618)
    # ---- random integer-weight graphs with memberships ----------------------
    for t in range(12):
        n = 20 + int(rng.integers(60))
        src, dst, w = ref.random_edges(n, 4 * n, 1.0, 9.0, 6000 + t, True, True)
        g = ref.build_csr(n, src, dst, w)
        memb = ref.random_membership(n, 1 + int(rng.integers(8)), 7000 + t)
        raw = memb.copy()
        memb, count = ref.renumber(memb)
        a = ref.louvain_aggregate(g, memb)
        b = ref.compact_aggregate(g, memb)
        ta, wa = canonical(a)
        tb, wb = canonical(b)
        assert (ta == tb).all() and (wa == wb).all(), "reference engines disagree"
        kw = ref.vertex_weights(g)
        cw = np.zeros(n)
        np.add.at(cw, memb, kw)
        to = np.zeros(n, np.uint32)
        gain = np.zeros(n)
        for u in range(n):
            to[u], gain[u] = ref.compact_evaluate_move(g, memb, kw, cw, g.total_weight, u, value_bits=64)
        p = f"rnd{t}_"
        out.update({
            p + "offsets": g.offsets, p + "targets": g.targets, p + "weights": g.weights,
            p + "total_weight": np.float64(g.total_weight), p + "raw_membership": raw,
            p + "membership": memb, p + "count": np.uint32(count),
            p + "modularity": np.float64(ref.modularity(g, memb)),
            p + "vertex_weights": kw,
            p + "agg_offsets": a.offsets, p + "agg_targets": ta, p + "agg_weights": wa,
            p + "agg_total_weight": np.float64(a.total_weight),
            p + "move_to": to, p + "move_gain": gain,
        })
    # ---- planted partitions: end-to-end quality ---------------------------------
    for t in range(4):
        n = 500 + 100 * t
        src, dst, w = ref.planted_partition(n, 10, 0.3, 0.01, 7000 + t)
        g = ref.build_csr(n, src, dst, w)
        seq = ref.louvain(g, "sequential")
        mc = ref.louvain(g, "mc", thread_count=1)
        p = f"pp{t}_"
        out.update({
            p + "offsets": g.offsets, p + "targets": g.targets, p + "weights": g.weights,
            p + "total_weight": np.float64(g.total_weight),
            p + "seq_membership": seq.membership, p + "seq_modularity": np.float64(seq.modularity),
            p + "seq_passes": np.int32(seq.passes), p + "seq_iterations": np.array(seq.iterations_per_pass, np.int32),
            p + "mc_modularity": np.float64(mc.modularity),
        })
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
