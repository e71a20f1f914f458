"""Test inputs: the reference's fixtures (proj/tests/support/fixtures.hpp:12-38)
and seeded random graphs, built through the oracle's restatement of build_csr
(graph.cpp:15-87)."""

import numpy as np

from oracle import port

TRIANGLE = (3, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)])
SINGLE_EDGE = (2, [(0, 1, 1.0)])
TWO_TRIANGLES = (6, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0), (3, 4, 1.0), (4, 5, 1.0), (3, 5, 1.0)])
BARBELL = (6, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0), (3, 4, 1.0), (4, 5, 1.0), (3, 5, 1.0), (2, 3, 1.0)])
# swap gadget (test_compact.cpp:185-187) and low-shrink input (test_mc.cpp:366-369)
SWAP_GADGET = (6, [(3, 5, 1.0), (0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0), (4, 4, 1.0)])
LOW_SHRINK = (10, [(8, 9, 1.0)] + [(v, v, 1.0) for v in range(8)])


def from_triples(spec, symmetrize=True):
    n, tr = spec
    src = np.array([t[0] for t in tr], np.uint32)
    dst = np.array([t[1] for t in tr], np.uint32)
    w = np.array([t[2] for t in tr], np.float64)
    return port.build_csr(n, src, dst, w, symmetrize)


def random_graph(n, edges, seed, wmin=1.0, wmax=8.0, self_loops=True, integer=True):
    return port.random_graph(n, edges, wmin, wmax, seed, self_loops, integer)


def random_membership(n, k, seed, contiguous=True):
    rng = np.random.default_rng(seed)
    m = rng.integers(0, k, n).astype(np.uint32)
    if contiguous:
        m, _ = port.renumber(m)
    return m


def planted(n, blocks, deg, mu, seed):
    """Planted-partition graph (SBM shape of config C2 at small scale)."""
    rng = np.random.default_rng(seed)
    e = n * deg // 2
    u = rng.integers(0, n, e)
    bs = n // blocks
    blk = np.minimum(u // bs, blocks - 1)
    inside = rng.random(e) >= mu
    v = np.where(inside, blk * bs + rng.integers(0, bs, e), rng.integers(0, n, e))
    keep = u != v
    return port.build_csr(n, u[keep].astype(np.uint32), v[keep].astype(np.uint32), np.ones(keep.sum()))


def rmat(scale, edgefactor, seed, a=0.57, b=0.19, c=0.19):
    """Graph500 R-MAT with dedupe (config C1 shape)."""
    rng = np.random.default_rng(seed)
    e = (1 << scale) * edgefactor
    u = np.zeros(e, np.uint64)
    v = np.zeros(e, np.uint64)
    for _ in range(scale):
        r = rng.random(e)
        bu = (r >= a + b).astype(np.uint64)
        bv = (((r >= a) & (r < a + b)) | (r >= a + b + c)).astype(np.uint64)
        u = (u << np.uint64(1)) | bu
        v = (v << np.uint64(1)) | bv
    keep = u != v
    u, v = u[keep], v[keep]
    key = np.unique(np.minimum(u, v) * np.uint64(1 << 32) + np.maximum(u, v))
    src = (key >> np.uint64(32)).astype(np.uint32)
    dst = (key & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    return port.build_csr(1 << scale, src, dst, np.ones(len(src)))


def canonical_rows(g):
    """(row, target, weight) triples sorted — arc_multiset (support/reference.hpp:88-98)."""
    n = len(g.offsets) - 1
    rows = np.repeat(np.arange(n, dtype=np.uint64), np.diff(g.offsets.astype(np.int64)))
    order = np.lexsort((g.targets, rows))
    return rows[order], g.targets[order], g.weights[order]
