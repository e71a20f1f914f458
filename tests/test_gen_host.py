"""The host restatement of the GPU input generators (oracle/gen_host.cpp, in
libref.so; bench.py's reference arm builds its graphs with it): canonical CSR
invariants, determinism, and the samples themselves against a pure-Python
restatement of the generator spec (generate.cu) on small cases."""

import numpy as np
import pytest

M64 = (1 << 64) - 1


def mix64(z):
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def unit(x):
    return float(x >> 11) * (1.0 / 9007199254740992.0)


def below(x, n):
    return (x * n) >> 64


def csr_from_samples(n, pairs):
    rows = [set() for _ in range(n)]
    for u, v in pairs:
        if u != v:
            rows[u].add(v)
            rows[v].add(u)
    off = np.zeros(n + 1, np.uint64)
    for u in range(n):
        off[u + 1] = off[u] + len(rows[u])
    tgt = np.array([t for u in range(n) for t in sorted(rows[u])], np.uint32)
    return off, tgt


def sbm_pairs(n, blocks, edges, mu, seed):
    bsize = n // blocks
    for e in range(edges):
        r0, r1, r2 = (mix64(seed ^ mix64(3 * e + i)) for i in range(3))
        u = below(r0, n)
        if unit(r1) < mu:
            v = below(r2, n)
        else:
            blk = min(u // bsize, blocks - 1)
            lo = blk * bsize
            hi = n if blk == blocks - 1 else lo + bsize
            v = lo + below(r2, hi - lo)
        yield u, v


def rmat_pairs(scale, edges, a, b, c, seed):
    for e in range(edges):
        u = v = 0
        base = mix64(seed ^ mix64(e))
        for lvl in range(scale):
            r = unit(mix64((base + lvl) & M64))
            bu, bv = (0, 0) if r < a else (0, 1) if r < a + b else (1, 0) if r < a + b + c else (1, 1)
            u, v = (u << 1) | bu, (v << 1) | bv
        yield u, v


def check_canonical(g):
    n = len(g.offsets) - 1
    off, tgt = g.offsets.astype(np.int64), g.targets
    assert (np.diff(off) >= 0).all()
    rows = np.repeat(np.arange(n), np.diff(off))
    assert (rows != tgt).all(), "self-loop"
    same_row = rows[1:] == rows[:-1]
    assert (tgt[1:][same_row] > tgt[:-1][same_row]).all(), "row not strictly ascending"
    fwd = rows.astype(np.uint64) << np.uint64(32) | tgt.astype(np.uint64)
    rev = tgt.astype(np.uint64) << np.uint64(32) | rows.astype(np.uint64)
    assert (np.sort(fwd) == np.sort(rev)).all(), "not symmetric"
    assert (g.weights == 1.0).all() and g.total_weight == len(tgt) / 2


def test_sbm_matches_python_restatement(ref):
    n, blocks, deg, mu, seed = 3000, 10, 8, 0.2, 11
    g = ref.export(ref.generate("sbm", seed=seed, n=n, blocks=blocks, avg_degree=deg, mu=mu))
    off, tgt = csr_from_samples(n, sbm_pairs(n, blocks, n * deg // 2, mu, seed))
    assert (g.offsets == off).all() and (g.targets == tgt).all()
    check_canonical(g)


def test_rmat_matches_python_restatement(ref):
    g = ref.export(ref.generate("rmat", seed=3, scale=10, edgefactor=4))
    off, tgt = csr_from_samples(1 << 10, rmat_pairs(10, (1 << 10) * 4, 0.57, 0.19, 0.19, 3))
    assert (g.offsets == off).all() and (g.targets == tgt).all()
    check_canonical(g)


@pytest.mark.parametrize("kind,kw", [
    ("grid", dict(side=100, p=0.6, seed=4)),
    ("web", dict(n=100_000, avg_degree=75.0, seed=5)),
    ("uniform", dict(n=5000, edges=30000, seed=2)),
])
def test_canonical_and_deterministic(ref, kind, kw):
    a = ref.export(ref.generate(kind, **kw))
    b = ref.export(ref.generate(kind, **kw))
    check_canonical(a)
    assert (a.offsets == b.offsets).all() and (a.targets == b.targets).all()
    if kind == "grid":  # lattice arcs only
        side = kw["side"]
        rows = np.repeat(np.arange(side * side), np.diff(a.offsets.astype(np.int64)))
        d = np.abs(rows - a.targets.astype(np.int64))
        assert np.isin(d, [1, side]).all()


def test_generate_rejects_bad_specs(ref):
    from oracle import OracleError

    with pytest.raises(OracleError):
        ref.generate("sbm", n=10, blocks=20)
    with pytest.raises(OracleError):
        ref.generate("web", n=5)
