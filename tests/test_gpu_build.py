"""Device CSR construction (lvn_build_csr) against build_csr (graph.cpp:15-87)
as restated in the oracle: bit-identical offsets, targets and f32 weights for
any weights (parallel arcs summed in fp64 in (target, weight) order), with and
without symmetrization; the reference's invalid_argument cases."""

import numpy as np
import pytest

from graphs import BARBELL

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lvn():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2501_19004_b200 as m

    return m


def same(a, b):
    assert (a.offsets == b.offsets).all()
    assert (a.targets == b.targets).all()
    assert (a.weights.view(np.uint32) == b.weights.view(np.uint32)).all()
    assert a.total_weight == pytest.approx(b.total_weight, rel=1e-12)


def triples(n, t, seed, dup=0.3, loops=0.05, integer=False):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, t).astype(np.uint32)
    dst = rng.integers(0, n, t).astype(np.uint32)
    k = int(dup * t)  # parallel arcs in the same and in the reverse orientation
    h = k // 2
    src[:h], dst[:h] = src[t - h:], dst[t - h:]
    src[h:k], dst[h:k] = dst[t - (k - h):], src[t - (k - h):]
    lp = rng.random(t) < loops
    dst[lp] = src[lp]
    w = rng.integers(1, 9, t).astype(np.float64) if integer else rng.random(t) * 3.0
    w[rng.random(t) < 0.02] = 0.0
    return src, dst, w


@pytest.mark.parametrize("sym", [True, False])
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_build_matches_reference(lvn, port, sym, seed):
    n = 3000 * seed
    src, dst, w = triples(n, 20000 * seed, seed, integer=seed == 3)
    same(lvn.build_csr(n, src, dst, w, sym), port.build_csr(n, src, dst, w, sym))


def test_build_fixtures(lvn, port):
    n, edges = BARBELL
    src = np.array([e[0] for e in edges], np.uint32)
    dst = np.array([e[1] for e in edges], np.uint32)
    w = np.array([e[2] for e in edges])
    g = lvn.build_csr(n, src, dst, w)
    same(g, port.build_csr(n, src, dst, w))
    assert g.num_arcs() == 14 and g.total_weight == 7.0
    # empty and isolated-only graphs
    e = lvn.build_csr(5, [], [], [])
    assert e.num_arcs() == 0 and (e.offsets == 0).all() and e.total_weight == 0.0
    # unit weights by default, a hub of parallel arcs
    h = lvn.build_csr(4, np.zeros(1000, np.uint32), np.full(1000, 3, np.uint32))
    assert list(h.offsets) == [0, 1, 1, 1, 2] and list(h.weights) == [1000.0, 1000.0]


def test_build_rejects_bad_input(lvn):
    with pytest.raises(ValueError):
        lvn.build_csr(3, [0], [3], [1.0])
    with pytest.raises(ValueError):
        lvn.build_csr(3, [0], [1], [-1.0])
    with pytest.raises(ValueError):
        lvn.build_csr(3, [0], [1], [float("nan")])
    with pytest.raises(ValueError):
        lvn.build_csr(3, [0], [1], [float("inf")])


# the GPU generators (generate.cu) against their host restatement
# (oracle/gen_host.cpp, what bench.py's reference arm runs on): bit-identical CSRs
GEN_CASES = [
    ("rmat", dict(scale=12, edgefactor=16, seed=1)),
    ("sbm", dict(n=50_000, blocks=50, avg_degree=32, mu=0.1, seed=2)),
    ("grid", dict(side=300, p=0.6, seed=4)),
    ("web", dict(n=200_000, avg_degree=75.0, seed=5)),
    ("uniform", dict(n=20_000, edges=100_000, seed=9)),
]


@pytest.mark.parametrize("kind,kw", GEN_CASES, ids=[c[0] for c in GEN_CASES])
def test_generate_matches_host_restatement(lvn, ref, kind, kw):
    dg = lvn.generate(kind, **kw)
    g = dg.download()
    dg.close()
    h = ref.export(ref.generate(kind, **kw))
    same(g, h)
    assert g.num_arcs() > 0
