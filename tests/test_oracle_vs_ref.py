"""Cross-checks the C restatement against the reference library built from
/root/reference (oracle/_ref/libref.so) on fresh seeded inputs. CPU only;
skipped where the reference library is absent."""

import numpy as np
import pytest

from graphs import canonical_rows

EMPTY = 0xFFFFFFFF


@pytest.mark.parametrize("seed", range(6))
def test_build_csr_and_quality(port, ref, seed):
    rng = np.random.default_rng(seed)
    n = 30 + int(rng.integers(200))
    src, dst, w = ref.random_edges(n, 5 * n, 0.25, 7.5, 100 + seed, True, False)
    gp, gr = port.build_csr(n, src, dst, w), ref.build_csr(n, src, dst, w)
    assert (gp.offsets == gr.offsets).all() and (gp.targets == gr.targets).all()
    assert (gp.weights == gr.weights).all() and gp.total_weight == gr.total_weight
    memb = ref.random_membership(n, 1 + int(rng.integers(n)), seed)
    assert port.modularity(gp, memb) == ref.modularity(gr, memb)
    assert port.count_communities(memb) == ref.count_communities(memb)
    mp, cp = port.renumber(memb)
    mr, cr = ref.renumber(memb)
    assert (mp == mr).all() and cp == cr


@pytest.mark.parametrize("seed", range(6))
def test_aggregate_matches_reference(port, ref, seed):
    rng = np.random.default_rng(50 + seed)
    n = 40 + int(rng.integers(300))
    src, dst, w = ref.random_edges(n, 4 * n, 1.0, 9.0, 300 + seed, True, True)
    g = ref.build_csr(n, src, dst, w)
    memb, _ = ref.renumber(ref.random_membership(n, 1 + int(rng.integers(20)), seed))
    a, b = port.aggregate(g, memb), ref.louvain_aggregate(g, memb)
    for x, y in zip(canonical_rows(a), canonical_rows(b)):
        assert (x == y).all()
    assert a.total_weight == b.total_weight == g.total_weight


@pytest.mark.parametrize("value_bits", [32, 64])
def test_evaluate_move_matches_compact(port, ref, value_bits):
    rng = np.random.default_rng(value_bits)
    for trial in range(4):
        n = 24 + int(rng.integers(60))
        src, dst, w = ref.random_edges(n, 4 * n, 0.5, 6.0, 2000 + trial, True, False)
        g = ref.build_csr(n, src, dst, w)
        memb, _ = ref.renumber(ref.random_membership(n, 1 + int(rng.integers(5)), 3000 + trial))
        kw = ref.vertex_weights(g)
        cw = np.zeros(n)
        np.add.at(cw, memb, kw)
        for u in range(n):
            assert port.evaluate_move(g, memb, kw, cw, g.total_weight, u, value_bits) == \
                ref.compact_evaluate_move(g, memb, kw, cw, g.total_weight, u, value_bits)


@pytest.mark.parametrize("seed", range(4))
def test_sequential_louvain_matches_reference(port, ref, seed):
    src, dst, w = ref.planted_partition(300 + 50 * seed, 6, 0.3, 0.02, 400 + seed)
    g = ref.build_csr(300 + 50 * seed, src, dst, w)
    a, b = port.sequential_louvain(g), ref.louvain(g, "sequential")
    assert (a.membership == b.membership).all() and a.modularity == b.modularity
    assert a.iterations_per_pass == b.iterations_per_pass and a.tolerance_per_pass == b.tolerance_per_pass


def test_hashtable_ops_match_reference(port, ref):
    rng = np.random.default_rng(606)
    for _ in range(200):
        degree = 1 + int(rng.integers(300))
        p1 = port.next_pow2(degree) - 1
        assert p1 == ref.next_pow2(degree) - 1
        ka, va = np.full(p1, EMPTY, np.uint32), np.zeros(p1)
        kb, vb = ka.copy(), va.copy()
        probing = int(rng.integers(4))
        for _ in range(int(rng.integers(degree + 2))):
            k = int(rng.integers(1 << 20))
            v = float(rng.integers(1, 64))
            if (ka != EMPTY).sum() >= degree and k not in set(ka.tolist()):
                continue
            assert port.ht_accumulate(ka, va, probing, k, v) == ref.ht_accumulate(kb, vb, probing, k, v)
        assert (ka == kb).all() and (va == vb).all()
        assert port.ht_max(ka, va) == ref.ht_max(kb, vb)
