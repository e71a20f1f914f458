"""Pins the C restatement (oracle/lvn_oracle.c) to the golden values and
known-answer tests the reference's own suites hold for this path
(SURVEY.md 8(c)). CPU only."""

import math

import numpy as np
import pytest

from graphs import BARBELL, LOW_SHRINK, SINGLE_EDGE, TRIANGLE, TWO_TRIANGLES, from_triples

EMPTY = 0xFFFFFFFF


# ---- quality anchors (test_quality.cpp:30-61, 86-89) -------------------------------
def test_modularity_anchors(port):
    g = from_triples((3, [(0, 1, 1.0), (1, 2, 2.0), (2, 2, 4.0)]))
    assert abs(port.modularity(g, [0, 0, 0])) <= 1e-12
    assert port.modularity(from_triples(TRIANGLE), [0, 1, 2]) == pytest.approx(-1 / 3, abs=1e-12)
    assert port.modularity(from_triples(BARBELL), [0, 0, 0, 1, 1, 1]) == pytest.approx(5 / 14, abs=1e-12)
    assert port.modularity(from_triples(SINGLE_EDGE), [0, 1]) == pytest.approx(-0.5, abs=1e-12)


def test_modularity_degenerate(port):
    g = from_triples((2, []))
    with pytest.raises(Exception) as e:
        port.modularity(g, [0, 1])
    assert e.value.code == 2  # DegenerateGraphError


def test_community_aggregates_barbell(port):
    st, si = port.community_aggregates(from_triples(BARBELL), [0, 0, 0, 1, 1, 1])
    assert list(st) == [7.0, 7.0] and list(si) == [6.0, 6.0]


def test_delta_modularity_worked_example(port):
    assert port.delta_modularity(1.0, 0.0, 2.0, 2.0, 2.0, 3.0) == pytest.approx(1 / 9)


def test_count_communities(port):
    assert port.count_communities(np.array([], np.uint32)) == 0
    assert port.count_communities([0, 0, 0]) == 1
    assert port.count_communities([5, 5, 2, 9]) == 3


# ---- renumber / lookup (test_mc.cpp:261-282) -------------------------------------------
def test_renumber_golden(port):
    m, c = port.renumber([5, 5, 2, 9])
    assert c == 3 and list(m) == [1, 1, 0, 2]
    m, c = port.renumber([0, 1, 2])
    assert c == 3 and list(m) == [0, 1, 2]
    m, c = port.renumber(np.array([], np.uint32))
    assert c == 0


def test_lookup_golden(port):
    assert list(port.lookup([0, 1, 1, 2], [2, 0, 1])) == [2, 0, 0, 1]
    with pytest.raises(Exception) as e:
        port.lookup([0, 5], [2, 0, 1])
    assert e.value.code == 3  # InternalError


# ---- aggregation (test_mc.cpp:199-219) -----------------------------------------------
def test_barbell_supergraph_golden(port):
    g = from_triples(BARBELL)
    a = port.aggregate(g, [0, 0, 0, 1, 1, 1])
    assert list(a.offsets) == [0, 2, 4]
    assert list(a.targets) == [0, 1, 0, 1]
    assert list(a.weights) == [6.0, 1.0, 1.0, 6.0]
    assert a.total_weight == g.total_weight


def test_aggregate_identity_on_singletons(port):
    g = from_triples(BARBELL)
    a = port.aggregate(g, list(range(6)))
    assert (a.offsets == g.offsets).all() and (a.targets == g.targets).all()
    assert (a.weights == g.weights).all()


def test_aggregate_rejects_gappy_membership(port):
    with pytest.raises(Exception) as e:
        port.aggregate(from_triples(TRIANGLE), [0, 2, 2])
    assert e.value.code == 1


# ---- hashtable KATs (test_hashtable.cpp:41-132) ----------------------------------------
def test_next_pow2_strictly_greater(port):
    for x, want in [(1, 2), (2, 4), (4, 8), (7, 8), (8, 16), (1023, 1024)]:
        assert port.next_pow2(x) == want
    with pytest.raises(Exception) as e:
        port.next_pow2(1 << 63)
    assert e.value.code == 4


def test_capacity_pairs_coprime(port):
    d = 1
    while d <= 1 << 16:
        p1 = port.next_pow2(d) - 1
        assert math.gcd(p1, 2 * p1 + 1) == 1
        d = 2 * d + 1


def test_probe_chain_worked_example(port):
    keys = np.full(7, EMPTY, np.uint32)
    vals = np.zeros(7)
    assert port.ht_accumulate(keys, vals, "quadratic_double", 10, 1.0)
    assert keys[3] == 10 and vals[3] == 1.0
    assert port.ht_accumulate(keys, vals, "quadratic_double", 17, 5.0)
    assert keys[4] == 17
    assert port.ht_accumulate(keys, vals, "quadratic_double", 24, 7.0)
    assert keys[1] == 24


def test_exhaustion_returns_false(port):
    keys = np.full(3, 999, np.uint32)
    vals = np.zeros(3)
    assert not port.ht_accumulate(keys, vals, "quadratic_double", 5, 1.0)
    assert not port.ht_accumulate(keys, vals, "linear", 5, 1.0)


def test_max_tie_lowest_key(port):
    keys = np.full(7, EMPTY, np.uint32)
    vals = np.zeros(7)
    assert port.ht_max(keys, vals) == (EMPTY, 0.0)
    port.ht_accumulate(keys, vals, "quadratic_double", 2, 1.5)
    port.ht_accumulate(keys, vals, "quadratic_double", 5, 1.5)
    port.ht_accumulate(keys, vals, "quadratic_double", 6, 0.5)
    assert port.ht_max(keys, vals) == (2, 1.5)


def test_hashtable_fuzz_matches_map(port):
    rng = np.random.default_rng(20240817)
    for _ in range(300):
        degree = 1 + int(rng.integers(512))
        p1 = port.next_pow2(degree) - 1
        keys = np.full(p1, EMPTY, np.uint32)
        vals = np.zeros(p1)
        probing = int(rng.integers(4))
        expect = {}
        for _ in range(int(rng.integers(2 * degree + 2))):
            k = int(rng.integers(1 << 31))
            if len(expect) >= degree and k not in expect:
                k = min(expect)
            v = float(1 + rng.integers(100))
            assert port.ht_accumulate(keys, vals, probing, k, v)
            expect[k] = expect.get(k, 0.0) + v
        live = {int(k): float(v) for k, v in zip(keys, vals) if k != EMPTY}
        assert live == expect
        for k, v in expect.items():
            assert port.ht_get(keys, vals, probing, k) == v


# ---- Pick-Less schedule (test_compact.cpp:37-47) ----------------------------------------
def test_pick_less_schedule(port):
    assert [i for i in range(16) if port.pick_less_active(i, 4)] == [2, 6, 10, 14]
    assert [i for i in range(16) if port.pick_less_active(i, 6)] == [3, 9, 15]


# ---- scan (test_prefix.cpp:10-25) ---------------------------------------------------------
def test_exclusive_scan_examples(port):
    assert list(port.exclusive_scan([2, 0, 3])) == [0, 2, 2, 5]
    assert list(port.exclusive_scan([])) == [0]
    assert list(port.exclusive_scan([7])) == [0, 7]


# ---- sequential engine (test_oracle.cpp:65-111, test_mc.cpp:284-376) -------------------------
def test_sequential_fixture_optima(port):
    assert port.sequential_louvain(from_triples(TWO_TRIANGLES)).modularity == pytest.approx(0.5, abs=1e-9)
    r = port.sequential_louvain(from_triples(BARBELL))
    assert r.modularity == pytest.approx(5 / 14, abs=1e-9) and r.num_communities == 2
    assert port.sequential_louvain(from_triples(TRIANGLE)).num_communities == 1
    r = port.sequential_louvain(from_triples(SINGLE_EDGE))
    assert r.num_communities == 1 and abs(r.modularity) <= 1e-12


def test_sequential_max_passes_zero(port):
    r = port.sequential_louvain(from_triples(BARBELL), max_passes=0)
    assert r.passes == 0 and r.num_communities == 6 and list(r.membership) == list(range(6))


def test_sequential_low_shrink(port):
    r = port.sequential_louvain(from_triples(LOW_SHRINK))
    assert r.aggregations == 0 and r.passes == 1 and r.num_communities == 9
    assert r.membership[8] == r.membership[9]


def test_sequential_tolerance_schedule(port):
    from graphs import planted

    r = port.sequential_louvain(planted(300, 6, 20, 0.05, 77))
    assert r.passes >= 2
    for p, t in enumerate(r.tolerance_per_pass):
        assert t == pytest.approx(0.01 / 10**p, rel=1e-12)
