"""Parity of the CUDA path (through the C-ABI) against the oracle on the same
inputs. Bars (BASELINE.json north_star): renumbering, community CSR and
canonical aggregation bit-exact (integer weights); modularity within 1e-9
relative; per-vertex decisions bit-exact on a fixed snapshot (integer weights
make fp32/fp64 accumulation exact); end-to-end modularity within 0.005 of the
reference's."""

import numpy as np
import pytest

import golden_data as G
from graphs import (BARBELL, LOW_SHRINK, SINGLE_EDGE, SWAP_GADGET, TRIANGLE, TWO_TRIANGLES, canonical_rows,
                    from_triples, planted, random_graph, random_membership, rmat)

pytestmark = pytest.mark.gpu

MOD_RTOL = 1e-9
Q_TOL = 0.005


@pytest.fixture(scope="module")
def lvn():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2501_19004_b200 as m

    return m


def G_(g, lvn):
    return lvn.CsrGraph(g.offsets, g.targets, g.weights, g.total_weight)


def assert_q(a, b):
    assert abs(a - b) <= MOD_RTOL * max(1.0, abs(b)), (a, b)


def star(n_leaves):
    """hub 0 joined to every leaf: a row longer than every smem table"""
    src = np.zeros(n_leaves, np.uint32)
    dst = np.arange(1, n_leaves + 1, dtype=np.uint32)
    from oracle import port

    return port.build_csr(n_leaves + 1, src, dst, np.ones(n_leaves))


# ---------------------------------------------------------------- modularity
def test_modularity_anchors(lvn):
    assert abs(lvn.modularity(G_(from_triples((3, [(0, 1, 1.0), (1, 2, 2.0), (2, 2, 4.0)])), lvn), [0, 0, 0])) <= 1e-12
    assert_q(lvn.modularity(G_(from_triples(TRIANGLE), lvn), [0, 1, 2]), -1 / 3)
    assert_q(lvn.modularity(G_(from_triples(BARBELL), lvn), [0, 0, 0, 1, 1, 1]), 5 / 14)
    assert_q(lvn.modularity(G_(from_triples(SINGLE_EDGE), lvn), [0, 1]), -0.5)
    with pytest.raises(lvn.DegenerateGraphError):
        lvn.modularity(G_(from_triples((2, [])), lvn), [0, 1])


@pytest.mark.parametrize("t", range(12))
def test_modularity_golden(lvn, t):
    p = f"rnd{t}_"
    g = G.graph(p)
    assert_q(lvn.modularity(G_(g, lvn), G.field(p, "membership")), float(G.field(p, "modularity")))
    assert np.allclose(lvn.vertex_weights(G_(g, lvn)), G.field(p, "vertex_weights"), rtol=1e-12, atol=0)


@pytest.mark.parametrize("seed", range(4))
def test_modularity_random_labels(lvn, port, seed):
    g = random_graph(3000, 20000, seed, 0.25, 7.5, True, False)
    memb = np.random.default_rng(seed).integers(0, 1 + 97 * seed, g.n).astype(np.uint32) * 7 + 1000
    assert_q(lvn.modularity(G_(g, lvn), memb), port.modularity(g, memb))


def test_modularity_hub_rows(lvn, port):
    g = star(20000)
    memb = random_membership(g.n, 50, 3)
    assert_q(lvn.modularity(G_(g, lvn), memb), port.modularity(g, memb))


def test_modularity_rmat16(lvn, port):
    g = rmat(16, 16, 1)
    memb = random_membership(g.n, 1000, 1)
    assert_q(lvn.modularity(G_(g, lvn), memb), port.modularity(g, memb))


# ------------------------------------------------------- renumber / lookup / CSR
def test_renumber_lookup_golden(lvn):
    m = np.array([5, 5, 2, 9], np.uint32)
    assert lvn.renumber_communities(m) == 3 and list(m) == [1, 1, 0, 2]
    m = np.array([0, 1, 1, 2], np.uint32)
    lvn.lookup_dendrogram(m, [2, 0, 1])
    assert list(m) == [2, 0, 0, 1]
    with pytest.raises(lvn.InternalError):
        lvn.lookup_dendrogram(np.array([0, 5], np.uint32), [2, 0, 1])
    assert lvn.count_communities([5, 5, 2, 9]) == 3
    assert lvn.count_communities(np.array([], np.uint32)) == 0


@pytest.mark.parametrize("n,k", [(1, 1), (1000, 7), (100000, 5000), (2_000_000, 300_000)])
def test_renumber_bit_exact(lvn, port, n, k):
    rng = np.random.default_rng(n)
    m = (rng.integers(0, k, n) * 3 + 11).astype(np.uint32)
    want, wc = port.renumber(m)
    got = m.copy()
    assert lvn.renumber_communities(got) == wc
    assert (got == want).all()
    assert lvn.count_communities(m) == port.count_communities(m)
    level = rng.permutation(wc).astype(np.uint32)
    a = want.copy()
    lvn.lookup_dendrogram(a, level)
    assert (a == port.lookup(want, level)).all()


@pytest.mark.parametrize("n,k", [(10, 3), (50000, 40), (300000, 30000), (20000, 1)])
def test_community_csr_bit_exact(lvn, port, n, k):
    m = random_membership(n, k, n + k)
    count = port.count_communities(m)
    off, mem = lvn.build_community_csr(m, count)
    woff, wmem = port.community_csr(m, count)
    assert (off == woff).all() and (mem == wmem).all()


# ---------------------------------------------------------------- aggregation
def agg_equal(a, want):
    assert (a.offsets == want.offsets).all()
    ra, ta, wa = canonical_rows(a)
    rb, tb, wb = canonical_rows(want)
    assert (ta == tb).all() and (wa == wb).all()
    assert (a.targets == ta).all(), "rows must come out canonically sorted"
    assert a.total_weight == want.total_weight


def test_aggregate_barbell_golden(lvn):
    a = lvn.compact_aggregate(G_(from_triples(BARBELL), lvn), [0, 0, 0, 1, 1, 1])
    assert list(a.offsets) == [0, 2, 4] and list(a.targets) == [0, 1, 0, 1]
    assert list(a.weights) == [6.0, 1.0, 1.0, 6.0] and a.total_weight == 7.0
    with pytest.raises(ValueError):
        lvn.compact_aggregate(G_(from_triples(TRIANGLE), lvn), [0, 2, 2])


@pytest.mark.parametrize("t", range(12))
def test_aggregate_golden(lvn, t):
    p = f"rnd{t}_"
    a = lvn.compact_aggregate(G_(G.graph(p), lvn), G.field(p, "membership"))
    assert (a.offsets == G.field(p, "agg_offsets")).all()
    assert (a.targets == G.field(p, "agg_targets")).all()
    assert (a.weights == G.field(p, "agg_weights")).all()
    assert a.total_weight == float(G.field(p, "agg_total_weight"))


@pytest.mark.parametrize("n,edges,k", [(2000, 8000, 3), (5000, 40000, 50), (20000, 100000, 2000),
                                       (100000, 400000, 30000), (4000, 200000, 9)])
def test_aggregate_bit_exact_random(lvn, port, n, edges, k):
    g = random_graph(n, edges, n + k)
    m = random_membership(n, k, k)
    agg_equal(lvn.compact_aggregate(G_(g, lvn), m), port.aggregate(g, m))


def test_aggregate_global_table_path(lvn, port):
    g = star(12000)  # community of the hub has 12000 distinct neighbours > smem table
    m = np.arange(g.n, dtype=np.uint32)
    agg_equal(lvn.compact_aggregate(G_(g, lvn), m), port.aggregate(g, m))
    m2 = random_membership(g.n, 9000, 5)
    agg_equal(lvn.compact_aggregate(G_(g, lvn), m2), port.aggregate(g, m2))


def hubs_graph(n, hubs, hub_deg, extra, seed):
    """`hubs` vertices with hub_deg random neighbours each (several 4096-arc
    chunks per hub) over a sparse random background of `extra` edges"""
    rng = np.random.default_rng(seed)
    src = [np.repeat(np.arange(hubs, dtype=np.uint32), hub_deg)]
    dst = [rng.integers(hubs, n, hubs * hub_deg).astype(np.uint32)]
    src.append(rng.integers(0, n, extra).astype(np.uint32))
    dst.append(rng.integers(0, n, extra).astype(np.uint32))
    w = rng.integers(1, 5, hubs * hub_deg + extra).astype(np.float64)
    from oracle import port

    return port.build_csr(n, np.concatenate(src), np.concatenate(dst), w)


@pytest.mark.parametrize("k_big", [1, 3, 17])
def test_aggregate_member_parallel(lvn, port, k_big):
    # communities whose member-degree budget exceeds block_max (4096) take the
    # member-parallel HBM-table path; mixed with small ones in the same call
    g = random_graph(40000, 400000, 90 + k_big)
    m = random_membership(g.n, 3000, k_big).astype(np.int64)
    m[: 24000] = np.arange(24000) % k_big  # k_big giant communities
    m = np.unique(m, return_inverse=True)[1].astype(np.uint32)
    agg_equal(lvn.compact_aggregate(G_(g, lvn), m), port.aggregate(g, m))


def test_aggregate_member_parallel_batched(lvn, port, monkeypatch):
    # a tiny table budget forces one batch per giant community
    monkeypatch.setenv("LVN_BIG_TABLE_BUDGET", "1")
    g = random_graph(40000, 400000, 93)
    m = random_membership(g.n, 3000, 7).astype(np.int64)
    m[: 24000] = np.arange(24000) % 5
    m = np.unique(m, return_inverse=True)[1].astype(np.uint32)
    agg_equal(lvn.compact_aggregate(G_(g, lvn), m), port.aggregate(g, m))


@pytest.mark.parametrize("mode", ["hash", "dense"])
def test_aggregate_member_parallel_modes(lvn, port, monkeypatch, mode):
    # giant-community regions: 16-byte-slot hash tables or dense fp64 arrays
    monkeypatch.setenv("LVN_BIG_MODE", mode)
    g = hubs_graph(30000, 4, 20000, 100000, 6)
    for m in ((np.arange(g.n) % 2).astype(np.uint32), random_membership(g.n, 50, 4)):
        agg_equal(lvn.compact_aggregate(G_(g, lvn), m), port.aggregate(g, m))
    g = random_graph(40000, 400000, 95)
    m = random_membership(g.n, 3000, 9).astype(np.int64)
    m[: 24000] = np.arange(24000) % 3
    m = np.unique(m, return_inverse=True)[1].astype(np.uint32)
    agg_equal(lvn.compact_aggregate(G_(g, lvn), m), port.aggregate(g, m))


def test_aggregate_member_parallel_hubs(lvn, port):
    g = hubs_graph(30000, 4, 20000, 100000, 5)
    for m in (np.zeros(g.n, np.uint32), (np.arange(g.n) % 2).astype(np.uint32),
              random_membership(g.n, 50, 4)):
        agg_equal(lvn.compact_aggregate(G_(g, lvn), m), port.aggregate(g, m))


def test_aggregate_planted(lvn, port):
    g = planted(50000, 100, 32, 0.1, 9)
    m = (np.arange(g.n) // 500).astype(np.uint32)
    agg_equal(lvn.compact_aggregate(G_(g, lvn), m), port.aggregate(g, m))


# ------------------------------------------------------------ move decisions
def decisions_equal(lvn, port, g, memb, force=-1, value_bits=64, live=False, probing=None):
    kw = port.vertex_weights(g)
    cw = np.zeros(g.n)
    np.add.at(cw, memb, kw)
    opts = lvn.CompactOptions(value_bits=value_bits)
    if probing is not None:
        opts.probing = probing
    to, gain = lvn.evaluate_moves(G_(g, lvn), memb, kw, cw, g.total_weight, opts, force, live)
    for u in range(g.n):
        want = port.evaluate_move(g, memb, kw, cw, g.total_weight, u, value_bits)
        assert (int(to[u]), float(gain[u])) == want, (u, g.offsets[u + 1] - g.offsets[u])


@pytest.mark.parametrize("t", range(12))
def test_decisions_golden(lvn, t):
    p = f"rnd{t}_"
    g = G.graph(p)
    memb = G.field(p, "membership")
    kw = G.field(p, "vertex_weights")
    cw = np.zeros(g.n)
    np.add.at(cw, memb, kw)
    # the fixtures are compact_evaluate_move<double> (value_bits 64)
    to, gain = lvn.evaluate_moves(G_(g, lvn), memb, kw, cw, g.total_weight, lvn.CompactOptions(value_bits=64))
    assert (to == G.field(p, "move_to")).all() and (gain == G.field(p, "move_gain")).all()


@pytest.mark.parametrize("force", [-1, 1, 2, 3, 4])
@pytest.mark.parametrize("value_bits", [32, 64])
def test_decisions_every_kernel_class(lvn, port, force, value_bits):
    # integer weights keep fp32 and fp64 accumulation exact, so every kernel
    # class must decide bit-identically (test_compact.cpp:114-144)
    g = random_graph(600, 6000, 11 + force, 1.0, 6.0, True, True)
    memb = random_membership(g.n, 40, 3)
    decisions_equal(lvn, port, g, memb, force, value_bits)


@pytest.mark.parametrize("force", [-1, 1, 2, 3, 4])
@pytest.mark.parametrize("value_bits", [32, 64])
@pytest.mark.parametrize("unit", [True, False])
def test_live_decisions_every_kernel_class(lvn, port, force, value_bits, unit):
    # the engine's own ranking path (lvn_probe_moves: reciprocal Eq. 2,
    # may_gain pruning, community-only keys on unit weights) must pick what
    # compact_evaluate_move picks, with the reference's exact gain
    g = random_graph(600, 6000, 31 + force, 1.0, 1.0 if unit else 6.0, True, True)
    for k in (40, 300):
        memb = random_membership(g.n, k, 5 + k)
        decisions_equal(lvn, port, g, memb, force, value_bits, live=True)


@pytest.mark.parametrize("value_bits", [32, 64])
def test_live_decisions_hubs_and_planted(lvn, port, value_bits):
    g = hubs_graph(25000, 5, 20000, 60000, 3)
    decisions_equal(lvn, port, g, random_membership(g.n, 300, 9), -1, value_bits, live=True)
    g = planted(20000, 50, 24, 0.1, 4)  # unit weights: community-only keys
    decisions_equal(lvn, port, g, (np.arange(g.n) // 400).astype(np.uint32), -1, value_bits, live=True)
    decisions_equal(lvn, port, g, np.arange(g.n, dtype=np.uint32), -1, value_bits, live=True)


def test_decisions_hub(lvn, port):
    g = star(9000)
    memb = random_membership(g.n, 700, 8)
    decisions_equal(lvn, port, g, memb)


@pytest.mark.parametrize("value_bits", [32, 64])
@pytest.mark.parametrize("k", [30, 3000])
def test_decisions_chunked_hubs(lvn, port, value_bits, k):
    # 5 hubs of 20000 arcs: 5 chunks of 4096 arcs each, merged in HBM tables
    g = hubs_graph(25000, 5, 20000, 60000, k)
    memb = random_membership(g.n, k, 9)
    decisions_equal(lvn, port, g, memb, -1, value_bits)


def test_engine_chunked_hubs(lvn, port):
    g = hubs_graph(60000, 8, 30000, 400000, 2)
    r = lvn.louvain_compact(G_(g, lvn))
    assert_q(r.modularity, port.modularity(g, np.asarray(r.membership, np.uint32)))
    assert r.modularity > 0.0


@pytest.mark.parametrize("opts", [dict(sweep_ranges=4), dict(sweep_ranges=16), dict(sweep_order=1),
                                  dict(singleton_rule=True), dict(sweep_chunk=1024), dict(value_bits=64),
                                  dict(sweep_ranges=4, sweep_order=1)])
def test_engine_sweep_options(lvn, port, opts):
    # every sweep-order knob over a multi-pass run (hubs, block rows and sort
    # bins in every range): Q recomputed by the oracle, contiguous ids, quality
    # within the reference gate of the default sweep
    g = hubs_graph(60000, 8, 30000, 400000, 2)
    base = lvn.louvain_compact(G_(g, lvn)).modularity
    r = lvn.louvain_compact(G_(g, lvn), None, lvn.CompactOptions(**opts))
    m = np.asarray(r.membership, np.uint32)
    assert_q(r.modularity, port.modularity(g, m))
    assert set(np.unique(m)) == set(range(r.num_communities)) and r.passes >= 2
    assert r.modularity >= base - 0.01


@pytest.mark.parametrize("probing", ["linear", "quadratic", "double_hash", "quadratic_double"])
def test_probing_modes_change_speed_not_results(lvn, port, probing):
    # the reference's four probing recurrences (compact_hashtable.hpp:60-82)
    # drive every device table: smem tables of the warp / block classes, the
    # hubs' HBM tables, the giant-community regions of aggregation
    mode = lvn.Probing[probing]
    g = hubs_graph(25000, 5, 20000, 60000, 3)
    memb = random_membership(g.n, 400, 9)
    for force in (2, 3, 4):
        decisions_equal(lvn, port, g, memb, force, 32, probing=mode)
    m = random_membership(g.n, 50, 4)
    agg_equal(lvn.compact_aggregate(G_(g, lvn), m, options=lvn.CompactOptions(probing=mode)), port.aggregate(g, m))
    s = star(12000)
    ms = np.arange(s.n, dtype=np.uint32)
    agg_equal(lvn.compact_aggregate(G_(s, lvn), ms, options=lvn.CompactOptions(probing=mode)), port.aggregate(s, ms))
    r = lvn.louvain_compact(G_(g, lvn), None, lvn.CompactOptions(probing=mode))
    assert_q(r.modularity, port.modularity(g, np.asarray(r.membership, np.uint32)))


# ------------------------------------------------------------ engine end to end
def test_engine_fixture_optima(lvn):
    r = lvn.louvain_compact(G_(from_triples(TWO_TRIANGLES), lvn))
    assert abs(r.modularity - 0.5) <= 1e-9 and r.num_communities == 2
    r = lvn.louvain_compact(G_(from_triples(BARBELL), lvn))
    assert abs(r.modularity - 5 / 14) <= 1e-9 and r.num_communities == 2
    r = lvn.louvain_compact(G_(from_triples(SINGLE_EDGE), lvn))
    assert r.num_communities == 1 and abs(r.modularity) <= 1e-12
    r = lvn.louvain_compact(G_(from_triples(TRIANGLE), lvn))
    assert r.num_communities == 1


def test_engine_params_and_errors(lvn):
    g = G_(from_triples(BARBELL), lvn)
    r = lvn.louvain_compact(g, lvn.LouvainParams(max_passes=0))
    assert r.passes == 0 and r.num_communities == 6 and list(r.membership) == list(range(6))
    r = lvn.louvain_compact(g, lvn.LouvainParams(max_iterations=0))
    assert r.passes == 1 and r.num_communities == 6
    for bad in (lvn.LouvainParams(max_passes=-1), lvn.LouvainParams(tolerance_drop=0.0),
                lvn.LouvainParams(aggregation_tolerance=0.0), lvn.LouvainParams(chunk_size=0)):
        with pytest.raises(ValueError):
            lvn.louvain_compact(g, bad)
    with pytest.raises(ValueError):
        lvn.louvain_compact(g, None, lvn.CompactOptions(pick_less=lvn.PickLessSchedule(3)))
    with pytest.raises(ValueError):
        lvn.louvain_compact(g, None, lvn.CompactOptions(value_bits=16))
    with pytest.raises(lvn.DegenerateGraphError):
        lvn.louvain_compact(G_(from_triples((3, [])), lvn))


def test_engine_low_shrink(lvn):
    r = lvn.louvain_compact(G_(from_triples(LOW_SHRINK), lvn))
    assert r.aggregations == 0 and r.passes == 1 and r.num_communities == 9
    assert r.membership[8] == r.membership[9]


def test_engine_swap_gadget(lvn, port):
    g = from_triples(SWAP_GADGET)
    r = lvn.louvain_compact(G_(g, lvn))
    assert r.membership[3] == r.membership[5]
    assert_q(r.modularity, port.modularity(g, r.membership))


def test_engine_tolerance_schedule_and_bookkeeping(lvn, port):
    g = planted(3000, 30, 24, 0.05, 77)
    r = lvn.louvain_compact(G_(g, lvn))
    assert r.passes >= 2 and r.aggregations <= r.passes
    for p, t in enumerate(r.tolerance_per_pass):
        assert t == pytest.approx(0.01 / 10**p, rel=1e-12)
    assert len(r.pass_seconds) == r.passes and len(r.iterations_per_pass) == r.passes
    assert r.phase.total() == pytest.approx(r.wall_seconds, rel=1e-9)
    m = r.membership.copy()
    assert port.count_communities(m) == r.num_communities == int(m.max()) + 1
    assert_q(r.modularity, port.modularity(g, r.membership))


@pytest.mark.parametrize("t", range(4))
def test_engine_quality_vs_reference_planted(lvn, t):
    p = f"pp{t}_"
    g = G.graph(p)
    r = lvn.louvain_compact(G_(g, lvn))
    assert r.modularity >= float(G.field(p, "seq_modularity")) - Q_TOL
    assert r.modularity >= float(G.field(p, "mc_modularity")) - Q_TOL


@pytest.mark.parametrize("value_bits", [32, 64])
def test_engine_quality_rmat16_c1(lvn, port, ref, value_bits):
    # config C1: RMAT scale 16, edge factor 16, dedupe, default parameters, against
    # the reference engines run on all host cores (5-run means, like the CPU
    # baseline). The engine re-implements louvain_compact (ν-Louvain), the entry
    # point it replaces, so that is the two-sided 0.005 gate; louvain_mc
    # (GVE-Louvain) sweeps in vertex-id order and finds ~0.005 more on this
    # skewed graph (the reference's own louvain_compact shows the same gap, and
    # the paper reports ν-Louvain below GVE-Louvain; DESIGN.md,
    # "quality"), so against it the gate is one-sided at 0.006.
    g = rmat(16, 16, 1)
    compact = float(np.mean([ref.louvain(g, "compact").modularity for _ in range(5)]))
    mc = float(np.mean([ref.louvain(g, "mc").modularity for _ in range(5)]))
    opts = lvn.CompactOptions(value_bits=value_bits)
    runs = [lvn.louvain_compact(G_(g, lvn), None, opts) for _ in range(5)]
    for r in runs:
        assert_q(r.modularity, port.modularity(g, r.membership))
    q = float(np.mean([r.modularity for r in runs]))
    assert abs(q - compact) <= Q_TOL, (q, compact)
    assert q >= mc - 0.006, (q, mc)


def test_engine_quality_planted_large(lvn, port):
    g = planted(200000, 200, 32, 0.1, 5)
    truth = (np.arange(g.n) // (g.n // 200)).astype(np.uint32)
    r = lvn.louvain_compact(G_(g, lvn))
    assert_q(r.modularity, port.modularity(g, r.membership))
    assert r.modularity >= port.modularity(g, truth) - Q_TOL


def test_engine_device_resident_input(lvn, port):
    g = rmat(14, 16, 2)
    dg = lvn.DeviceGraph.upload(G_(g, lvn))
    r = lvn.louvain_compact(dg)
    assert_q(r.modularity, port.modularity(g, r.membership))
    r2 = lvn.louvain_compact(dg, membership_on_device=True)
    assert r2.membership_device_ptr and r2.num_communities > 0


# ----------------------------------------------------------------- generators
@pytest.mark.parametrize("kind,kw", [("rmat", dict(scale=12, edgefactor=16)),
                                     ("sbm", dict(n=20000, blocks=20, avg_degree=16, mu=0.1)),
                                     ("grid", dict(side=60, p=0.6)),
                                     ("uniform", dict(n=5000, edges=20000)),
                                     ("web", dict(n=20000, avg_degree=20))])
def test_generators_produce_valid_csr(lvn, kind, kw):
    dg = lvn.generate(kind, seed=3, **kw)
    g = dg.download()
    n = g.num_vertices()
    rows = np.repeat(np.arange(n), np.diff(g.offsets.astype(np.int64)))
    assert (np.diff(g.offsets.astype(np.int64)) >= 0).all()
    assert (g.targets < n).all() and (g.weights == 1.0).all()
    assert not (rows == g.targets).any(), "self-loops"
    key = rows.astype(np.uint64) << np.uint64(32) | g.targets.astype(np.uint64)
    assert (np.diff(key.astype(np.int64)) > 0).all(), "rows sorted and deduplicated"
    rev = g.targets.astype(np.uint64) << np.uint64(32) | rows.astype(np.uint64)
    assert np.array_equal(np.sort(rev), key), "symmetric"
    assert g.total_weight == g.num_arcs() / 2


# ---------------------------------------------------------------- dendrogram
def test_dendrogram_levels(lvn, port):
    # keep_levels: one local membership per pass; composing them in order
    # (lookup_dendrogram, louvain_mc.cpp:145-160) gives the final partition
    g = planted(20000, 40, 24, 0.2, 12)
    r = lvn.louvain_compact(G_(g, lvn), keep_levels=True)
    assert len(r.levels) == r.passes >= 2
    assert [len(l) for l in r.levels] == r.vertices_per_pass
    glob = np.arange(g.n)
    for k, lvl in enumerate(r.levels):
        glob = lvl[glob]
        if k + 1 < len(r.levels):  # aggregated levels are renumbered to the next graph
            assert lvl.max() + 1 == r.vertices_per_pass[k + 1]
    a, b = glob, r.membership
    pairs = set(zip(a.tolist(), b.tolist()))
    assert len(pairs) == len(set(a.tolist())) == len(set(b.tolist())) == r.num_communities
    assert lvn.louvain_compact(G_(g, lvn)).levels == []


def test_uniform_weight_passes(lvn, port):
    # equal arc weights (any value) take community-only sort keys in the first
    # pass; modularity is scale-free, so scaled weights must land where unit
    # weights do, and a single odd weight takes the packed-key path
    g = planted(30000, 60, 24, 0.15, 21)
    r1 = lvn.louvain_compact(G_(g, lvn))
    src, dst = edge_arrays(g)
    g25 = port.build_csr(g.n, src, dst, np.full(len(src), 2.5))
    r25 = lvn.louvain_compact(G_(g25, lvn))
    assert abs(r25.modularity - r1.modularity) < 0.01
    assert_q(r25.modularity, port.modularity(g25, r25.membership))
    w = g.weights.copy()
    w[7] = 3.0
    gx = lvn.CsrGraph(g.offsets, g.targets, w, float(w.astype(np.float64).sum()) / 2)
    rx = lvn.louvain_compact(gx)
    assert rx.modularity > r1.modularity - 0.01


def edge_arrays(g):
    src = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.offsets).astype(np.int64))
    keep = src < g.targets
    return src[keep], g.targets[keep]
