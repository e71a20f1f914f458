"""The C restatement reproduces the reference's own outputs (golden fixtures
generated from oracle/_ref by tests/golden/make_golden.py) bit for bit. CPU only;
needs no reference sources at run time."""

import numpy as np
import pytest

import golden_data as G
from graphs import canonical_rows


@pytest.mark.parametrize("t", range(12))
def test_random_fixture(port, t):
    p = f"rnd{t}_"
    g = G.graph(p)
    memb = G.field(p, "membership")
    assert port.modularity(g, memb) == float(G.field(p, "modularity"))
    assert (port.vertex_weights(g) == G.field(p, "vertex_weights")).all()
    m, c = port.renumber(G.field(p, "raw_membership"))
    assert (m == memb).all() and c == int(G.field(p, "count"))
    a = port.aggregate(g, memb)
    _, tgt, w = canonical_rows(a)
    assert (a.offsets == G.field(p, "agg_offsets")).all()
    assert (tgt == G.field(p, "agg_targets")).all() and (w == G.field(p, "agg_weights")).all()
    assert a.total_weight == float(G.field(p, "agg_total_weight"))
    kw = port.vertex_weights(g)
    cw = np.zeros(g.n)
    np.add.at(cw, memb, kw)
    to, gain = G.field(p, "move_to"), G.field(p, "move_gain")
    for u in range(g.n):
        assert port.evaluate_move(g, memb, kw, cw, g.total_weight, u, 64) == (int(to[u]), float(gain[u]))


@pytest.mark.parametrize("t", range(4))
def test_planted_fixture_sequential(port, t):
    p = f"pp{t}_"
    g = G.graph(p)
    r = port.sequential_louvain(g)
    assert (r.membership == G.field(p, "seq_membership")).all()
    assert r.modularity == float(G.field(p, "seq_modularity"))
    assert r.passes == int(G.field(p, "seq_passes"))
    assert r.iterations_per_pass == list(G.field(p, "seq_iterations"))
