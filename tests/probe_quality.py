"""Quality probe (run by hand on the GPU box): GPU modularity vs the reference
engines for several sweep_chunk settings."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import golden_data as G  # noqa: E402
import paper_2501_19004_b200 as lvn  # noqa: E402
from graphs import planted, random_graph, rmat  # noqa: E402
from oracle import port, ref, ref_available  # noqa: E402

cases = [(f"pp{t}", G.graph(f"pp{t}_")) for t in range(4)]
cases += [("rnd4000", random_graph(4000, 24000, 7, 1.0, 6.0, False, True)), ("rmat16", rmat(16, 16, 1)),
          ("planted200k", planted(200000, 200, 32, 0.1, 5))]
chunks = [int(x) for x in sys.argv[1:]] or [0xFFFFFFFF, 65536, 8192, 2048, 512, 128, 32]
for name, g in cases:
    t0 = time.time()
    seq = port.sequential_louvain(g).modularity
    mc = ref.louvain(g, "mc", thread_count=16).modularity if ref_available() else float("nan")
    cp = ref.louvain(g, "compact", thread_count=16).modularity if ref_available() else float("nan")
    row = [f"{name:12s} n={g.n:7d} seq={seq:.4f} mc16={mc:.4f} compact16={cp:.4f} |"]
    dg = lvn.CsrGraph(g.offsets, g.targets, g.weights, g.total_weight)
    for c in chunks:
        qs = [lvn.louvain_compact(dg, None, lvn.CompactOptions(sweep_chunk=c)).modularity for _ in range(3)]
        row.append(f"{c}:{np.mean(qs):.4f}")
    print(" ".join(row), f"({time.time() - t0:.1f}s)", flush=True)
