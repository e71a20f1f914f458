"""GPU vs reference engines on mid-size RMAT graphs (tuning aid)."""
import os, sys, time
sys.path.insert(0, '.')
import paper_2501_19004_b200 as lvn
from oracle import Csr, ref
for scale in [int(x) for x in sys.argv[1:]] or [18, 20]:
    dg = lvn.generate("rmat", scale=scale, edgefactor=16, seed=3)
    g = dg.download()
    qs = [lvn.louvain_compact(dg).modularity for _ in range(3)]
    h = ref.handle(Csr(g.offsets, g.targets, g.weights, g.total_weight))
    out = [f"rmat{scale} arcs={g.num_arcs()} gpu={sum(qs)/3:.5f}"]
    for eng, th in (("mc", 16), ("compact", 16), ("compact", 1), ("sequential", 1)):
        if eng != "mc" and scale > 20:
            continue
        t0 = time.time()
        r = ref.louvain(h, eng, thread_count=th)
        out.append(f"{eng}{th}={r.modularity:.5f} {r.iterations_per_pass} ({time.time()-t0:.1f}s)")
    print(" ".join(out), flush=True)
