"""Reference engines' pass structure on a config (tuning aid)."""
import sys, os
sys.path.insert(0, '.')
import numpy as np
import paper_2501_19004_b200 as lvn
from bench import CONFIGS
from oracle import Csr, ref
cfg = sys.argv[1]
c = CONFIGS[cfg]
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
g = dg.download()
r = lvn.louvain_compact(dg)
sizes = np.bincount(r.membership)
print("gpu", round(r.modularity, 5), r.passes, r.iterations_per_pass, "V/pass", r.vertices_per_pass, "communities", r.num_communities,
      "largest", sorted(sizes)[-5:], flush=True)
h = ref.handle(Csr(g.offsets, g.targets, g.weights, g.total_weight))
for eng in sys.argv[2:] or ["mc"]:
    x = ref.louvain(h, eng, thread_count=os.cpu_count())
    sizes = np.bincount(x.membership)
    print(eng, round(x.modularity, 5), x.passes, x.iterations_per_pass, "communities", x.num_communities,
          "largest", sorted(sizes)[-5:], "tol", x.tolerance_per_pass, flush=True)
