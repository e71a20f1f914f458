"""Diagnostic: host-input (e2e) run breakdown for a config."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2501_19004_b200 as lvn
from bench import CONFIGS

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
n, arcs = dg.num_vertices(), dg.num_arcs()
host = dg.download(np.empty(n + 1, np.uint64), torch.empty(arcs, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32),
                   torch.empty(arcs, dtype=torch.float32, pin_memory=True).numpy())
off_pinned = torch.empty(n + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
off_pinned[:] = host.offsets
hg = lvn.CsrGraph(off_pinned, host.targets, host.weights, host.total_weight)
for i in range(4):
    t0 = time.time()
    r = lvn.louvain_compact(hg)
    print(f"wall {time.time() - t0:.3f} engine {r.wall_seconds:.3f} h2d {r.h2d_seconds:.3f} d2h {r.d2h_seconds:.3f} "
          f"move {r.phase.local_moving:.3f} agg {r.phase.aggregation:.3f} other {r.phase.other:.3f}", flush=True)
for i in range(2):
    t0 = time.time()
    r = lvn.louvain_compact(dg, membership_on_device=True)
    print(f"device wall {time.time() - t0:.3f} engine {r.wall_seconds:.3f}", flush=True)
