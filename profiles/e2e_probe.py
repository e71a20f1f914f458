"""End-to-end (host input) timing of one config through the public API, with
the input in pinned host memory as bench.py's e2e leg has it: per run wall
time, upload time and bytes, per-phase device time; optional CompactOptions
overrides (key=value). python profiles/e2e_probe.py c5 [runs] [key=value ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2501_19004_b200 as lvn
from bench import CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 3
over = dict(a.split("=") for a in sys.argv[3:])
opts = lvn.CompactOptions(**{k: int(v) for k, v in over.items()})
c = CONFIGS[cfg]
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
n, arcs = dg.num_vertices(), dg.num_arcs()
off = torch.empty(n + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
tgt = torch.empty(arcs, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
w = torch.empty(arcs, dtype=torch.float32, pin_memory=True).numpy()
h = dg.download(off, tgt, w)
dg.close()
for i in range(runs + 1):
    r = lvn.louvain_compact(h, None, opts)
    print(cfg, i, "wall_ms", round(r.wall_seconds * 1e3, 1), "h2d_ms", round(r.h2d_seconds * 1e3, 1),
          "h2d_GB", round(r.h2d_bytes / 1e9, 2), {k: round(s.seconds * 1e3, 1) for k, s in r.stats.items()},
          "pass_ms", [round(x * 1e3, 1) for x in r.pass_seconds], "Q", round(r.modularity, 5), flush=True)
