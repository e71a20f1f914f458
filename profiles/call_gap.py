import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2501_19004_b200 as lvn
from bench import CONFIGS
for cfg in ("c2", "c5"):
    c = CONFIGS[cfg]
    dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
    res = []
    for i in range(6):
        torch.cuda.synchronize()
        t = time.perf_counter()
        r = lvn.louvain_compact(dg, membership_on_device=True)
        dt = time.perf_counter() - t
        res.append(r)
        print(cfg, i, "python", round(dt * 1e3, 1), "engine", round(r.wall_seconds * 1e3, 1), flush=True)
    del res
    dg.close()
