"""Per-run breakdown of repeated Louvain runs on one config (step-time
variance study): wall, summed device time per kernel family, host remainder."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_19004_b200 as lvn
from bench import CONFIGS

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 8
c = CONFIGS[cfg]
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
for i in range(runs):
    r = lvn.louvain_compact(dg, membership_on_device=True)
    ks = {k: round(s.seconds * 1e3, 1) for k, s in r.stats.items()}
    tot = sum(s.seconds for s in r.stats.values()) * 1e3
    print(cfg, i, "wall", round(r.wall_seconds * 1e3, 1), "kernels", round(tot, 1), "host", round(r.wall_seconds * 1e3 - tot, 1),
          ks, "passes", [round(x * 1e3, 1) for x in r.pass_seconds], "Q", round(r.modularity, 5), flush=True)
