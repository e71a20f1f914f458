"""Profiling driver (run under ncu on the GPU box): one warm-up and N runs of a config.
  python profiles/prof_run.py <config | kind:key=value,...> [runs] [option=value ...]
e.g. web:n=10000000,avg_degree=75,seed=5 for a scaled-down C5 shape."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_19004_b200 as lvn
from bench import CONFIGS
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
runs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
# optional CompactOptions overrides: key=value ...
over = dict(a.split("=") for a in sys.argv[3:])
opts = lvn.CompactOptions(**{k: int(v) for k, v in over.items()})
if cfg in CONFIGS:
    c = dict(CONFIGS[cfg])
else:
    kind, _, rest = cfg.partition(":")
    c = {"kind": kind}
    for kv in filter(None, rest.split(",")):
        k, v = kv.split("=")
        c[k] = float(v) if "." in v or k in ("mu", "p", "avg_degree") else int(v)
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
for i in range(runs):
    r = lvn.louvain_compact(dg, None, opts, membership_on_device=True)
    print(cfg, round(r.modularity, 5), r.passes, r.iterations_per_pass, "V", r.vertices_per_pass, "A", r.arcs_per_pass,
          {k: round(s.seconds * 1e3, 2) for k, s in r.stats.items()}, "pass_ms", [round(x * 1e3, 1) for x in r.pass_seconds],
          "move_GBps", round(r.stats["move"].gbps, 1), "move_arcs", r.stats["move"].arcs, "total_ms", round(r.wall_seconds * 1e3, 1), flush=True)
