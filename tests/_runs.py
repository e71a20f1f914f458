"""Per-run wall times of N consecutive runs (tuning aid)."""
import sys
sys.path.insert(0, '.')
import paper_2501_19004_b200 as lvn
from bench import CONFIGS
cfg, n = sys.argv[1], int(sys.argv[2])
c = CONFIGS[cfg]
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
ws = [round(lvn.louvain_compact(dg, membership_on_device=True).wall_seconds * 1e3, 1) for _ in range(n)]
print(cfg, ws, flush=True)
