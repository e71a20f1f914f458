"""Quality probe (tuning aid): Q and passes under LouvainParams / CompactOptions overrides.
   python tests/_qprobe.py c3 prune=0 initial_tolerance=0.001 ..."""
import sys
sys.path.insert(0, '.')
import paper_2501_19004_b200 as lvn
from bench import CONFIGS
cfg = sys.argv[1]
kv = dict(a.split("=") for a in sys.argv[2:])
c = CONFIGS[cfg]
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
pf = {f for f in lvn.LouvainParams.__dataclass_fields__}
p = lvn.LouvainParams(**{k: type(getattr(lvn.LouvainParams(), k))(float(v) if "." in v else int(v)) for k, v in kv.items() if k in pf})
o = lvn.CompactOptions(**{k: int(v) for k, v in kv.items() if k not in pf})
for i in range(2):
    r = lvn.louvain_compact(dg, p, o, membership_on_device=True)
print(cfg, kv, round(r.modularity, 5), r.passes, r.iterations_per_pass, round(r.wall_seconds * 1e3, 1), "ms", flush=True)
