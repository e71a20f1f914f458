"""RMAT-20 quality under engine knobs (tuning aid)."""
import sys
sys.path.insert(0, '.')
import paper_2501_19004_b200 as lvn
kv = dict(a.split("=") for a in sys.argv[1:])
dg = lvn.generate("rmat", scale=int(kv.pop("scale", 20)), edgefactor=16, seed=3)
pf = set(lvn.LouvainParams.__dataclass_fields__)
p = lvn.LouvainParams(**{k: int(v) for k, v in kv.items() if k in pf})
o = lvn.CompactOptions(**{k: int(v) for k, v in kv.items() if k not in pf})
rs = [lvn.louvain_compact(dg, p, o) for _ in range(3)]
print(sys.argv[1:], [round(r.modularity, 5) for r in rs], rs[-1].iterations_per_pass, round(rs[-1].wall_seconds * 1e3, 1), "ms", flush=True)
