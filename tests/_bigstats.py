"""Diagnostic: community budget / distinct-neighbour distribution after pass 0 of a config."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2501_19004_b200 as lvn
from bench import CONFIGS

c = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
r = lvn.louvain_compact(dg, lvn.LouvainParams(max_passes=1))
g = dg.download()
C = torch.from_numpy(np.asarray(r.membership, np.int64)).cuda()
off = torch.from_numpy(g.offsets.astype(np.int64)).cuda()
deg = off[1:] - off[:-1]
n = deg.numel()
k = int(C.max()) + 1
budget = torch.zeros(k, dtype=torch.int64, device="cuda").index_add_(0, C, deg)
big = budget > 4096
print("communities", k, "big", int(big.sum()), "arcs in big", int(budget[big].sum()), "of", int(deg.sum()))
top = torch.topk(budget, 10)
print("top budgets", top.values.tolist())
src = torch.repeat_interleave(torch.arange(n, device="cuda"), deg)
tgt = torch.from_numpy(g.targets.astype(np.int64)).cuda()
cs, ct = C[src], C[tgt]
del src, tgt
m = big[cs]
keys = cs[m] * k + ct[m]
del cs, ct
u = torch.unique(keys)
print("distinct (c,key) pairs in big", u.numel(), "tuples", keys.numel())
uc = torch.bincount(u // k, minlength=k)
print("distinct per top community", uc[top.indices].tolist())
