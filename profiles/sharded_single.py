"""The sharded algorithm (lvn_louvain_sharded with the library NCCL
communicator) at world size 1 on a BASELINE config: the per-rank cost of the
sharded machinery (rounds, OR-reduced marks, aggregation by own rows) against
the single-GPU engine on the same graph. python profiles/sharded_single.py c5"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
import torch
import torch.distributed as dist

import paper_2501_19004_b200 as lvn
from bench import CONFIGS
from paper_2501_19004_b200.distributed import NcclComm

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
torch.cuda.set_device(0)
dist.init_process_group("gloo", rank=0, world_size=1)
c = CONFIGS[cfg]
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
comm = NcclComm()
for i in range(3):
    r = lvn.louvain_compact(dg, membership_on_device=True)
    print(cfg, "single ", round(r.wall_seconds * 1e3, 1), "ms Q", round(r.modularity, 5), flush=True)
os.environ["LVN_SHARD_SINGLE"] = "1"
for i in range(3):
    r = lvn.louvain_sharded(dg, comm, options=lvn.CompactOptions(shard_rounds=2), membership_on_device=True)
    print(cfg, "sharded", round(r.wall_seconds * 1e3, 1), "ms Q", round(r.modularity, 5), "sharded passes",
          r.sharded_passes, "exchange", round(r.exchange_seconds * 1e3, 1), "ms",
          {k: round(s.seconds * 1e3, 1) for k, s in r.stats.items()}, flush=True)
comm.close()
dist.destroy_process_group()
