"""Per-pass quality: GPU vs reference compact/mc with max_passes = 1, 2, 3 (tuning aid)."""
import sys
sys.path.insert(0, '.')
import paper_2501_19004_b200 as lvn
from oracle import Csr, ref
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dg = lvn.generate("rmat", scale=scale, edgefactor=16, seed=3)
g = dg.download()
h = ref.handle(Csr(g.offsets, g.targets, g.weights, g.total_weight))
for mp in (1, 2, 3):
    gq = [lvn.louvain_compact(dg, lvn.LouvainParams(max_passes=mp)) for _ in range(2)]
    row = [f"passes<={mp}: gpu {gq[-1].modularity:.5f} {gq[-1].iterations_per_pass} comms {gq[-1].num_communities}"]
    for eng, th in (("compact", 16), ("compact", 1), ("mc", 16)):
        r = ref.louvain(h, eng, max_passes=mp, thread_count=th)
        row.append(f"{eng}{th} {r.modularity:.5f} {r.iterations_per_pass} comms {r.num_communities}")
    print(" | ".join(row), flush=True)
