import sys; sys.path.insert(0,'.')
import paper_2501_19004_b200 as lvn
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 16
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dg = lvn.generate("rmat", scale=scale, edgefactor=16, seed=1)
print("generated", dg.num_vertices(), dg.num_arcs(), flush=True)
for i in range(reps):
    r = lvn.louvain_compact(dg)
    print("ok", r.modularity, r.passes, r.iterations_per_pass, flush=True)
