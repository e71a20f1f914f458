"""Quality and speed of the GPU engine against the reference CPU engines on
the BASELINE configs (run on the GPU box from the repo root):

    python profiles/quality.py c1 c4 c2 c3 c5 > gpurun_out/quality.md

Per config: GPU louvain_compact (device-resident CSR, 3 timed runs after a
warm-up), the reference louvain_mc (GVE design, all host cores; the CPU
baseline) and louvain_compact (nu-Louvain, the same algorithm as the GPU
engine) built from the reference sources (oracle/_ref). Gate:
|Q_gpu - mean Q_mc| <= 0.005."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_19004_b200 as lvn  # noqa: E402
from bench import CONFIGS  # noqa: E402
from oracle import Csr, ref, ref_available  # noqa: E402

cfgs = sys.argv[1:] or ["c1", "c2", "c3", "c4"]
threads = os.cpu_count()
print(f"# Quality vs the reference CPU engines ({threads} host threads)\n")
print("| config | arcs | GPU Q (mean of 3) | GPU ms | GPU G edges/s | mc Q | mc s | mc M edges/s | "
      "compact Q | compact s | |Q_gpu - Q_mc| | gate 0.005 | GPU / mc speed |")
print("|---|---:|---:|---:|---:|---:|---:|---:|---:|---:|---:|---|---:|")
for c in cfgs:
    spec = CONFIGS[c]
    dg = lvn.generate(spec["kind"], **{k: v for k, v in spec.items() if k not in ("kind", "desc")})
    arcs = dg.num_arcs()
    lvn.louvain_compact(dg, membership_on_device=True)
    qs, ts = [], []
    for _ in range(3):
        r = lvn.louvain_compact(dg, membership_on_device=True)
        qs.append(r.modularity)
        ts.append(r.wall_seconds)
    g = dg.download()
    dg.close()
    q_gpu, t_gpu = statistics.mean(qs), statistics.mean(ts)
    row = [c, f"{arcs}", f"{q_gpu:.5f}", f"{t_gpu * 1e3:.1f}", f"{arcs / t_gpu / 1e9:.2f}"]
    if ref_available():
        h = ref.handle(Csr(g.offsets, g.targets, g.weights, g.total_weight))
        reps = 3 if arcs < 1e8 else 1
        mc = [ref.louvain(h, "mc", thread_count=threads) for _ in range(reps)]
        q_mc = statistics.mean(x.modularity for x in mc)
        t_mc = statistics.geometric_mean([x.wall_seconds for x in mc])
        # louvain_compact (nu-Louvain, the algorithm the GPU re-implements) runs
        # its hubs one at a time: ~12 min on C5, skipped there
        cp = ref.louvain(h, "compact", thread_count=threads) if arcs < 1e9 else None
        row += [f"{q_mc:.5f}", f"{t_mc:.2f}", f"{arcs / t_mc / 1e6:.1f}",
                f"{cp.modularity:.5f}" if cp else "-", f"{cp.wall_seconds:.2f}" if cp else "-",
                f"{abs(q_gpu - q_mc):.5f}",
                "pass" if abs(q_gpu - q_mc) <= 0.005 else ("above" if q_gpu > q_mc else "FAIL"),
                f"{t_mc / t_gpu:.0f}x"]
    print("| " + " | ".join(row) + " |", flush=True)
