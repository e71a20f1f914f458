"""Probe for sporadic slow runs (tuning aid): wall time per run with and without idle gaps."""
import sys, time
sys.path.insert(0, '.')
import paper_2501_19004_b200 as lvn
from bench import CONFIGS
cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
c = CONFIGS[cfg]
dg = lvn.generate(c["kind"], **{k: v for k, v in c.items() if k not in ("kind", "desc")})
for gap in (0.0, 0.2, 1.0):
    ws = []
    for i in range(8):
        if gap: time.sleep(gap)
        t0 = time.perf_counter()
        r = lvn.louvain_compact(dg, membership_on_device=True)
        ws.append((round(r.wall_seconds * 1e3, 1), round((time.perf_counter() - t0) * 1e3, 1),
                   {k: round(s.seconds * 1e3, 1) for k, s in r.stats.items() if s.seconds > 0.0005}))
    print(cfg, "gap", gap, [w[0] for w in ws], flush=True)
    slow = [w for w in ws if w[0] > 1.5 * min(x[0] for x in ws)]
    for w in slow[:3]:
        print("   slow:", w, flush=True)
