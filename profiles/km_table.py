"""Summarise a kernel_metrics.sh CSV: one row per launch (or aggregated per kernel)."""
import csv, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; rows = rows[1:]
I = {k: h.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value")}
L = collections.OrderedDict()
for r in rows:
    key = (r[I["ID"]], r[I["Kernel Name"]].split("(")[0].replace("void ", "").replace("lvn::<unnamed>::", ""))
    L.setdefault(key, {})[r[I["Metric Name"]]] = float(r[I["Metric Value"]].replace(",", "") or 0)
short = {"gpu__time_duration.sum": "us", "smsp__inst_executed.sum": "Minst", "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
         "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%", "dram__bytes_read.sum": "rdMB", "dram__bytes_write.sum": "wrMB",
         "lts__t_sector_hit_rate.pct": "L2hit", "launch__registers_per_thread": "regs", "launch__grid_size": "grid",
         "smsp__thread_inst_executed_per_inst_executed.ratio": "thr/inst"}
stall = lambda k: k.split("stalled_")[1].split("_per")[0] if "stalled_" in k else None
agg = "--agg" in sys.argv
if agg:
    A = collections.OrderedDict()
    for (i, k), m in L.items():
        a = A.setdefault(k, collections.Counter()); a["n"] += 1
        t = m.get("gpu__time_duration.sum", 0)
        for mk, v in m.items():
            a[mk] += v * (t if ("pct" in mk or "ratio" in mk or "regs" in mk) else 1)
        a["_t"] += t
    tot = sum(a["_t"] for a in A.values())
    print(f"{'kernel':34s} {'n':>3s} {'ms':>8s} {'share':>6s} {'Minst':>8s} {'issue%':>6s} {'occ%':>5s} {'L2hit':>5s} {'GB/s':>7s}  top stalls (warps per issue)")
    for k, a in sorted(A.items(), key=lambda x: -x[1]["_t"]):
        t = a["_t"]; w = lambda mk: a[mk] / t if t else 0
        st = sorted(((stall(mk), w(mk)) for mk in a if stall(mk)), key=lambda x: -x[1])[:3]
        gbs = (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / t if t else 0
        print(f"{k[:34]:34s} {a["n"]:3d} {t/1e6:8.3f} {100*t/tot:5.1f}% {a['smsp__inst_executed.sum']/1e6:8.1f} {w('smsp__issue_active.avg.pct_of_peak_sustained_active'):6.1f} "
              f"{w('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f} {w('lts__t_sector_hit_rate.pct'):5.1f} {gbs:7.0f}  " + ", ".join(f"{s}={v:.1f}" for s, v in st))
else:
    for (i, k), m in L.items():
        st = sorted(((stall(mk), v) for mk, v in m.items() if stall(mk)), key=lambda x: -x[1])[:3]
        print(i, k[:30], " ".join(f"{short[mk]}={v:.4g}" for mk, v in m.items() if mk in short), "|", ", ".join(f"{s}={v:.1f}" for s, v in st))
