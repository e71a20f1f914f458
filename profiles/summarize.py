"""Turn the raw captures of profiles/collect.sh (gpurun_out/) into the committed
summaries: profiles/<round>_<cfg>.md and the roofline.traffic figure that
bench.py reads from profiles/traffic.json.

    python profiles/summarize.py r02 c5
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
         "s": 1e3, "second": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def rows_of(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    for r in rows:
        if hdr is None:
            if "Kernel Name" in r:
                hdr = r
            continue
        yield dict(zip(hdr, r))


def short(name):
    base = name.split("(")[0]
    return base.replace("lvn::<unnamed>::", "").replace("void ", "")[-60:]


def launch_table(path, top=20):
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in rows_of(path):
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        t = float(d["Metric Value"].replace(",", "")) * SCALE[d["Metric Unit"]]
        agg[short(d["Kernel Name"])][0] += 1
        agg[short(d["Kernel Name"])][1] += t
    total = sum(v[1] for v in agg.values())
    lines = [f"| kernel | launches | ms | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        lines.append(f"| `{k}` | {v[0]} | {v[1]:.3f} | {100 * v[1] / total:.1f}% |")
    move = sum(v[1] for k, v in agg.items() if k.startswith("lm_"))
    return "\n".join(lines), total, move


def move_traffic(path):
    per = collections.defaultdict(dict)
    for d in rows_of(path):
        per[d["ID"]][d["Metric Name"]] = float(d["Metric Value"].replace(",", "")) * SCALE.get(d["Metric Unit"], 1.0)
        per[d["ID"]]["name"] = short(d["Kernel Name"])
    launches = [v for v in per.values() if "dram__bytes_read.sum" in v]
    rd = sum(v["dram__bytes_read.sum"] for v in launches)
    wr = sum(v.get("dram__bytes_write.sum", 0.0) for v in launches)
    t = sum(v.get("gpu__time_duration.sum", 0.0) for v in launches)
    return len(launches), rd, wr, t


def full_capture(rep):
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "smsp__inst_executed.sum", "launch__grid_size"]
    try:
        if rep.endswith(".csv"):
            raw = open(rep).read()
        else:
            raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                                 check=True).stdout
    except Exception as e:  # noqa: BLE001
        return f"(ncu import failed: {e})"
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {w: hdr.index(w) for w in want if w in hdr}
    lines = ["| kernel | " + " | ".join(w.split(".")[0].replace("__", ".") + f" ({units[idx[w]]})" for w in idx) + " |",
             "|---|" + "---:|" * len(idx)]
    for r in rows[2:]:
        lines.append(f"| `{short(r[hdr.index('Kernel Name')])}` | " + " | ".join(r[i] for i in idx.values()) + " |")
    return "\n".join(lines)


def main():
    rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
    cfg = sys.argv[2] if len(sys.argv) > 2 else "c2"
    bench = json.load(open(os.path.join(OUT, f"bench_{cfg}.json")))
    table, total, move = launch_table(os.path.join(OUT, f"launches_{cfg}.csv"))
    n, rd, wr, t = move_traffic(os.path.join(OUT, f"move_traffic_{cfg}.csv"))
    # bench.py's roofline unit is one sweep (every local-moving kernel of one
    # iteration); the traffic run's iteration count is in its log
    sweeps = sum(bench["iterations_per_pass"])
    try:
        line = open(os.path.join(OUT, f"move_traffic_{cfg}.log")).read().split("\n")[0].split()
        sweeps = sum(int(x.strip("[],")) for x in line[line.index("V") - 3:line.index("V")])
    except Exception:  # noqa: BLE001
        pass
    per_launch = (rd + wr) / sweeps if sweeps else None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    traffic[cfg] = per_launch
    traffic[f"{cfg}_note"] = (f"{rnd}: dram read+write bytes per local-moving sweep ({n} lm_* launches "
                              f"over {sweeps} sweeps of one Louvain run, ncu --metrics dram__bytes_*.sum)")
    json.dump(traffic, open(tpath, "w"), indent=1)
    rf = bench["roofline"]
    md = [f"# {rnd} {cfg}: {bench['config']['desc']}", "",
          "Bench line (no profiler attached): "
          f"value {bench['value'] / 1e9:.3f} G edges/s, {bench['ms_per_step']:.2f} ms/step, "
          f"e2e {bench['e2e']['value'] / 1e9:.3f} G edges/s, modularity {bench['modularity']:.4f}, "
          f"CPU reference {bench['cpu_baseline']['value'] / 1e6:.1f} M edges/s on {bench['cpu_baseline']['cores']} cores "
          f"(Q {bench['cpu_modularity']:.4f}), clocks {bench['clocks']}.", "",
          f"Roofline (local-moving family): achieved {rf['achieved']:.1f} GB/s algorithmic "
          f"(12 B/arc + 32 B/vertex) of {rf['peak']} GB/s measured peak = {100 * rf['frac']:.2f}%; "
          f"algorithmic bytes per sweep (one 'launch' = all local-moving kernels of one iteration) "
          f"{rf['bytes_per_launch'] / 1e6:.1f} MB, "
          f"DRAM traffic per sweep {per_launch / 1e6:.1f} MB "
          f"({(per_launch or 0) / rf['bytes_per_launch']:.2f}x algorithmic).", "",
          f"## Launch list (ncu, cold-cache, serialised; {total:.2f} ms total, local moving "
          f"{move:.2f} ms = {100 * move / total:.1f}%)", "", table, "",
          f"## Local-moving DRAM traffic over one run: {n} launches, read {rd / 1e9:.3f} GB, "
          f"write {wr / 1e9:.3f} GB, {t:.2f} ms", "",
          "## Full capture of the dominant sort-bin kernel (pass 0, second sweep)", "",
          full_capture(os.path.join(OUT, f"prof_lm_sort_{cfg}.raw.csv")), ""]
    path = os.path.join(ROOT, "profiles", f"{rnd}_{cfg}.md")
    open(path, "w").write("\n".join(md))
    print(path)


if __name__ == "__main__":
    main()
