"""Key counters of every kernel in an ncu report (raw page), or of a raw-page
CSV export: python profiles/ncu_summary.py rep.ncu-rep|raw.csv"""
import csv
import io
import subprocess
import sys

if sys.argv[1].endswith(".csv"):
    out = open(sys.argv[1]).read()
else:
    out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, data = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct", "lts__t_sectors_srcunit_tex_op_read.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
stalls = [c for c in h if c.startswith("smsp__average_warps_issue_stalled_") and c.endswith("_per_issue_active.ratio")]
for r in data:
    print("=====", r[h.index("Kernel Name")][:110])
    for w in want:
        if w in h:
            print(f"   {w:70s} {r[h.index(w)]} {units[h.index(w)]}")
    st = sorted(((float(r[h.index(c)] or 0), c) for c in stalls), reverse=True)[:6]
    print("   stalls/issue: " + ", ".join(f"{c.split('stalled_')[1].split('_per')[0]}={v:.2f}" for v, c in st))
