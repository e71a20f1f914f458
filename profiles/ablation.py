"""CompactOptions ablations on the GPU (the paper's tuning
study of Pick-Less period, scan-table value width, switch degrees and probing,
PAPER.md:461-523, reproduced on B200). Run on the GPU box:

    python profiles/ablation.py c1 c2 c3 c5 > profiles/r02_ablation.md

Each row: mean modularity and mean device-resident wall time of 3 runs after a
warm-up, relative to the default row. The probing rows run the device tables
with the reference's probe recurrences (compact_hashtable.hpp:60-82; the
default is quadratic-double, as in the reference)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2501_19004_b200 as lvn  # noqa: E402
from bench import CONFIGS  # noqa: E402

L, O = lvn.LouvainParams, lvn.CompactOptions
variants = [
    ("default", L(), O()),
    ("value_bits=64", L(), O(value_bits=64)),
    ("pick_less period 2", L(), O(pick_less=lvn.PickLessSchedule(period=2))),
    ("pick_less period 8", L(), O(pick_less=lvn.PickLessSchedule(period=8))),
    ("pick_less period 1000 (never)", L(), O(pick_less=lvn.PickLessSchedule(period=1000))),
    ("probing linear", L(), O(probing=lvn.Probing.linear)),
    ("probing quadratic", L(), O(probing=lvn.Probing.quadratic)),
    ("probing double", L(), O(probing=lvn.Probing.double_hash)),
    ("bins: thread_max 0", L(), O(bins=lvn.DeviceBins(thread_max=0))),
    ("bins: thread_max 8", L(), O(bins=lvn.DeviceBins(thread_max=8))),
    ("bins: group_max 64 (hash above)", L(), O(bins=lvn.DeviceBins(group_max=64))),
    ("bins: group_max 128", L(), O(bins=lvn.DeviceBins(group_max=128))),
    ("bins: block_max 1024", L(), O(bins=lvn.DeviceBins(block_max=1024))),
    ("prune off", L(prune=False), O()),
    ("sweep_chunk 65536", L(), O(sweep_chunk=65536)),
    ("sweep_ranges 8", L(), O(sweep_ranges=8)),
    ("singleton rule", L(), O(singleton_rule=True)),
]
cfgs = sys.argv[1:] or ["c1", "c2"]
print("# CompactOptions ablations on one B200\n")
for c in cfgs:
    spec = CONFIGS[c]
    dg = lvn.generate(spec["kind"], **{k: v for k, v in spec.items() if k not in ("kind", "desc")})
    print(f"## {c}: {spec['desc']} ({dg.num_arcs()} arcs)\n")
    print("| variant | Q (mean of 3) | ms (mean of 3) | passes | iterations | vs default ms |")
    print("|---|---:|---:|---:|---|---:|")
    base = None
    for _ in range(3):  # pool and clocks warm before the first row
        lvn.louvain_compact(dg, membership_on_device=True)
    for name, p, o in variants:
        lvn.louvain_compact(dg, p, o, membership_on_device=True)
        rs = [lvn.louvain_compact(dg, p, o, membership_on_device=True) for _ in range(3)]
        q = statistics.mean(r.modularity for r in rs)
        t = statistics.mean(r.wall_seconds for r in rs) * 1e3
        base = base or t
        print(f"| {name} | {q:.5f} | {t:.1f} | {rs[-1].passes} | {rs[-1].iterations_per_pass} | {t / base:.2f}x |",
              flush=True)
    print()
    dg.close()
