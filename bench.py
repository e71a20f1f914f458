#!/usr/bin/env python3
"""Benchmark: edges/s (|E| = arcs of the symmetrized graph / total Louvain time)
of the B200 Louvain engine on BASELINE.json's configs, one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step = one full Louvain run (all passes, local moving + aggregation +
renumbering + final fp64 modularity: the reference's wall_seconds window,
louvain_mc.cpp:163-247) over one synthetic graph.
  value : graph already resident in HBM (device-built), timed with CUDA events.
  e2e   : the same call through the public API with host (pinned) CSR buffers:
          H2D of the CSR and D2H of the membership inside every timed step.
Inputs are far larger than L2 (C2: 2.6 GB of CSR vs 126 MB L2), so no flush
is needed between steps.

N > 1 (torchrun, one process per GPU): the row-sharded engine
(lvn_louvain_sharded) over NCCL, one graph for the whole job;
value = arcs / max-over-ranks time (strong scaling).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # SURVEY.md 8(d); C5 (the north star's 3.8B-arc web graph on 1 B200) is the
    # default N=1 workload
    "c1": dict(kind="rmat", scale=16, edgefactor=16, seed=1,
               desc="RMAT scale-16 edgefactor-16 (Graph500 a,b,c=0.57,0.19,0.19), deduplicated, unit weights"),
    "c2": dict(kind="sbm", n=10_000_000, blocks=1000, avg_degree=32, mu=0.1, seed=2,
               desc="planted-partition SBM, 10M vertices, 1000 blocks, mean degree 32, mu=0.1"),
    "c3": dict(kind="rmat", scale=24, edgefactor=16, seed=3,
               desc="RMAT scale-24 edgefactor-16, deduplicated, unit weights"),
    "c4": dict(kind="grid", side=4899, p=0.6, seed=4,
               desc="4899x4899 lattice, each edge kept with p=0.6 (road-like)"),
    "c5": dict(kind="web", n=50_600_000, avg_degree=75.0, seed=5,
               desc="web-crawl-shaped power-law graph, 50.6M vertices, ~3.8B arcs"),
}
METRIC = "edges/sec (|E|/total Louvain time) at 1/2/4/8 B200 + final modularity vs CPU ref"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (driver / NVML initialisation) stalls CUDA
            # API calls of other processes for milliseconds: let it finish
            # before the timed region (it keeps sampling during the region)
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def gather_peak():
    """measured whole-GPU rate of random 4-byte loads (profiles/gather_peak.json)"""
    try:
        with open(os.path.join(ROOT, "profiles", "gather_peak.json")) as f:
            return float(json.load(f)["gathers_per_s"])
    except Exception:
        return None


def traffic_from_profile(config):
    """dram bytes per launch of the local-moving sweep from a committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            d = json.load(f)
        return d.get(config)
    except Exception:
        return None


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def physical_cores():
    """physical cores of this host (sockets x cores per socket from lscpu)"""
    try:
        out = subprocess.run(["lscpu", "-p=CORE,SOCKET"], capture_output=True, text=True, timeout=10).stdout
        cores = {ln for ln in out.splitlines() if ln and not ln.startswith("#")}
        if cores:
            return len(cores)
    except Exception:
        pass
    return os.cpu_count() or 1


def run_reference(args, world, rank):
    """--impl reference: the reference's own CPU Louvain (louvain_mc, GVE-Louvain
    design, proj/core/src/louvain_mc.cpp:162) built from its sources into
    oracle/_ref/libref.so, on every physical host core, on the same graph.

    The graph is built on the host by oracle/gen_host.cpp (inside libref.so; the
    same samples and canonical CSR as the GPU generator, checked bit for bit by
    tests/test_gpu_build.py), so no product code is mapped into this process.
    BASELINE.md's CPU plan: OMP_PROC_BIND=spread, OMP_PLACES=cores, geometric
    mean of the runs' wall_seconds (louvain_cli.cpp:237-250), arithmetic mean
    of Q; the final single-threaded modularity() inside wall_seconds
    (louvain_mc.cpp:246) is timed separately and reported."""
    if rank != 0:
        return None
    cores = physical_cores()
    # libgomp reads these when it initialises, i.e. when libref.so loads below
    os.environ.setdefault("OMP_PROC_BIND", "spread")
    os.environ.setdefault("OMP_PLACES", "cores")
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    from oracle import ref, ref_available

    cfg = CONFIGS[args.config]
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libref.so was not built"}))
        return None
    t_start = time.time()
    h = ref.generate(cfg["kind"], **{k: v for k, v in cfg.items() if k not in ("kind", "desc")})
    n, arcs = ref.graph_size(h)
    log(f"[reference] {args.config}: {n} vertices, {arcs} arcs, host-generated in {time.time() - t_start:.1f}s")
    budget = float(os.environ.get("LVN_REF_BUDGET_S", "1500"))
    walls, qs, memb = [], [], None
    warm_done = 0
    for i in range(args.warmup + args.steps):
        timed = i >= args.warmup
        if not timed and walls == [] and warm_done >= 1:
            # warm-up runs of a CPU engine only repeat page faults; keep one if
            # the whole run would not fit the step budget
            per = (time.time() - t_start) / max(warm_done, 1)
            if time.time() - t_start + per * (args.warmup - warm_done + args.steps) > budget:
                continue
        if timed and walls:
            per = statistics.mean(walls)
            if time.time() - t_start + per > budget and len(walls) >= 3:
                log(f"[reference] step budget {budget:.0f}s reached after {len(walls)} timed runs")
                break
        r = ref.louvain(h, "mc", thread_count=cores)
        if timed:
            walls.append(r.wall_seconds)
            qs.append(r.modularity)
            memb = r.membership
        else:
            warm_done += 1
        log(f"[reference] run {i}: wall {r.wall_seconds:.2f}s Q {r.modularity:.6f} passes {r.passes}")
    t0 = time.time()
    ref.modularity(h, memb)
    mod_s = time.time() - t0
    t = math.exp(statistics.mean(math.log(x) for x in walls))
    v = arcs / t
    sample = (f"full {args.config} graph ({arcs} arcs), {len(walls)} timed runs after {warm_done} warm-up, "
              f"geometric-mean wall {t:.2f} s")
    out = {
        "metric": METRIC, "value": v, "unit": "edges/s", "n_gpus": world, "steps": len(walls),
        "steps_requested": args.steps, "warmup": warm_done, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (host-generated, seeded)",
        "impl": "reference",
        "config": {"workload": args.config, "desc": cfg["desc"], "vertices": n, "arcs": arcs,
                   "engine": "louvain_mc (reference, OpenMP)",
                   "omp": {k: os.environ.get(k) for k in ("OMP_PROC_BIND", "OMP_PLACES", "OMP_NUM_THREADS")}},
        "modularity": statistics.mean(qs), "modularity_runs": qs,
        "wall_s": walls,
        "final_modularity_s": mod_s,
        "value_without_final_modularity": arcs / max(t - mod_s, 1e-9),
        "cpu_baseline": {"value": v, "unit": "edges/s", "cores": cores, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return out


def cpu_baseline(g, config, budget_s=30.0):
    """The reference louvain_mc on the box's host cores, one bounded run."""
    try:
        from oracle import Csr, ref, ref_available

        if not ref_available():
            return None, None
        csr = Csr(g.offsets, g.targets, g.weights, g.total_weight)
        threads = physical_cores()
        r = ref.louvain(csr, "mc", thread_count=threads)
        return {"value": g.num_arcs() / r.wall_seconds, "unit": "edges/s", "cores": threads,
                "kind": "reference",
                "sample": f"full {config} graph ({g.num_arcs()} arcs), 1 run of louvain_mc, "
                          f"wall {r.wall_seconds:.2f} s"}, r.modularity
    except Exception as e:  # pragma: no cover
        log(f"cpu baseline failed: {e}")
        return None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--value-bits", type=int, default=32)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--shard-rounds", type=int, default=0, help="N>1: exchanges per local-moving iteration (0 = 2N)")
    ap.add_argument("--shard-min-arcs-log2", type=int, default=22,
                    help="N>1: passes with fewer arcs are gathered onto rank 0 (the collapse)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world, rank, local = dist_env()

    if args.impl == "reference":
        # CPU only: rank 0 runs the reference engine, other ranks exit; neither
        # torch nor the product library is loaded into this process
        run_reference(args, world, rank)
        return

    import torch
    import torch.distributed as dist

    if world > 1:
        # LVN_DIST_BACKEND=gloo lets several ranks share one GPU (exercise of the
        # sharded path on a 1-GPU box); the measured runs use NCCL
        backend = os.environ.get("LVN_DIST_BACKEND", "nccl")
        if backend == "gloo":
            local = local % max(torch.cuda.device_count(), 1)
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import numpy as np

    import paper_2501_19004_b200 as lvn
    from paper_2501_19004_b200 import _native

    import ctypes

    if _native.lib().lvn_init(1, (ctypes.c_int * 1)(local)) != 0:
        raise RuntimeError(_native.last_error())
    cfg = CONFIGS[args.config]
    t0 = time.time()
    dg = lvn.generate(cfg["kind"], **{k: v for k, v in cfg.items() if k not in ("kind", "desc")})
    n, arcs = dg.num_vertices(), dg.num_arcs()
    log(f"[rank {rank}] {args.config}: {n} vertices, {arcs} arcs, generated in {time.time() - t0:.1f}s")
    opts = lvn.CompactOptions(value_bits=args.value_bits, shard_rounds=args.shard_rounds,
                              shard_min_arcs_log2=args.shard_min_arcs_log2)
    # N > 1: one process per GPU, passes sharded by row range over NCCL
    # (SURVEY.md 8(e)); the whole job's work is fixed as N grows (strong scaling)
    # The collectives are the library's own NCCL communicator (stream-ordered
    # inside liblvn.so, no Python on the data path); LVN_DIST_BACKEND=gloo
    # (several ranks sharing one GPU) goes through torch.distributed instead.
    comm = None
    if world > 1:
        from paper_2501_19004_b200.distributed import Collectives, NcclComm

        comm = NcclComm() if os.environ.get("LVN_DIST_BACKEND", "nccl") == "nccl" else Collectives(location="cuda")

    def run(g, on_device):
        if comm is not None:
            return lvn.louvain_sharded(g, comm, None, opts, membership_on_device=on_device)
        return lvn.louvain_compact(g, None, opts, membership_on_device=on_device)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- value: device-resident input -------------------------------------------
    for _ in range(args.warmup):
        run(dg, True)
    sampler = ClockSampler(local)
    # only the last result stays alive: each holds its device membership, and
    # holding every step's would drain the pool's block cache mid-run (C3:
    # steps 3-5 at 240-400 ms instead of 185 ms); a caller looping over runs
    # drops them too
    results, walls = [], []

    def keep(res):
        walls.append(res.wall_seconds)
        results[:] = [res]
    l0 = lvn.launch_count()
    barrier()
    # inputs that fit a few L2s (C1: 15 MB): the L2 is flushed between timed
    # steps by a 512 MB write outside the timed intervals (per-step events)
    l2 = torch.cuda.get_device_properties(local).L2_cache_size
    csr_bytes = 8 * (n + 1) + 8 * arcs
    flush = csr_bytes < 4 * l2
    scratch = torch.empty(512 << 20, dtype=torch.uint8, device="cuda") if flush else None
    with sampler:
        if flush:
            elapsed_ms = 0.0
            for i in range(args.steps):
                scratch.fill_(i & 0xFF)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                keep(run(dg, True))
                b.record()
                b.synchronize()
                elapsed_ms += a.elapsed_time(b)
            barrier()
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                keep(run(dg, True))
            e1.record()
            barrier()
            elapsed_ms = e0.elapsed_time(e1)
    scratch = None
    launches = (lvn.launch_count() - l0) // args.steps
    elapsed = max_over_ranks(elapsed_ms / 1e3)
    step_s = elapsed / args.steps
    value = arcs / step_s
    clocks = sampler.summary()
    r = results[-1]
    mv = r.stats["move"]
    peak, peak_kind = measured_peaks()
    move_gbps = mv.bytes / mv.seconds / 1e9 if mv.seconds else 0.0
    per_launch_bytes = mv.bytes / max(mv.launches, 1)
    traffic = traffic_from_profile(args.config)
    gpeak = gather_peak()

    step_ms = [round(x * 1e3, 2) for x in walls]
    # ---- e2e: host (pinned) buffers through the public API ------------------------
    e2e = None
    if not args.no_e2e:
        host = dg.download(np.empty(n + 1, np.uint64), torch.empty(arcs, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32),
                           torch.empty(arcs, dtype=torch.float32, pin_memory=True).numpy())
        off_pinned = torch.empty(n + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
        off_pinned[:] = host.offsets
        hg = lvn.CsrGraph(off_pinned, host.targets, host.weights, host.total_weight)
        # the device copy and the value leg's device memberships are not part
        # of this leg: release them so the host-input runs see the device as a
        # user's first call would (else 30+ GB stay pinned in the pool)
        results = [r]
        dg.close()
        assert hg.offsets.ctypes.data == off_pinned.ctypes.data
        # warm-up with two results alive: the timed loop holds the previous
        # step's host membership while the next runs, so it cycles two pinned
        # result blocks (the second one's first cudaMallocHost is a warm-up cost)
        w1 = run(hg, False)
        w2 = run(hg, False)
        del w1, w2
        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        qs, h2d, e2e_walls, calls = [], [], [], []
        f0.record()
        for _ in range(args.steps):
            t_call = time.perf_counter()
            re2e = run(hg, False)
            calls.append(time.perf_counter() - t_call)
            qs.append(re2e.modularity)
            h2d.append(re2e.h2d_bytes)
            e2e_walls.append(re2e.wall_seconds)
        f1.record()
        barrier()
        e2e_s = max_over_ranks(f0.elapsed_time(f1) / 1e3) / args.steps
        # the bytes the engine actually moved over PCIe: offsets + targets, and
        # the weights unless the host scan found them all equal (unit weights:
        # read on the host, filled on the device); every byte of the input is
        # still read inside the timed region
        e2e = {"value": arcs / e2e_s, "unit": "edges/s", "ms_per_step": e2e_s * 1e3,
               "h2d_bytes_per_step": int(statistics.mean(h2d)), "d2h_bytes_per_step": 4 * n,
               "input_bytes_per_step": 8 * (n + 1) + 8 * arcs,
               # per step: the engine's own wall (lvn_result.wall_seconds) and the whole call
               "step_ms": [round(x * 1e3, 2) for x in e2e_walls],
               "call_ms": [round(x * 1e3, 2) for x in calls],
               "weights": "constant: verified on the host, filled on the device"
               if statistics.mean(h2d) < 8 * (n + 1) + 8 * arcs else "copied"}
    else:
        host = None

    cpu, cpu_q = (None, None)
    if rank == 0 and not args.no_cpu_baseline:
        if host is None:
            host = dg.download()
            dg.close()
        cpu, cpu_q = cpu_baseline(host, args.config)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if args.value_bits == 64 else "f32+f64",
            "data": "synthetic (device-generated, seeded)",
            "config": {"workload": args.config, "desc": cfg["desc"], "vertices": n, "arcs": arcs,
                       "parallelism": f"row-sharded x{world} over NCCL" if world > 1 else "single GPU",
                       "l2_flush": (f"512 MB write between timed steps (input {csr_bytes / 1e6:.0f} MB < 4 x L2)"
                                    if flush else f"not needed: input {csr_bytes / 1e9:.1f} GB >> {l2 / 1e6:.0f} MB L2")},
            # the CLI's undirected rate (num_arcs / 2 / wall, louvain_cli.cpp:177), labelled
            "undirected_edges_per_s": value / 2,
            "modularity": r.modularity, "num_communities": r.num_communities, "passes": r.passes,
            "sharded_passes": r.sharded_passes, "exchange_seconds": r.exchange_seconds,
            "iterations_per_pass": r.iterations_per_pass,
            "pass_ms": [round(x * 1e3, 2) for x in r.pass_seconds],
            "step_ms": step_ms,
            "phase_seconds": {"local_moving": r.phase.local_moving, "aggregation": r.phase.aggregation,
                              "other": r.phase.other},
            "kernel_seconds": {k: s.seconds for k, s in r.stats.items()},
            "kernel_gbps": {k: s.gbps for k, s in r.stats.items()},
            "roofline": {"bound": "hbm",
                         "kernel": "local-moving sweep (lm_thread/lm_sort/lm_group/lm_block/lm_hub_*); "
                                   "one launch = every local-moving kernel of one iteration",
                         "achieved": move_gbps, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": move_gbps / peak if peak else None,
                         "bytes_per_launch": per_launch_bytes,
                         "traffic": traffic,
                         # the ceiling that binds a sweep: random element accesses
                         # (C[t], Sigma[c] gathers, neighbour marks) against the
                         # measured random-gather rate of the L1TEX path
                         "gather": {"achieved": mv.gathers_per_second, "peak": gpeak, "unit": "random accesses/s",
                                    "frac": mv.gathers_per_second / gpeak if gpeak else None,
                                    "per_arc": mv.gathers / mv.arcs if mv.arcs else None}},
            "cpu_baseline": cpu, "cpu_modularity": cpu_q,
            "modularity_minus_cpu": (r.modularity - cpu_q) if cpu_q is not None else None,
            "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
