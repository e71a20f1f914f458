"""The sharded engine (lvn_louvain_sharded) end to end on the
GPU: 2 and 3 ranks share the one B200 of the test box over gloo (device
buffers staged through the host; NCCL needs one GPU per rank, which the
8-GPU bench uses). Each rank holds only its own rows; replicated membership
and Sigma are exchanged every round, marks every iteration, and each
super-row is merged by one rank, so all ranks must return the same
membership, whose modularity the oracle recomputes. Below the collapse
threshold rank 0 runs alone and the others receive its result. The
library's own NCCL communicator is exercised at world size 1 (its
collectives through the public callbacks, and a whole run)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from graphs import planted, random_graph, rmat

pytestmark = pytest.mark.gpu


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def make(case):
    if case == "planted":
        return planted(30000, 60, 24, 0.15, 4)
    if case == "rmat":
        return rmat(14, 16, 9)
    if case == "hubs":
        from test_gpu_parity import hubs_graph

        return hubs_graph(30000, 3, 12000, 150000, 6)
    return random_graph(20000, 120000, 5)


def _worker(rank, world, port, case, min_log2, q, rounds=0, env=None):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    os.environ.update(env or {})
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2501_19004_b200 as lvn
        from paper_2501_19004_b200.distributed import Collectives

        g = make(case)
        G = lvn.CsrGraph(g.offsets, g.targets, g.weights, g.total_weight)
        comm = Collectives(location="cuda")
        r = lvn.louvain_sharded(G, comm, options=lvn.CompactOptions(shard_min_arcs_log2=min_log2,
                                                                     shard_rounds=rounds))
        q.put((rank, dict(q=r.modularity, m=np.asarray(r.membership), sp=r.sharded_passes, ns=r.num_shards,
                          passes=r.passes, calls=dict(comm.calls), err=comm.errors)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc()))


def run(world, case, min_log2=0, rounds=0, env=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, min_log2, q, rounds, env)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
    for r, v in out.items():
        assert isinstance(v, dict), v
        assert not v["err"], v["err"]
    return out


@pytest.mark.parametrize("world,case", [(2, "planted"), (2, "rmat"), (3, "hubs"), (2, "random")])
def test_sharded_lockstep_and_quality(lvn_single, port, world, case):
    out = run(world, case)
    g = make(case)
    single = lvn_single(g)
    m0 = out[0]["m"]
    for r, v in out.items():
        assert v["ns"] == world and v["sp"] >= 1
        assert v["calls"]["allreduce"] > 0 and v["calls"]["allgatherv"] > 0 and v["calls"]["alltoallv"] > 0
        assert (v["m"] == m0).all(), f"rank {r} diverged from rank 0"
        assert abs(v["q"] - port.modularity(g, v["m"])) <= 1e-9 * max(1.0, abs(v["q"]))
    k = int(m0.max()) + 1
    assert set(np.unique(m0)) == set(range(k))  # contiguous ids
    # stale cross-rank reads cost little quality against the single-GPU engine
    assert out[0]["q"] >= single - 0.01, (out[0]["q"], single)


def test_sharded_collapse_threshold(lvn_single, port):
    # no pass reaches 2^40 arcs: rank 0 runs everything, the others get its result
    out = run(2, "planted", min_log2=40)
    m0 = out[0]["m"]
    g = make("planted")
    for v in out.values():
        assert v["sp"] == 0 and v["calls"]["alltoallv"] == 0
        assert (v["m"] == m0).all() and v["q"] == out[0]["q"] and v["passes"] == out[0]["passes"]
    assert abs(out[0]["q"] - port.modularity(g, m0)) <= 1e-9


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_collapse_mid_run(lvn_single, port, world):
    # pass 0 (~720 K arcs) sharded, the aggregated graphs gathered onto rank 0
    out = run(world, "planted", min_log2=16, rounds=1)
    m0 = out[0]["m"]
    g = make("planted")
    for v in out.values():
        assert v["sp"] == 1 and v["calls"]["alltoallv"] == 2
        assert (v["m"] == m0).all() and v["q"] == out[0]["q"] and v["passes"] == out[0]["passes"]
    assert abs(out[0]["q"] - port.modularity(g, m0)) <= 1e-9
    assert out[0]["q"] >= lvn_single(g) - 0.01


def test_sharded_aggregation_in_slices(lvn_single, port):
    # the sort variant of the partial super-edges, built from 4096-arc slices
    # (the C5-scale memory bound) and merged
    out = run(2, "rmat", env={"LVN_SHARD_AGG_SORT": "1", "LVN_SHARD_SLICE_LOG2": "12"})
    g = make("rmat")
    m0 = out[0]["m"]
    for v in out.values():
        assert (v["m"] == m0).all() and v["sp"] >= 1
    assert abs(out[0]["q"] - port.modularity(g, m0)) <= 1e-9
    assert out[0]["q"] >= lvn_single(g) - 0.01


def _nccl_worker(port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=0, world_size=1)
        import ctypes as C

        import paper_2501_19004_b200 as lvn
        from paper_2501_19004_b200 import _native as N
        from paper_2501_19004_b200.distributed import NcclComm

        v = C.c_int()
        assert N.lib().lvn_nccl_version(C.byref(v)) == 0 and v.value >= 22700
        comm = NcclComm()
        st = comm.struct
        assert (st.rank, st.size) == (0, 1)
        x = torch.arange(1000, dtype=torch.float64, device="cuda")
        assert st.allreduce(st.user, x.data_ptr(), 1000, N.LVN_F64, N.LVN_SUM) == 0
        assert torch.equal(x, torch.arange(1000, dtype=torch.float64, device="cuda"))
        y = torch.zeros(64, dtype=torch.uint8, device="cuda")
        src = torch.arange(64, dtype=torch.uint8, device="cuda")
        assert st.allgatherv(st.user, src.data_ptr(), y.data_ptr(), (C.c_uint64 * 1)(64)) == 0
        assert torch.equal(y, src)
        z = torch.zeros(64, dtype=torch.uint8, device="cuda")
        assert st.alltoallv(st.user, src.data_ptr(), (C.c_uint64 * 1)(64), z.data_ptr(), (C.c_uint64 * 1)(64)) == 0
        assert torch.equal(z, src)
        g = make("planted")
        G = lvn.CsrGraph(g.offsets, g.targets, g.weights, g.total_weight)
        r = lvn.louvain_sharded(G, comm)
        # the sharded algorithm itself over the library's NCCL collectives
        # (stream-ordered allgatherv / alltoallv / allreduce at world size 1):
        # every pass sharded, then collapsed onto rank 0 below 2^16 arcs
        os.environ["LVN_SHARD_SINGLE"] = "1"
        r2 = lvn.louvain_sharded(G, comm, options=lvn.CompactOptions(shard_min_arcs_log2=0))
        r3 = lvn.louvain_sharded(G, comm, options=lvn.CompactOptions(shard_min_arcs_log2=16))
        del os.environ["LVN_SHARD_SINGLE"]
        comm.close()
        assert r2.sharded_passes >= 2 and r3.sharded_passes == 1, (r2.sharded_passes, r3.sharded_passes)
        assert r2.exchange_seconds > 0.0
        q.put(("ok", r.modularity, np.asarray(r.membership), r2.modularity, np.asarray(r2.membership),
               r3.modularity, np.asarray(r3.membership)))
        dist.destroy_process_group()
    except Exception:  # noqa: BLE001
        import traceback

        q.put((traceback.format_exc(),) + (None,) * 6)


def test_nccl_comm_world1(port, lvn_single):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(free_port(), q))
    p.start()
    st, qq, m, q2, m2, q3, m3 = q.get(timeout=300)
    p.join(timeout=60)
    assert st == "ok", st
    g = make("planted")
    single = lvn_single(g)
    for qx, mx in ((qq, m), (q2, m2), (q3, m3)):
        assert abs(qx - port.modularity(g, mx)) <= 1e-9
        assert qx >= single - 0.01


@pytest.fixture(scope="module")
def lvn_single():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a B200")
    import paper_2501_19004_b200 as lvn

    def f(g):
        return lvn.louvain_compact(lvn.CsrGraph(g.offsets, g.targets, g.weights, g.total_weight)).modularity

    return f
