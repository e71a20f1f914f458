"""Host side of the sharded engine on CPU: the row split
rule and the torch.distributed collectives the engine calls, exercised by two
gloo ranks exactly as lvn_louvain_sharded calls them (through the ctypes
function pointers of the lvn_comm struct, on host buffers)."""

import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from graphs import random_graph, rmat


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def split_rule(offsets, parts):
    """bounds[k] = first row whose offset reaches floor(k*A/parts); bounds[parts] = n"""
    off = np.asarray(offsets, np.uint64)
    n, A = len(off) - 1, int(off[-1])
    b = [int(np.searchsorted(off, (k * A) // parts, side="left")) for k in range(parts)] + [n]
    return np.array(b, np.uint32)


@pytest.mark.parametrize("parts", [1, 2, 3, 8, 64])
def test_partition_rows_rule_and_balance(parts):
    import paper_2501_19004_b200 as lvn

    for g in (random_graph(5000, 40000, 3), rmat(12, 16, 5)):
        b = lvn.partition_rows(g.offsets, parts)
        assert (b == split_rule(g.offsets, parts)).all()
        assert b[0] == 0 and b[-1] == g.n and (np.diff(b.astype(np.int64)) >= 0).all()
        arcs = np.diff(g.offsets[b.astype(np.int64)].astype(np.int64))
        maxdeg = int(np.diff(g.offsets.astype(np.int64)).max())
        assert arcs.max() <= g.offsets[-1] / parts + maxdeg  # within one row of balanced


def test_partition_rows_degenerate():
    import paper_2501_19004_b200 as lvn

    off = np.zeros(11, np.uint64)  # 10 rows, no arcs
    assert list(lvn.partition_rows(off, 4)) == [0, 0, 0, 0, 10]
    assert list(lvn.partition_rows(np.array([0, 5], np.uint64), 3)) == [0, 1, 1, 1]  # one row: rank 0


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_19004_b200 import _native as N
        from paper_2501_19004_b200.distributed import Collectives

        comm = Collectives(location="cpu")
        st = comm.struct
        assert (st.rank, st.size) == (rank, world)
        rng = np.random.default_rng(rank)
        # Sigma deltas: f64 sum
        d = rng.standard_normal(1000)
        want = sum(np.random.default_rng(r).standard_normal(1000) for r in range(world))
        assert st.allreduce(None, d.ctypes.data, d.size, N.LVN_F64, N.LVN_SUM) == 0
        assert np.allclose(d, want, rtol=0, atol=1e-12)
        # neighbour marks: u8 max (only own marks set, remote ones OR in)
        f = np.zeros(97, np.uint8)
        f[rank::world] = 1
        assert st.allreduce(None, f.ctypes.data, f.size, N.LVN_U8, N.LVN_MAX) == 0
        assert f.all()
        # counters: u64 sum
        c = np.array([rank + 1, 2 ** 40 + rank, 7], np.uint64)
        assert st.allreduce(None, c.ctypes.data, 3, N.LVN_U64, N.LVN_SUM) == 0
        tot = sum(range(1, world + 1))
        assert list(c) == [tot, world * 2 ** 40 + sum(range(world)), 7 * world]
        # membership of own rows: uneven u32 ranges, send aliases recv, one empty range
        n = 1001
        bounds = [0] + [n * k // world for k in range(1, world)] + [n]
        if world > 2:
            bounds[1] = 0  # rank 0 owns nothing
        C_ = np.full(n, 0xFFFFFFFF, np.uint32)
        lo, hi = bounds[rank], bounds[rank + 1]
        C_[lo:hi] = np.arange(lo, hi, dtype=np.uint32) * 3
        counts = (C.c_uint64 * world)(*[4 * (bounds[k + 1] - bounds[k]) for k in range(world)])
        assert st.allgatherv(None, C_.ctypes.data + 4 * lo, C_.ctypes.data, counts) == 0
        assert (C_ == np.arange(n, dtype=np.uint32) * 3).all()
        # partial super-edges routed to row owners: rank r sends (r + 1) * (k + 1) u64
        # entries to rank k, each tagged (sender, receiver, index)
        scounts = [(rank + 1) * (k + 1) for k in range(world)]
        rcounts = [(j + 1) * (rank + 1) for j in range(world)]
        send = np.concatenate([np.array([(rank << 40) | (k << 20) | i for i in range(scounts[k])], np.uint64)
                               for k in range(world)])
        recv = np.zeros(sum(rcounts), np.uint64)
        sb = (C.c_uint64 * world)(*[8 * x for x in scounts])
        rb = (C.c_uint64 * world)(*[8 * x for x in rcounts])
        assert st.alltoallv(None, send.ctypes.data, sb, recv.ctypes.data, rb) == 0
        want = np.concatenate([np.array([(j << 40) | (rank << 20) | i for i in range(rcounts[j])], np.uint64)
                               for j in range(world)])
        assert (recv == want).all()
        # a failing collective is reported, not raised
        assert st.allreduce(None, d.ctypes.data, d.size, 99, N.LVN_SUM) == 1
        assert comm.errors
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        import traceback

        q.put((rank, traceback.format_exc() + repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_collectives_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert all(v == "ok" for v in res.values()), res
