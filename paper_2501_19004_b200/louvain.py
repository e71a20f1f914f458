"""Python mirror of the reference's Louvain interface, backed by liblvn.so.

Names, argument meaning and error behaviour follow the reference C++ API so
the parity tests read like the reference's own tests:

    LouvainParams / PhaseTimes / LouvainResult   proj/core/include/louvain/louvain.hpp:9-39
    CompactOptions / PickLessSchedule /
        SwitchDegrees                            proj/core/include/louvain/louvain_compact.hpp:17-40
    CsrGraph                                     proj/core/include/louvain/graph.hpp:38-54
    louvain_compact (the GPU engine)             louvain_compact.hpp:57-58
    compact_aggregate / louvain_aggregate        louvain_compact.hpp:76-77, louvain_mc.hpp:96-97
    compact_evaluate_move                        louvain_compact.hpp:65-72
    renumber_communities / lookup_dendrogram     louvain_mc.hpp:101-105
    modularity / count_communities               quality.hpp:27-40
    vertex_weights                               graph.hpp:79
    DegenerateGraphError / InternalError /
        ParseError                               errors.hpp:10-31

Every call goes through the C-ABI (include/lvn.h) to CUDA kernels on the
B200; nothing here computes on the CPU.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _native as N

# --------------------------------------------------------------------------
# errors (errors.hpp:10-31; status codes of include/lvn.h)
# --------------------------------------------------------------------------


class ParseError(RuntimeError):
    """Input could not be parsed (errors.hpp:10-22)."""


class DegenerateGraphError(RuntimeError):
    """Graph cannot be clustered, m == 0 (errors.hpp:25-27)."""


class InternalError(RuntimeError):
    """A structural invariant was violated (errors.hpp:29-31)."""


class CudaError(RuntimeError):
    """CUDA failure inside liblvn."""


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = N.last_error()
    if rc == 1:
        raise ValueError(msg)  # std::invalid_argument
    if rc == 2:
        raise DegenerateGraphError(msg)
    if rc == 3:
        raise InternalError(msg)
    if rc == 5:
        raise MemoryError(msg)
    raise CudaError(msg)


# --------------------------------------------------------------------------
# options and results
# --------------------------------------------------------------------------


class Probing(IntEnum):  # compact_hashtable.hpp:13-18
    linear = 0
    quadratic = 1
    double_hash = 2
    quadratic_double = 3


@dataclass
class LouvainParams:  # louvain.hpp:9-18
    max_passes: int = 10
    max_iterations: int = 20
    initial_tolerance: float = 0.01
    tolerance_drop: float = 10.0
    aggregation_tolerance: float = 0.8
    thread_count: int = 0  # validated for parity; the GPU ignores it
    chunk_size: int = 2048  # validated for parity; the GPU ignores it
    prune: bool = True


@dataclass
class PickLessSchedule:  # louvain_compact.hpp:17-19
    period: int = 4


def pick_less_active(iteration: int, period: int) -> bool:  # louvain_compact.hpp:22-24
    return (iteration + period // 2) % period == 0


@dataclass
class SwitchDegrees:  # louvain_compact.hpp:30-33
    move: int = 64
    aggregate: int = 128


@dataclass
class DeviceBins:
    """Degree classes of the device kernels (thread / 8-lane group / warp /
    block-with-smem-table / block-with-global-table)."""

    thread_max: int = 4
    group_max: int = 256
    warp_max: int = 256
    block_max: int = 4096


@dataclass
class CompactOptions:  # louvain_compact.hpp:35-40
    pick_less: PickLessSchedule = field(default_factory=PickLessSchedule)
    switch_degrees: SwitchDegrees = field(default_factory=SwitchDegrees)
    probing: Probing = Probing.quadratic_double
    value_bits: int = 32
    bins: DeviceBins = field(default_factory=DeviceBins)
    sweep_chunk: int = 0  # vertices per launch of a sweep; 0 automatic, 2**32-1 unbounded
    sweep_order: int = 0  # 0 low degree first (reference compact order), 1 hubs first
    sweep_ranges: int = 0  # vertex-id ranges per sweep (1 = compact order); 0 automatic
    singleton_rule: bool = False  # singleton joins singleton only toward the lower id
    shard_min_arcs_log2: int = 22  # louvain_sharded: shard passes with >= 2**this arcs
    shard_rounds: int = 0  # louvain_sharded: exchanges per iteration (rounds over own rows); 0 = 2 x ranks
    first_range_arcs_log2: int = 27  # >= 16 * 2**this arcs: pass 0's first sweep in 16 id ranges (upload overlap); 0 off


@dataclass
class PhaseTimes:  # louvain.hpp:20-26
    local_moving: float = 0.0
    aggregation: float = 0.0
    other: float = 0.0

    def total(self) -> float:
        return self.local_moving + self.aggregation + self.other


@dataclass
class KernelStats:
    seconds: float
    bytes: float
    launches: int
    items: int
    arcs: int
    gathers: int = 0  # random element accesses (local moving: C[t], Sigma[c], neighbour marks)

    @property
    def gbps(self) -> float:
        return self.bytes / self.seconds / 1e9 if self.seconds > 0 else 0.0

    @property
    def gathers_per_second(self) -> float:
        return self.gathers / self.seconds if self.seconds > 0 else 0.0


@dataclass
class LouvainResult:  # louvain.hpp:28-39 (+ device breakdown)
    membership: np.ndarray
    num_communities: int = 0
    modularity: float = 0.0
    passes: int = 0
    aggregations: int = 0
    iterations_per_pass: list = field(default_factory=list)
    tolerance_per_pass: list = field(default_factory=list)
    pass_seconds: list = field(default_factory=list)
    phase: PhaseTimes = field(default_factory=PhaseTimes)
    wall_seconds: float = 0.0
    vertices_per_pass: list = field(default_factory=list)
    arcs_per_pass: list = field(default_factory=list)
    h2d_seconds: float = 0.0
    h2d_bytes: int = 0  # input bytes copied host -> device (constant weights are filled on the device)
    d2h_seconds: float = 0.0
    stats: dict = field(default_factory=dict)
    num_shards: int = 1
    sharded_passes: int = 0
    exchange_seconds: float = 0.0
    levels: list = field(default_factory=list)  # dendrogram (keep_levels=True)


@dataclass
class CsrGraph:  # graph.hpp:38-54
    offsets: np.ndarray
    targets: np.ndarray
    weights: np.ndarray
    total_weight: float

    def __post_init__(self):
        self.offsets = np.ascontiguousarray(self.offsets, dtype=np.uint64)
        self.targets = np.ascontiguousarray(self.targets, dtype=np.uint32)
        self.weights = np.ascontiguousarray(self.weights, dtype=np.float32)

    def num_vertices(self) -> int:
        return len(self.offsets) - 1

    def num_arcs(self) -> int:
        return int(self.offsets[-1]) if len(self.offsets) else 0

    def degree(self, u: int) -> int:
        return int(self.offsets[u + 1] - self.offsets[u])

    def _csr(self) -> N.lvn_csr:
        return N.lvn_csr(self.num_vertices(), self.num_arcs(), self.offsets.ctypes.data,
                         self.targets.ctypes.data, self.weights.ctypes.data, float(self.total_weight),
                         N.LVN_HOST)


class DeviceGraph:
    """A CSR resident in device memory (built by the device generators or
    uploaded once); pass it anywhere a CsrGraph is accepted."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        self._view = N.lvn_csr()
        _check(N.lib().lvn_dgraph_view(self._h, C.byref(self._view)))

    @classmethod
    def upload(cls, g: CsrGraph) -> "DeviceGraph":
        h = C.c_void_p()
        csr = g._csr()
        _check(N.lib().lvn_dgraph_upload(C.byref(csr), C.byref(h)))
        return cls(h.value)

    def num_vertices(self) -> int:
        return self._view.num_vertices

    def num_arcs(self) -> int:
        return self._view.num_arcs

    @property
    def total_weight(self) -> float:
        return self._view.total_weight

    @property
    def device_pointers(self):
        return self._view.offsets, self._view.targets, self._view.weights

    def _csr(self) -> N.lvn_csr:
        return self._view

    def download(self, offsets=None, targets=None, weights=None) -> CsrGraph:
        n, a = self.num_vertices(), self.num_arcs()
        off = offsets if offsets is not None else np.empty(n + 1, np.uint64)
        tgt = targets if targets is not None else np.empty(max(a, 1), np.uint32)
        w = weights if weights is not None else np.empty(max(a, 1), np.float32)
        _check(N.lib().lvn_dgraph_download(self._h, off.ctypes.data, tgt.ctypes.data, w.ctypes.data))
        return CsrGraph(off, tgt[:a], w[:a], self.total_weight)

    def close(self) -> None:
        if self._h and self._h.value:
            N.lib().lvn_dgraph_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def generate(kind: str, seed: int = 1, **kw) -> DeviceGraph:
    """Device-built synthetic graphs (SURVEY.md 8(d) shapes): rmat(scale,
    edgefactor), sbm(n, blocks, avg_degree, mu), grid(side, p), web(n,
    avg_degree), uniform(n, edges). Unit weights, deduplicated, no self-loops."""
    gp = N.lvn_gen_params()
    gp.seed = seed
    if kind == "rmat":
        gp.kind, gp.scale = 0, kw["scale"]
        gp.edges = (1 << kw["scale"]) * kw.get("edgefactor", 16)
        gp.a, gp.b, gp.c = kw.get("a", 0.57), kw.get("b", 0.19), kw.get("c", 0.19)
    elif kind == "sbm":
        gp.kind, gp.n, gp.blocks = 1, kw["n"], kw["blocks"]
        gp.edges = int(kw["n"] * kw.get("avg_degree", 32) / 2)
        gp.mu = kw.get("mu", 0.1)
    elif kind == "grid":
        gp.kind, gp.n, gp.p = 2, kw["side"], kw.get("p", 0.6)
    elif kind == "web":
        gp.kind, gp.n, gp.avg_degree = 3, kw["n"], kw.get("avg_degree", 75.0)
    elif kind == "uniform":
        gp.kind, gp.n, gp.edges = 4, kw["n"], kw["edges"]
    else:
        raise ValueError(f"unknown generator {kind}")
    h = C.c_void_p()
    _check(N.lib().lvn_generate(C.byref(gp), C.byref(h)))
    return DeviceGraph(h.value)


# --------------------------------------------------------------------------
# parameter marshalling
# --------------------------------------------------------------------------


def _params(params: LouvainParams | None, options: CompactOptions | None, on_device=False,
            keep_levels=False) -> N.lvn_params:
    params = params or LouvainParams()
    options = options or CompactOptions()
    p = N.lvn_params()
    N.lib().lvn_params_default(C.byref(p))
    p.max_passes = params.max_passes
    p.max_iterations = params.max_iterations
    p.initial_tolerance = params.initial_tolerance
    p.tolerance_drop = params.tolerance_drop
    p.aggregation_tolerance = params.aggregation_tolerance
    p.thread_count = params.thread_count
    p.chunk_size = params.chunk_size
    p.prune = int(bool(params.prune))
    p.pick_less_period = options.pick_less.period
    p.switch_move = options.switch_degrees.move & 0xFFFFFFFFFFFFFFFF
    p.switch_aggregate = options.switch_degrees.aggregate & 0xFFFFFFFFFFFFFFFF
    p.probing = int(options.probing)
    p.value_bits = options.value_bits
    p.bin_thread_max = options.bins.thread_max
    p.bin_group_max = options.bins.group_max
    p.bin_warp_max = options.bins.warp_max
    p.bin_block_max = options.bins.block_max
    p.membership_on_device = int(on_device)
    p.sweep_chunk = options.sweep_chunk
    p.sweep_order = options.sweep_order
    p.sweep_ranges = options.sweep_ranges
    p.singleton_rule = int(bool(options.singleton_rule))
    p.shard_min_arcs_log2 = options.shard_min_arcs_log2
    p.shard_rounds = options.shard_rounds
    p.keep_levels = int(bool(keep_levels))
    p.first_range_arcs_log2 = options.first_range_arcs_log2
    return p


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint32)


def _graph_out(ptr) -> CsrGraph:
    go = ptr.contents
    n, a = go.num_vertices, go.num_arcs
    off = np.ctypeslib.as_array(go.offsets, (n + 1,)).copy()
    tgt = np.ctypeslib.as_array(go.targets, (max(a, 1),))[:a].copy()
    w = np.ctypeslib.as_array(go.weights, (max(a, 1),))[:a].copy()
    out = CsrGraph(off, tgt, w, go.total_weight)
    N.lib().lvn_graph_free(ptr)
    return out


# --------------------------------------------------------------------------
# engine and phase APIs
# --------------------------------------------------------------------------


def louvain_compact(g, params: LouvainParams | None = None, options: CompactOptions | None = None,
                    membership_on_device: bool = False, keep_levels: bool = False) -> LouvainResult:
    """The ν-Louvain engine on the B200 (louvain_compact.hpp:57-58). With
    keep_levels the result carries the dendrogram: `levels[k]` maps the
    vertices of pass k's graph to their communities (lookup_dendrogram,
    louvain_mc.cpp:145-160, composes them into `membership`)."""
    p = _params(params, options, membership_on_device, keep_levels)
    csr = g._csr()
    out = C.POINTER(N.lvn_result)()
    _check(N.lib().lvn_louvain(C.byref(csr), C.byref(p), C.byref(out)))
    return _result(out)


def louvain_sharded(g, comm, params: LouvainParams | None = None, options: CompactOptions | None = None,
                    membership_on_device: bool = False) -> LouvainResult:
    """louvain_compact sharded over the ranks of `comm` (one process per GPU,
    SURVEY.md 8(e)); `comm` is a paper_2501_19004_b200.distributed.Collectives
    (or anything exposing a ctypes `lvn_comm` as `.struct`). Every rank passes
    the same graph and gets the same result."""
    p = _params(params, options, membership_on_device)
    csr = g._csr()
    out = C.POINTER(N.lvn_result)()
    _check(N.lib().lvn_louvain_sharded(C.byref(csr), C.byref(p), C.byref(comm.struct), C.byref(out)))
    return _result(out)


def partition_rows(offsets, parts: int) -> np.ndarray:
    """Row split of a sharded pass: bounds[k] = first row whose offset reaches
    floor(k*A/parts), bounds[parts] = n (the engine's rule, host copy)."""
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = len(off) - 1
    out = np.empty(parts + 1, np.uint32)
    _check(N.lib().lvn_partition_rows(off.ctypes.data, n, parts, out.ctypes.data))
    return out


class _ResultHandle:
    """Keeps an lvn_result alive while its device membership is in use."""

    def __init__(self, out):
        self.out = out

    def __del__(self):
        try:
            N.lib().lvn_result_free(self.out)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def _result(out) -> LouvainResult:
    keep = False
    try:
        r = out.contents
        k = r.passes
        lst = lambda ptr: [ptr[i] for i in range(k)]  # noqa: E731
        if r.membership_on_device:
            membership = np.empty(0, np.uint32)
            dev_ptr = C.cast(r.membership, C.c_void_p).value
        else:
            # zero-copy view of the library's pinned result block: the block
            # goes back to the library (lvn_result_free) when the last array
            # viewing it is collected (a 50 M-vertex copy costs 20-40 ms)
            n = r.num_vertices
            addr = C.cast(r.membership, C.c_void_p).value
            if n and addr:
                buf = (C.c_uint32 * n).from_address(addr)
                buf._lvn_handle = _ResultHandle(out)
                keep = True
                membership = np.frombuffer(buf, dtype=np.uint32, count=n)
            else:
                membership = np.empty(0, np.uint32)
            dev_ptr = None
        res = LouvainResult(
            membership=membership,
            num_communities=r.num_communities,
            modularity=r.modularity,
            passes=r.passes,
            aggregations=r.aggregations,
            iterations_per_pass=lst(r.iterations_per_pass),
            tolerance_per_pass=lst(r.tolerance_per_pass),
            pass_seconds=lst(r.pass_seconds),
            phase=PhaseTimes(r.local_moving, r.aggregation, r.other),
            wall_seconds=r.wall_seconds,
            vertices_per_pass=lst(r.vertices_per_pass),
            arcs_per_pass=lst(r.arcs_per_pass),
            h2d_seconds=r.h2d_seconds,
            h2d_bytes=int(r.h2d_bytes),
            d2h_seconds=r.d2h_seconds,
            stats={name: KernelStats(s.seconds, s.bytes, s.launches, s.items, s.arcs, s.gathers)
                   for name, s in zip(N.STAT_NAMES, r.stats)},
            num_shards=max(r.num_shards, 1),
            sharded_passes=r.sharded_passes,
            exchange_seconds=r.exchange_seconds,
        )
        res.levels = [np.ctypeslib.as_array(r.levels[i], (max(r.vertices_per_pass[i], 1),))[: r.vertices_per_pass[i]].copy()
                      for i in range(r.num_levels)]
        res.membership_device_ptr = dev_ptr
        if dev_ptr is not None:  # valid while the result object lives
            res._handle = _ResultHandle(out)
            keep = True
        return res
    finally:
        if not keep:
            N.lib().lvn_result_free(out)


louvain_gpu = louvain_compact


def modularity(g, membership) -> float:
    """Q of an arbitrary labelling, fp64 on the device (quality.hpp:27)."""
    m = _u32(membership)
    q = C.c_double()
    csr = g._csr()
    _check(N.lib().lvn_modularity(C.byref(csr), m.ctypes.data, N.LVN_HOST, C.byref(q)))
    return q.value


def vertex_weights(g) -> np.ndarray:
    out = np.empty(max(g.num_vertices(), 1), np.float64)
    csr = g._csr()
    _check(N.lib().lvn_vertex_weights(C.byref(csr), out.ctypes.data))
    return out[: g.num_vertices()]


def count_communities(membership) -> int:
    m = _u32(membership)
    c = C.c_uint32()
    _check(N.lib().lvn_count_communities(m.ctypes.data, len(m), N.LVN_HOST, C.byref(c)))
    return c.value


def renumber_communities(membership: np.ndarray) -> int:
    """In place, ascending old-id order; returns the count (louvain_mc.hpp:101)."""
    if membership.dtype != np.uint32 or not membership.flags.c_contiguous:
        raise TypeError("membership must be a contiguous uint32 array (renumbered in place)")
    c = C.c_uint32()
    _check(N.lib().lvn_renumber(membership.ctypes.data, len(membership), N.LVN_HOST, C.byref(c)))
    return c.value


def lookup_dendrogram(membership: np.ndarray, level) -> None:
    """membership[i] <- level[membership[i]] in place (louvain_mc.hpp:105)."""
    if membership.dtype != np.uint32 or not membership.flags.c_contiguous:
        raise TypeError("membership must be a contiguous uint32 array (updated in place)")
    lv = _u32(level)
    _check(N.lib().lvn_lookup_dendrogram(membership.ctypes.data, len(membership), lv.ctypes.data, len(lv),
                                         N.LVN_HOST))


def build_community_csr(membership, count: int):
    """(offsets u64[count+1], members u32[n]) with members ascending per community."""
    m = _u32(membership)
    off = np.empty(count + 1, np.uint64)
    mem = np.empty(max(len(m), 1), np.uint32)
    _check(N.lib().lvn_community_csr(m.ctypes.data, len(m), count, N.LVN_HOST, off.ctypes.data,
                                     mem.ctypes.data))
    return off, mem[: len(m)]


def compact_aggregate(g, membership, params: LouvainParams | None = None,
                      options: CompactOptions | None = None, canonical: bool = True) -> CsrGraph:
    """Super-vertex graph of a contiguous membership (louvain_compact.hpp:76-77);
    fp64 accumulation narrowed once to f32, rows sorted when canonical."""
    m = _u32(membership)
    p = _params(params, options)
    csr = g._csr()
    out = C.POINTER(N.lvn_graph_out)()
    _check(N.lib().lvn_aggregate(C.byref(csr), m.ctypes.data, N.LVN_HOST, int(canonical), C.byref(p),
                                 C.byref(out)))
    return _graph_out(out)


louvain_aggregate = compact_aggregate


def build_csr(num_vertices: int, sources, targets, weights=None, symmetrize: bool = True) -> CsrGraph:
    """build_csr (graph.cpp:15-87) on the device: rows sorted by target, parallel
    arcs merged in fp64 (one f32 narrowing), reverse arcs added when
    symmetrizing. Missing weights default to 1 (io.hpp). Raises ValueError for
    endpoints out of range or weights that are not finite and non-negative."""
    src = _u32(sources)
    dst = _u32(targets)
    if len(src) != len(dst):
        raise ValueError("sources and targets differ in length")
    w = np.ones(len(src)) if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    if len(w) != len(src):
        raise ValueError("weights differ in length")
    out = C.POINTER(N.lvn_graph_out)()
    _check(N.lib().lvn_build_csr(int(num_vertices), len(src), src.ctypes.data, dst.ctypes.data, w.ctypes.data,
                                 int(bool(symmetrize)), C.byref(out)))
    return _graph_out(out)


def evaluate_moves(g, membership, vertex_w, community_w, m: float, options: CompactOptions | None = None,
                   force_kernel: int = -1, live: bool = False):
    """Decision of every vertex on one fixed snapshot, nothing applied
    (compact_evaluate_move, louvain_compact.hpp:65-72, batched). live=True runs
    the engine's own ranking kernels (lvn_probe_moves) instead of the
    reference-order evaluation."""
    memb = _u32(membership)
    kw = np.ascontiguousarray(vertex_w, dtype=np.float64)
    cw = np.ascontiguousarray(community_w, dtype=np.float64)
    n = g.num_vertices()
    to = np.empty(max(n, 1), np.uint32)
    gain = np.empty(max(n, 1), np.float64)
    p = _params(None, options)
    csr = g._csr()
    fn = N.lib().lvn_probe_moves if live else N.lib().lvn_evaluate_moves
    _check(fn(C.byref(csr), memb.ctypes.data, kw.ctypes.data, cw.ctypes.data, float(m),
              C.byref(p), int(force_kernel), to.ctypes.data, gain.ctypes.data))
    return to[:n], gain[:n]


def compact_evaluate_move(g, membership, vertex_w, community_w, m: float, u: int,
                          options: CompactOptions | None = None):
    to, gain = evaluate_moves(g, membership, vertex_w, community_w, m, options)
    return int(to[u]), float(gain[u])


def launch_count() -> int:
    """Kernels launched by liblvn in this process."""
    return int(N.lib().lvn_launch_count())
