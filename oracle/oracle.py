"""ctypes bindings for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

See ``oracle/__init__.py``. Arrays are numpy; graphs are any object with
``offsets`` (u64[n+1]), ``targets`` (u32[A]), ``weights`` (f32[A]) and
``total_weight`` (float) attributes.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref.so")
REFERENCE_SRC = "/root/reference/proj/core"

u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

PROBING = {"linear": 0, "quadratic": 1, "double_hash": 2, "quadratic_double": 3}


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"oracle rc={code} {what}")
        self.code = code


@dataclass
class Csr:
    offsets: np.ndarray
    targets: np.ndarray
    weights: np.ndarray
    total_weight: float

    @property
    def n(self) -> int:
        return len(self.offsets) - 1

    @property
    def arcs(self) -> int:
        return int(self.offsets[-1])


def build(with_ref: bool | None = None) -> None:
    """Compile the checkers (make). The reference build needs /root/reference."""
    targets = ["oracle"]
    if with_ref is None:
        with_ref = os.path.isdir(REFERENCE_SRC)
    if with_ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, *targets], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _arr(x, dt):
    return np.ascontiguousarray(x, dtype=dt)


def _g(g):
    return (_arr(g.offsets, np.uint64), _arr(g.targets, np.uint32), _arr(g.weights, np.float32))


# --------------------------------------------------------------------------
# plain-C restatement
# --------------------------------------------------------------------------


class _OrcParams(C.Structure):
    _fields_ = [
        ("max_passes", C.c_int),
        ("max_iterations", C.c_int),
        ("initial_tolerance", C.c_double),
        ("tolerance_drop", C.c_double),
        ("aggregation_tolerance", C.c_double),
        ("prune", C.c_int),
    ]


@dataclass
class SeqResult:
    membership: np.ndarray
    num_communities: int
    modularity: float
    passes: int
    aggregations: int
    iterations_per_pass: list = field(default_factory=list)
    tolerance_per_pass: list = field(default_factory=list)


class _Port:
    def __init__(self):
        self._lib = None

    @property
    def lib(self):
        if self._lib is None:
            if not os.path.exists(PORT_SO):
                build(with_ref=False)
            L = C.CDLL(PORT_SO)
            L.orc_next_pow2.argtypes = [C.c_uint64, C.POINTER(C.c_uint64)]
            L.orc_ht_accumulate.argtypes = [u32p, f64p, C.c_uint64, C.c_int, C.c_uint32, C.c_double]
            L.orc_ht_get.argtypes = [u32p, f64p, C.c_uint64, C.c_int, C.c_uint32]
            L.orc_ht_get.restype = C.c_double
            L.orc_ht_max.argtypes = [u32p, f64p, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
            L.orc_pick_less_active.argtypes = [C.c_int, C.c_int]
            L.orc_delta_modularity.argtypes = [C.c_double] * 6
            L.orc_delta_modularity.restype = C.c_double
            L.orc_exclusive_scan_u64.argtypes = [u64p, C.c_uint64, u64p]
            L.orc_vertex_weights.argtypes = [C.c_uint32, u64p, f32p, f64p]
            L.orc_community_aggregates.argtypes = [C.c_uint32, u64p, u32p, f32p, u32p, f64p, f64p]
            L.orc_modularity.argtypes = [C.c_uint32, u64p, u32p, f32p, C.c_double, u32p, C.POINTER(C.c_double)]
            L.orc_count_communities.argtypes = [u32p, C.c_uint64]
            L.orc_count_communities.restype = C.c_uint32
            L.orc_renumber.argtypes = [u32p, C.c_uint64]
            L.orc_renumber.restype = C.c_uint32
            L.orc_lookup.argtypes = [u32p, C.c_uint64, u32p, C.c_uint64]
            L.orc_community_csr.argtypes = [u32p, C.c_uint32, C.c_uint32, u64p, u32p]
            L.orc_aggregate.argtypes = [C.c_uint32, u64p, u32p, f32p, u32p, u64p, u32p, f32p,
                                        C.POINTER(C.c_double), C.POINTER(C.c_uint32)]
            L.orc_evaluate_move.argtypes = [C.c_uint32, u64p, u32p, f32p, u32p, f64p, f64p, C.c_double,
                                            C.c_uint32, C.c_int, C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
            L.orc_build_csr.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, f64p, C.c_int, u64p, u32p, f32p,
                                        C.POINTER(C.c_double)]
            L.orc_sequential_louvain.argtypes = [C.c_uint32, u64p, u32p, f32p, C.c_double, C.POINTER(_OrcParams),
                                                 u32p, C.POINTER(C.c_uint32), C.POINTER(C.c_double),
                                                 C.POINTER(C.c_int), C.POINTER(C.c_int), i32p, f64p]
            L.orc_random_triples.argtypes = [C.c_uint32, C.c_uint64, C.c_double, C.c_double, C.c_uint64,
                                             C.c_int, C.c_int, u32p, u32p, f64p]
            self._lib = L
        return self._lib

    @staticmethod
    def _rc(rc):
        if rc:
            raise OracleError(rc)

    # hashtable ------------------------------------------------------------
    def next_pow2(self, x: int) -> int:
        out = C.c_uint64()
        self._rc(self.lib.orc_next_pow2(x, C.byref(out)))
        return out.value

    def ht_accumulate(self, keys, values, probing, key, value) -> bool:
        return bool(self.lib.orc_ht_accumulate(keys, values, len(keys), PROBING.get(probing, probing), key, value))

    def ht_get(self, keys, values, probing, key) -> float:
        return self.lib.orc_ht_get(keys, values, len(keys), PROBING.get(probing, probing), key)

    def ht_max(self, keys, values):
        k, v = C.c_uint32(), C.c_double()
        self.lib.orc_ht_max(keys, values, len(keys), C.byref(k), C.byref(v))
        return k.value, v.value

    def pick_less_active(self, it, period) -> bool:
        return bool(self.lib.orc_pick_less_active(it, period))

    def delta_modularity(self, *a) -> float:
        return self.lib.orc_delta_modularity(*a)

    # plumbing -------------------------------------------------------------
    def exclusive_scan(self, x):
        x = _arr(x, np.uint64)
        out = np.empty(len(x) + 1, np.uint64)
        self.lib.orc_exclusive_scan_u64(x, len(x), out)
        return out

    def vertex_weights(self, g):
        off, _, w = _g(g)
        out = np.empty(len(off) - 1, np.float64)
        self.lib.orc_vertex_weights(len(off) - 1, off, w, out)
        return out

    def community_aggregates(self, g, memb):
        off, tgt, w = _g(g)
        memb = _arr(memb, np.uint32)
        width = int(memb.max()) + 1 if len(memb) else 0
        st = np.zeros(max(width, 1), np.float64)
        si = np.zeros(max(width, 1), np.float64)
        self.lib.orc_community_aggregates(len(off) - 1, off, tgt, w, memb, st, si)
        return st[:width], si[:width]

    def modularity(self, g, memb) -> float:
        off, tgt, w = _g(g)
        q = C.c_double()
        self._rc(self.lib.orc_modularity(len(off) - 1, off, tgt, w, float(g.total_weight),
                                         _arr(memb, np.uint32), C.byref(q)))
        return q.value

    def count_communities(self, memb) -> int:
        memb = _arr(memb, np.uint32)
        return int(self.lib.orc_count_communities(memb, len(memb)))

    def renumber(self, memb):
        memb = _arr(memb, np.uint32).copy()
        count = self.lib.orc_renumber(memb, len(memb))
        return memb, int(count)

    def lookup(self, memb, level):
        memb = _arr(memb, np.uint32).copy()
        level = _arr(level, np.uint32)
        self._rc(self.lib.orc_lookup(memb, len(memb), level, len(level)))
        return memb

    def community_csr(self, memb, count):
        memb = _arr(memb, np.uint32)
        off = np.empty(count + 1, np.uint64)
        mem = np.empty(max(len(memb), 1), np.uint32)
        self._rc(self.lib.orc_community_csr(memb, len(memb), count, off, mem))
        return off, mem[: len(memb)]

    def aggregate(self, g, memb) -> Csr:
        off, tgt, w = _g(g)
        memb = _arr(memb, np.uint32)
        n = len(off) - 1
        count_guess = int(memb.max()) + 1 if n else 0
        oo = np.empty(count_guess + 1, np.uint64)
        ot = np.empty(max(len(tgt), 1), np.uint32)
        ow = np.empty(max(len(tgt), 1), np.float32)
        tw, cnt = C.c_double(), C.c_uint32()
        self._rc(self.lib.orc_aggregate(n, off, tgt, w, memb, oo, ot, ow, C.byref(tw), C.byref(cnt)))
        a = int(oo[cnt.value])
        return Csr(oo[: cnt.value + 1].copy(), ot[:a].copy(), ow[:a].copy(), tw.value)

    def evaluate_move(self, g, memb, kw, cw, m, u, value_bits=64):
        off, tgt, w = _g(g)
        to, gain = C.c_uint32(), C.c_double()
        self._rc(self.lib.orc_evaluate_move(len(off) - 1, off, tgt, w, _arr(memb, np.uint32),
                                            _arr(kw, np.float64), _arr(cw, np.float64), float(m), int(u),
                                            value_bits, C.byref(to), C.byref(gain)))
        return to.value, gain.value

    def build_csr(self, n, src, dst, w, symmetrize=True) -> Csr:
        src, dst, w = _arr(src, np.uint32), _arr(dst, np.uint32), _arr(w, np.float64)
        cap = max(2 * len(src), 1)
        oo = np.empty(n + 1, np.uint64)
        ot = np.empty(cap, np.uint32)
        ow = np.empty(cap, np.float32)
        tw = C.c_double()
        self._rc(self.lib.orc_build_csr(n, len(src), src, dst, w, int(symmetrize), oo, ot, ow, C.byref(tw)))
        a = int(oo[n])
        return Csr(oo, ot[:a].copy(), ow[:a].copy(), tw.value)

    def random_triples(self, n, count, wmin=1.0, wmax=1.0, seed=1, self_loops=False, integer=False):
        src = np.empty(count, np.uint32)
        dst = np.empty(count, np.uint32)
        w = np.empty(count, np.float64)
        self.lib.orc_random_triples(n, count, wmin, wmax, seed, int(self_loops), int(integer), src, dst, w)
        return src, dst, w

    def random_graph(self, n, count, wmin=1.0, wmax=1.0, seed=1, self_loops=False, integer=False) -> Csr:
        return self.build_csr(n, *self.random_triples(n, count, wmin, wmax, seed, self_loops, integer))

    def sequential_louvain(self, g, max_passes=10, max_iterations=20, initial_tolerance=0.01,
                           tolerance_drop=10.0, aggregation_tolerance=0.8, prune=True) -> SeqResult:
        off, tgt, w = _g(g)
        n = len(off) - 1
        p = _OrcParams(max_passes, max_iterations, initial_tolerance, tolerance_drop, aggregation_tolerance,
                       int(prune))
        memb = np.empty(max(n, 1), np.uint32)
        cnt, q, passes, aggs = C.c_uint32(), C.c_double(), C.c_int(), C.c_int()
        its = np.zeros(max(max_passes, 1), np.int32)
        tols = np.zeros(max(max_passes, 1), np.float64)
        self._rc(self.lib.orc_sequential_louvain(n, off, tgt, w, float(g.total_weight), C.byref(p), memb,
                                                 C.byref(cnt), C.byref(q), C.byref(passes), C.byref(aggs),
                                                 its, tols))
        k = passes.value
        return SeqResult(memb[:n], cnt.value, q.value, k, aggs.value, its[:k].tolist(), tols[:k].tolist())


# --------------------------------------------------------------------------
# the reference library itself
# --------------------------------------------------------------------------


@dataclass
class RefResult:
    membership: np.ndarray
    num_communities: int
    modularity: float
    passes: int
    aggregations: int
    iterations_per_pass: list
    tolerance_per_pass: list
    pass_seconds: list
    wall_seconds: float
    local_moving: float
    aggregation: float
    other: float


class _Ref:
    ENGINES = {"mc": 0, "compact": 1, "sequential": 2}

    def __init__(self):
        self._lib = None

    @property
    def lib(self):
        if self._lib is None:
            if not os.path.exists(REF_SO):
                if not os.path.isdir(REFERENCE_SRC):
                    raise FileNotFoundError(f"{REF_SO} missing and the reference sources are absent")
                build(with_ref=True)
            L = C.CDLL(REF_SO)
            vp = C.c_void_p
            L.ref_last_error.restype = C.c_char_p
            L.ref_graph_from_arrays.argtypes = [C.c_uint32, u64p, u32p, f32p, C.c_double]
            L.ref_graph_from_arrays.restype = vp
            L.ref_graph_free.argtypes = [vp]
            for f in ("ref_graph_n",):
                getattr(L, f).argtypes = [vp]
                getattr(L, f).restype = C.c_uint32
            L.ref_graph_arcs.argtypes = [vp]
            L.ref_graph_arcs.restype = C.c_uint64
            L.ref_graph_total_weight.argtypes = [vp]
            L.ref_graph_total_weight.restype = C.c_double
            L.ref_graph_export.argtypes = [vp, u64p, u32p, f32p]
            L.ref_generate.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32] + [C.c_double] * 6 + \
                [C.c_uint64, C.POINTER(vp)]
            L.ref_build_csr.argtypes = [C.c_uint32, C.c_uint64, u32p, u32p, f64p, C.c_int, C.POINTER(vp)]
            L.ref_random_edges.argtypes = [C.c_uint32, C.c_uint64, C.c_double, C.c_double, C.c_uint64, C.c_int,
                                           C.c_int]
            L.ref_random_edges.restype = vp
            L.ref_planted_partition.argtypes = [C.c_uint32, C.c_int, C.c_double, C.c_double, C.c_uint64]
            L.ref_planted_partition.restype = vp
            L.ref_edgelist_size.argtypes = [vp]
            L.ref_edgelist_size.restype = C.c_uint64
            L.ref_edgelist_export.argtypes = [vp, u32p, u32p, f64p]
            L.ref_edgelist_free.argtypes = [vp]
            L.ref_random_membership.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, u32p]
            L.ref_modularity.argtypes = [vp, u32p, C.POINTER(C.c_double)]
            L.ref_community_aggregates.argtypes = [vp, u32p, f64p, f64p]
            L.ref_delta_modularity.argtypes = [C.c_double] * 6
            L.ref_delta_modularity.restype = C.c_double
            L.ref_count_communities.argtypes = [u32p, C.c_uint64]
            L.ref_count_communities.restype = C.c_uint32
            L.ref_vertex_weights.argtypes = [vp, f64p]
            L.ref_renumber.argtypes = [u32p, C.c_uint64, C.c_int, C.POINTER(C.c_uint32)]
            L.ref_lookup.argtypes = [u32p, C.c_uint64, u32p, C.c_uint64]
            L.ref_exclusive_scan_u64.argtypes = [u64p, C.c_uint64, C.c_int, u64p]
            L.ref_louvain_aggregate.argtypes = [vp, u32p, C.c_int, C.POINTER(vp)]
            L.ref_compact_aggregate.argtypes = [vp, u32p, C.c_int, C.c_int, C.c_int, C.c_uint64, C.POINTER(vp)]
            L.ref_compact_evaluate_move.argtypes = [vp, u32p, f64p, f64p, C.c_double, C.c_uint32, C.c_int, C.c_int,
                                                    C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
            L.ref_best_community.argtypes = [vp, u32p, f64p, f64p, C.c_double, C.c_uint32, C.POINTER(C.c_uint32),
                                             C.POINTER(C.c_double)]
            L.ref_check_delta.argtypes = [vp, u32p, C.c_uint32, C.c_uint32, C.POINTER(C.c_double),
                                          C.POINTER(C.c_double)]
            L.ref_exhaustive_best_partition.argtypes = [vp, u32p, C.POINTER(C.c_double)]
            L.ref_louvain.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_int,
                                      C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_int, C.c_int,
                                      C.POINTER(vp)]
            L.ref_result_free.argtypes = [vp]
            L.ref_result_ints.argtypes = [vp, i64p]
            L.ref_result_doubles.argtypes = [vp, f64p]
            L.ref_result_membership.argtypes = [vp, u32p]
            L.ref_result_passes.argtypes = [vp, i32p, f64p, f64p]
            L.ref_next_pow2.argtypes = [C.c_uint64, C.POINTER(C.c_uint64)]
            L.ref_ht_accumulate.argtypes = [u32p, f64p, C.c_uint64, C.c_int, C.c_uint32, C.c_double]
            L.ref_ht_get.argtypes = [u32p, f64p, C.c_uint64, C.c_int, C.c_uint32]
            L.ref_ht_get.restype = C.c_double
            L.ref_ht_max.argtypes = [u32p, f64p, C.c_uint64, C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
            L.ref_pick_less_active.argtypes = [C.c_int, C.c_int]
            L.ref_max_threads.restype = C.c_int
            self._lib = L
        return self._lib

    def _rc(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    # graph handles ------------------------------------------------------------
    class _Handle:
        def __init__(self, lib, h):
            self.lib, self.h = lib, h

        def __del__(self):
            if self.h:
                self.lib.ref_graph_free(self.h)
                self.h = None

    def handle(self, g):
        if isinstance(g, _Ref._Handle):
            return g
        off, tgt, w = _g(g)
        h = self.lib.ref_graph_from_arrays(len(off) - 1, off, tgt, w, float(g.total_weight))
        return _Ref._Handle(self.lib, h)

    def generate(self, kind: str, seed: int = 1, **kw) -> "_Ref._Handle":
        """The GPU engine's synthetic inputs built on the host (gen_host.cpp),
        same parameters as paper_2501_19004_b200.generate; returns a graph
        handle (use n/arcs/export on it)."""
        a, b, c, mu, p, deg = 0.57, 0.19, 0.19, 0.1, 0.6, 16.0
        n = edges = scale = blocks = 0
        if kind == "rmat":
            k, scale = 0, kw["scale"]
            edges = (1 << scale) * kw.get("edgefactor", 16)
            a, b, c = kw.get("a", a), kw.get("b", b), kw.get("c", c)
        elif kind == "sbm":
            k, n, blocks = 1, kw["n"], kw["blocks"]
            edges = int(kw["n"] * kw.get("avg_degree", 32) / 2)
            mu = kw.get("mu", mu)
        elif kind == "grid":
            k, n, p = 2, kw["side"], kw.get("p", p)
        elif kind == "web":
            k, n, deg = 3, kw["n"], kw.get("avg_degree", 75.0)
        elif kind == "uniform":
            k, n, edges = 4, kw["n"], kw["edges"]
        else:
            raise ValueError(f"unknown generator {kind}")
        h = C.c_void_p()
        self._rc(self.lib.ref_generate(k, n, edges, scale, blocks, a, b, c, mu, p, deg, seed, C.byref(h)))
        return _Ref._Handle(self.lib, h.value)

    def graph_size(self, g) -> tuple[int, int]:
        """(vertices, arcs) of a graph handle"""
        return int(self.lib.ref_graph_n(g.h)), int(self.lib.ref_graph_arcs(g.h))

    def export(self, g) -> Csr:
        """copy a graph handle's CSR out (the handle stays valid)"""
        L = self.lib
        n, a = self.graph_size(g)
        off = np.empty(n + 1, np.uint64)
        tgt = np.empty(max(a, 1), np.uint32)
        w = np.empty(max(a, 1), np.float32)
        L.ref_graph_export(g.h, off, tgt, w)
        return Csr(off, tgt[:a], w[:a], L.ref_graph_total_weight(g.h))

    def _export(self, h) -> Csr:
        L = self.lib
        n, a = L.ref_graph_n(h), L.ref_graph_arcs(h)
        off = np.empty(n + 1, np.uint64)
        tgt = np.empty(max(a, 1), np.uint32)
        w = np.empty(max(a, 1), np.float32)
        L.ref_graph_export(h, off, tgt, w)
        tw = L.ref_graph_total_weight(h)
        L.ref_graph_free(h)
        return Csr(off, tgt[:a].copy(), w[:a].copy(), tw)

    def build_csr(self, n, src, dst, w, symmetrize=True) -> Csr:
        h = C.c_void_p()
        self._rc(self.lib.ref_build_csr(n, len(src), _arr(src, np.uint32), _arr(dst, np.uint32),
                                        _arr(w, np.float64), int(symmetrize), C.byref(h)))
        return self._export(h)

    def _edgelist(self, h):
        if not h:
            raise OracleError(1, self.lib.ref_last_error().decode())
        k = self.lib.ref_edgelist_size(h)
        src = np.empty(max(k, 1), np.uint32)
        dst = np.empty(max(k, 1), np.uint32)
        w = np.empty(max(k, 1), np.float64)
        self.lib.ref_edgelist_export(h, src, dst, w)
        self.lib.ref_edgelist_free(h)
        return src[:k].copy(), dst[:k].copy(), w[:k].copy()

    def random_edges(self, n, edges, wmin, wmax, seed, self_loops=False, integer=False):
        return self._edgelist(self.lib.ref_random_edges(n, edges, wmin, wmax, seed, int(self_loops), int(integer)))

    def planted_partition(self, n, blocks, p_in, p_out, seed):
        return self._edgelist(self.lib.ref_planted_partition(n, blocks, p_in, p_out, seed))

    def random_membership(self, n, communities, seed):
        out = np.empty(max(n, 1), np.uint32)
        self._rc(self.lib.ref_random_membership(n, communities, seed, out))
        return out[:n]

    # quality ----------------------------------------------------------------
    def modularity(self, g, memb) -> float:
        q = C.c_double()
        gh = self.handle(g)
        self._rc(self.lib.ref_modularity(gh.h, _arr(memb, np.uint32), C.byref(q)))
        return q.value

    def community_aggregates(self, g, memb):
        memb = _arr(memb, np.uint32)
        width = int(memb.max()) + 1 if len(memb) else 0
        st = np.zeros(max(width, 1))
        si = np.zeros(max(width, 1))
        gh = self.handle(g)
        self._rc(self.lib.ref_community_aggregates(gh.h, memb, st, si))
        return st[:width], si[:width]

    def delta_modularity(self, *a):
        return self.lib.ref_delta_modularity(*a)

    def count_communities(self, memb):
        memb = _arr(memb, np.uint32)
        return int(self.lib.ref_count_communities(memb, len(memb)))

    def vertex_weights(self, g):
        out = np.empty(max(len(g.offsets) - 1, 1))
        gh = self.handle(g)
        self._rc(self.lib.ref_vertex_weights(gh.h, out))
        return out[: len(g.offsets) - 1]

    def renumber(self, memb, threads=1):
        memb = _arr(memb, np.uint32).copy()
        cnt = C.c_uint32()
        self._rc(self.lib.ref_renumber(memb, len(memb), threads, C.byref(cnt)))
        return memb, cnt.value

    def lookup(self, memb, level):
        memb = _arr(memb, np.uint32).copy()
        level = _arr(level, np.uint32)
        self._rc(self.lib.ref_lookup(memb, len(memb), level, len(level)))
        return memb

    def exclusive_scan(self, x, threads=1):
        x = _arr(x, np.uint64)
        out = np.empty(len(x) + 1, np.uint64)
        self._rc(self.lib.ref_exclusive_scan_u64(x, len(x), threads, out))
        return out

    def louvain_aggregate(self, g, memb, threads=1) -> Csr:
        h = C.c_void_p()
        gh = self.handle(g)
        self._rc(self.lib.ref_louvain_aggregate(gh.h, _arr(memb, np.uint32), threads, C.byref(h)))
        return self._export(h)

    def compact_aggregate(self, g, memb, threads=1, probing="quadratic_double", value_bits=32,
                          switch_aggregate=128) -> Csr:
        h = C.c_void_p()
        gh = self.handle(g)
        self._rc(self.lib.ref_compact_aggregate(gh.h, _arr(memb, np.uint32), threads,
                                                PROBING[probing], value_bits, switch_aggregate, C.byref(h)))
        return self._export(h)

    def compact_evaluate_move(self, g, memb, kw, cw, m, u, value_bits=64, probing="quadratic_double",
                              switch_move=64):
        to, gain = C.c_uint32(), C.c_double()
        gh = self.handle(g)
        self._rc(self.lib.ref_compact_evaluate_move(gh.h, _arr(memb, np.uint32), _arr(kw, np.float64),
                                                    _arr(cw, np.float64), float(m), int(u), value_bits,
                                                    PROBING[probing], switch_move, C.byref(to), C.byref(gain)))
        return to.value, gain.value

    def best_community(self, g, memb, kw, cw, m, u):
        to, gain = C.c_uint32(), C.c_double()
        gh = self.handle(g)
        self._rc(self.lib.ref_best_community(gh.h, _arr(memb, np.uint32), _arr(kw, np.float64),
                                             _arr(cw, np.float64), float(m), int(u), C.byref(to), C.byref(gain)))
        return to.value, gain.value

    def check_delta(self, g, memb, i, target):
        f, d = C.c_double(), C.c_double()
        gh = self.handle(g)
        self._rc(self.lib.ref_check_delta(gh.h, _arr(memb, np.uint32), i, target, C.byref(f),
                                          C.byref(d)))
        return f.value, d.value

    def exhaustive_best_partition(self, g):
        out = np.empty(len(g.offsets) - 1, np.uint32)
        q = C.c_double()
        gh = self.handle(g)
        self._rc(self.lib.ref_exhaustive_best_partition(gh.h, out, C.byref(q)))
        return out, q.value

    def louvain(self, g, engine="mc", max_passes=10, max_iterations=20, initial_tolerance=0.01,
                tolerance_drop=10.0, aggregation_tolerance=0.8, thread_count=0, chunk_size=2048, prune=True,
                pl_period=4, switch_move=64, switch_aggregate=128, probing="quadratic_double",
                value_bits=32) -> RefResult:
        h = C.c_void_p()
        gh = self.handle(g)
        self._rc(self.lib.ref_louvain(gh.h, self.ENGINES[engine], max_passes, max_iterations, initial_tolerance,
                                      tolerance_drop, aggregation_tolerance, thread_count, chunk_size, int(prune),
                                      pl_period, switch_move, switch_aggregate, PROBING[probing], value_bits,
                                      C.byref(h)))
        L = self.lib
        ints = np.zeros(3, np.int64)
        dbl = np.zeros(5)
        L.ref_result_ints(h, ints)
        L.ref_result_doubles(h, dbl)
        n = len(g.offsets) - 1 if not isinstance(g, _Ref._Handle) else L.ref_graph_n(gh.h)
        memb = np.empty(max(n, 1), np.uint32)
        L.ref_result_membership(h, memb)
        k = int(ints[1])
        its = np.zeros(max(k, 1), np.int32)
        tols = np.zeros(max(k, 1))
        secs = np.zeros(max(k, 1))
        L.ref_result_passes(h, its, tols, secs)
        L.ref_result_free(h)
        return RefResult(memb[:n], int(ints[0]), float(dbl[0]), k, int(ints[2]), its[:k].tolist(),
                         tols[:k].tolist(), secs[:k].tolist(), float(dbl[1]), float(dbl[2]), float(dbl[3]),
                         float(dbl[4]))

    # hashtable --------------------------------------------------------------
    def next_pow2(self, x):
        out = C.c_uint64()
        self._rc(self.lib.ref_next_pow2(x, C.byref(out)))
        return out.value

    def ht_accumulate(self, keys, values, probing, key, value):
        return bool(self.lib.ref_ht_accumulate(keys, values, len(keys), PROBING.get(probing, probing), key, value))

    def ht_get(self, keys, values, probing, key):
        return self.lib.ref_ht_get(keys, values, len(keys), PROBING.get(probing, probing), key)

    def ht_max(self, keys, values):
        k, v = C.c_uint32(), C.c_double()
        self.lib.ref_ht_max(keys, values, len(keys), C.byref(k), C.byref(v))
        return k.value, v.value

    def pick_less_active(self, it, period):
        return bool(self.lib.ref_pick_less_active(it, period))

    def max_threads(self):
        return int(self.lib.ref_max_threads())


port = _Port()
ref = _Ref()
