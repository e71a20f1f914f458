"""ctypes binding of liblvn.so (the C-ABI of include/lvn.h).

There is no CPU fallback: if the library is missing or cannot initialise a
B200, every call raises.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
# LVN_LIB overrides the library path (A/B timing of two builds)
LIB_PATH = os.environ.get("LVN_LIB") or os.path.join(HERE, "lib", "liblvn.so")
CSRC = os.path.join(HERE, "csrc")

LVN_HOST, LVN_DEVICE = 0, 1
STAT_NAMES = ("move", "aggregate", "renumber", "reset", "modularity")


class lvn_csr(C.Structure):
    _fields_ = [
        ("num_vertices", C.c_uint32),
        ("num_arcs", C.c_uint64),
        ("offsets", C.c_void_p),
        ("targets", C.c_void_p),
        ("weights", C.c_void_p),
        ("total_weight", C.c_double),
        ("location", C.c_int),
    ]


class lvn_graph_out(C.Structure):
    _fields_ = [
        ("num_vertices", C.c_uint32),
        ("num_arcs", C.c_uint64),
        ("offsets", C.POINTER(C.c_uint64)),
        ("targets", C.POINTER(C.c_uint32)),
        ("weights", C.POINTER(C.c_float)),
        ("total_weight", C.c_double),
    ]


class lvn_params(C.Structure):
    _fields_ = [
        ("max_passes", C.c_int),
        ("max_iterations", C.c_int),
        ("initial_tolerance", C.c_double),
        ("tolerance_drop", C.c_double),
        ("aggregation_tolerance", C.c_double),
        ("thread_count", C.c_int),
        ("chunk_size", C.c_int),
        ("prune", C.c_int),
        ("pick_less_period", C.c_int),
        ("switch_move", C.c_uint64),
        ("switch_aggregate", C.c_uint64),
        ("probing", C.c_int),
        ("value_bits", C.c_int),
        ("bin_thread_max", C.c_uint32),
        ("bin_group_max", C.c_uint32),
        ("bin_warp_max", C.c_uint32),
        ("bin_block_max", C.c_uint32),
        ("membership_on_device", C.c_int),
        ("sweep_chunk", C.c_uint32),
        ("sweep_order", C.c_int),
        ("sweep_ranges", C.c_int),
        ("singleton_rule", C.c_int),
        ("shard_min_arcs_log2", C.c_int),
        ("shard_rounds", C.c_int),
        ("keep_levels", C.c_int),
        ("first_range_arcs_log2", C.c_int),
    ]


class lvn_phase_stats(C.Structure):
    _fields_ = [
        ("seconds", C.c_double),
        ("bytes", C.c_double),
        ("launches", C.c_uint64),
        ("items", C.c_uint64),
        ("arcs", C.c_uint64),
        ("gathers", C.c_uint64),
    ]


class lvn_result(C.Structure):
    _fields_ = [
        ("membership", C.POINTER(C.c_uint32)),
        ("num_vertices", C.c_uint32),
        ("num_communities", C.c_uint32),
        ("modularity", C.c_double),
        ("passes", C.c_int),
        ("aggregations", C.c_int),
        ("iterations_per_pass", C.POINTER(C.c_int)),
        ("tolerance_per_pass", C.POINTER(C.c_double)),
        ("pass_seconds", C.POINTER(C.c_double)),
        ("vertices_per_pass", C.POINTER(C.c_uint32)),
        ("arcs_per_pass", C.POINTER(C.c_uint64)),
        ("local_moving", C.c_double),
        ("aggregation", C.c_double),
        ("other", C.c_double),
        ("wall_seconds", C.c_double),
        ("h2d_seconds", C.c_double),
        ("d2h_seconds", C.c_double),
        ("stats", lvn_phase_stats * 5),
        ("membership_on_device", C.c_int),
        ("num_shards", C.c_int),
        ("sharded_passes", C.c_int),
        ("exchange_seconds", C.c_double),
        ("num_levels", C.c_int),
        ("levels", C.POINTER(C.POINTER(C.c_uint32))),
        ("h2d_bytes", C.c_uint64),
    ]


LVN_U8, LVN_U32, LVN_U64, LVN_F64 = 0, 1, 2, 3
LVN_SUM, LVN_MAX = 0, 1
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int)
ALLGATHERV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64))
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p,
                           C.POINTER(C.c_uint64))


class lvn_comm(C.Structure):
    _fields_ = [
        ("rank", C.c_int),
        ("size", C.c_int),
        ("user", C.c_void_p),
        ("allreduce", ALLREDUCE_FN),
        ("allgatherv", ALLGATHERV_FN),
        ("alltoallv", ALLTOALLV_FN),
    ]


class lvn_gen_params(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("n", C.c_uint64),
        ("edges", C.c_uint64),
        ("scale", C.c_uint32),
        ("blocks", C.c_uint32),
        ("a", C.c_double),
        ("b", C.c_double),
        ("c", C.c_double),
        ("mu", C.c_double),
        ("p", C.c_double),
        ("avg_degree", C.c_double),
        ("seed", C.c_uint64),
    ]


# every symbol include/lvn.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "lvn_init", "lvn_finalize", "lvn_last_error", "lvn_version", "lvn_params_default",
    "lvn_result_free", "lvn_graph_free", "lvn_louvain", "lvn_modularity", "lvn_vertex_weights",
    "lvn_count_communities", "lvn_renumber", "lvn_lookup_dendrogram", "lvn_community_csr",
    "lvn_aggregate", "lvn_evaluate_moves", "lvn_probe_moves", "lvn_generate", "lvn_dgraph_upload", "lvn_dgraph_view",
    "lvn_dgraph_download", "lvn_dgraph_free", "lvn_device_alloc", "lvn_device_free", "lvn_memcpy",
    "lvn_louvain_sharded", "lvn_partition_rows", "lvn_build_csr",
    "lvn_nccl_version", "lvn_nccl_unique_id", "lvn_comm_nccl_create", "lvn_comm_destroy",
)

_lib = None


def build() -> None:
    """Compile liblvn.so in-tree (nvcc, sm_100a)."""
    subprocess.run(["make", "-s", "-j8", "-C", CSRC], check=True)


def lib() -> C.CDLL:
    """Load liblvn.so; raises if it has not been built (there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `make -C {CSRC}` (or __graft_entry__.build()); "
            "the engine has no CPU fallback"
        )
    L = C.CDLL(LIB_PATH)
    vp, i = C.c_void_p, C.c_int
    L.lvn_init.argtypes = [i, C.POINTER(i)]
    L.lvn_finalize.argtypes = []
    L.lvn_last_error.restype = C.c_char_p
    L.lvn_version.restype = C.c_char_p
    L.lvn_launch_count.restype = C.c_ulonglong
    L.lvn_params_default.argtypes = [C.POINTER(lvn_params)]
    L.lvn_params_default.restype = None
    L.lvn_result_free.argtypes = [C.POINTER(lvn_result)]
    L.lvn_result_free.restype = None
    L.lvn_graph_free.argtypes = [C.POINTER(lvn_graph_out)]
    L.lvn_graph_free.restype = None
    L.lvn_louvain.argtypes = [C.POINTER(lvn_csr), C.POINTER(lvn_params), C.POINTER(C.POINTER(lvn_result))]
    if hasattr(L, "lvn_louvain_sharded"):  # absent only in older builds loaded through LVN_LIB
        L.lvn_louvain_sharded.argtypes = [C.POINTER(lvn_csr), C.POINTER(lvn_params), C.POINTER(lvn_comm),
                                          C.POINTER(C.POINTER(lvn_result))]
        L.lvn_partition_rows.argtypes = [vp, C.c_uint32, i, vp]
        L.lvn_nccl_version.argtypes = [C.POINTER(i)]
        L.lvn_nccl_unique_id.argtypes = [vp]
        L.lvn_comm_nccl_create.argtypes = [i, i, vp, C.POINTER(C.POINTER(lvn_comm))]
        L.lvn_comm_destroy.argtypes = [C.POINTER(lvn_comm)]
    L.lvn_modularity.argtypes = [C.POINTER(lvn_csr), vp, i, C.POINTER(C.c_double)]
    L.lvn_vertex_weights.argtypes = [C.POINTER(lvn_csr), vp]
    L.lvn_count_communities.argtypes = [vp, C.c_uint64, i, C.POINTER(C.c_uint32)]
    L.lvn_renumber.argtypes = [vp, C.c_uint64, i, C.POINTER(C.c_uint32)]
    L.lvn_lookup_dendrogram.argtypes = [vp, C.c_uint64, vp, C.c_uint64, i]
    L.lvn_community_csr.argtypes = [vp, C.c_uint32, C.c_uint32, i, vp, vp]
    L.lvn_aggregate.argtypes = [C.POINTER(lvn_csr), vp, i, i, C.POINTER(lvn_params),
                                C.POINTER(C.POINTER(lvn_graph_out))]
    L.lvn_build_csr.argtypes = [C.c_uint32, C.c_uint64, vp, vp, vp, i, C.POINTER(C.POINTER(lvn_graph_out))]
    L.lvn_evaluate_moves.argtypes = [C.POINTER(lvn_csr), vp, vp, vp, C.c_double, C.POINTER(lvn_params), i,
                                     vp, vp]
    L.lvn_probe_moves.argtypes = [C.POINTER(lvn_csr), vp, vp, vp, C.c_double, C.POINTER(lvn_params), i,
                                     vp, vp]
    L.lvn_generate.argtypes = [C.POINTER(lvn_gen_params), C.POINTER(vp)]
    L.lvn_dgraph_upload.argtypes = [C.POINTER(lvn_csr), C.POINTER(vp)]
    L.lvn_dgraph_view.argtypes = [vp, C.POINTER(lvn_csr)]
    L.lvn_dgraph_download.argtypes = [vp, vp, vp, vp]
    L.lvn_dgraph_free.argtypes = [vp]
    L.lvn_dgraph_free.restype = None
    L.lvn_device_alloc.argtypes = [C.c_size_t, C.POINTER(vp)]
    L.lvn_device_free.argtypes = [vp]
    L.lvn_memcpy.argtypes = [vp, vp, C.c_size_t, i]
    _lib = L
    return L


def last_error() -> str:
    return lib().lvn_last_error().decode(errors="replace")
