"""B200-native Louvain community detection (arXiv 2501.19004 GPU hot path).

The local-moving and aggregation phases (plus renumbering, the community CSR
and an fp64 modularity reduction) run as hand-written CUDA kernels for sm_100a
in ``lib/liblvn.so``, behind the C-ABI of ``include/lvn.h``. This package is
the Python mirror of the reference's C++ interface on top of that ABI.
"""

from ._native import build  # noqa: F401
from .louvain import (  # noqa: F401
    CompactOptions,
    CsrGraph,
    CudaError,
    DegenerateGraphError,
    DeviceBins,
    DeviceGraph,
    InternalError,
    KernelStats,
    LouvainParams,
    LouvainResult,
    ParseError,
    PhaseTimes,
    PickLessSchedule,
    Probing,
    SwitchDegrees,
    build_community_csr,
    build_csr,
    compact_aggregate,
    compact_evaluate_move,
    count_communities,
    evaluate_moves,
    generate,
    launch_count,
    lookup_dendrogram,
    louvain_aggregate,
    louvain_compact,
    louvain_gpu,
    louvain_sharded,
    modularity,
    partition_rows,
    pick_less_active,
    renumber_communities,
    vertex_weights,
)
