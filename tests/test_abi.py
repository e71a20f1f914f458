"""The C-ABI library builds, loads and exports every symbol include/lvn.h
declares; without a GPU every compute entry point fails loudly (there is no
CPU fallback). CPU only."""

import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lvn.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lvn_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("lvn_louvain", "lvn_modularity", "lvn_aggregate", "lvn_evaluate_moves", "lvn_probe_moves", "lvn_renumber",
              "lvn_lookup_dendrogram", "lvn_community_csr", "lvn_count_communities", "lvn_init",
              "lvn_finalize", "lvn_last_error", "lvn_result_free"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_2501_19004_b200 import _native

    lib = _native.lib()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_native.EXPORTS) <= set(declared_symbols())


def test_struct_layouts_match_header():
    from paper_2501_19004_b200 import _native as N

    # offsets the C compiler gives lvn.h (checked with a tiny C program)
    import subprocess
    import tempfile

    prog = r'''
#include <stddef.h>
#include <stdio.h>
#include "lvn.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu\n", sizeof(lvn_csr), sizeof(lvn_params), sizeof(lvn_result),
         sizeof(lvn_gen_params), sizeof(lvn_graph_out));
  printf("%zu %zu %zu\n", offsetof(lvn_params, value_bits), offsetof(lvn_result, stats),
         offsetof(lvn_result, membership_on_device));
  printf("%zu %zu %zu %zu\n", sizeof(lvn_comm), offsetof(lvn_comm, allgatherv),
         offsetof(lvn_params, shard_min_arcs_log2), offsetof(lvn_result, exchange_seconds));
  return 0;
}'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.run(["/usr/bin/gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout.split()
    sizes = [int(x) for x in out]
    assert sizes[:5] == [C.sizeof(N.lvn_csr), C.sizeof(N.lvn_params), C.sizeof(N.lvn_result),
                         C.sizeof(N.lvn_gen_params), C.sizeof(N.lvn_graph_out)]
    assert sizes[5] == N.lvn_params.value_bits.offset
    assert sizes[6] == N.lvn_result.stats.offset
    assert sizes[7] == N.lvn_result.membership_on_device.offset
    assert sizes[8:] == [C.sizeof(N.lvn_comm), N.lvn_comm.allgatherv.offset,
                         N.lvn_params.shard_min_arcs_log2.offset, N.lvn_result.exchange_seconds.offset]


def test_params_defaults_mirror_reference():
    from paper_2501_19004_b200 import _native as N

    p = N.lvn_params()
    N.lib().lvn_params_default(C.byref(p))
    # LouvainParams (louvain.hpp:9-18) and CompactOptions (louvain_compact.hpp:17-40)
    assert (p.max_passes, p.max_iterations) == (10, 20)
    assert (p.initial_tolerance, p.tolerance_drop, p.aggregation_tolerance) == (0.01, 10.0, 0.8)
    assert (p.thread_count, p.chunk_size, p.prune) == (0, 2048, 1)
    assert (p.pick_less_period, p.switch_move, p.switch_aggregate, p.probing, p.value_bits) == (4, 64, 128, 3, 32)


def test_no_gpu_means_loud_failure():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2501_19004_b200 as lvn

    g = lvn.CsrGraph(np.array([0, 1, 2], np.uint64), np.array([1, 0], np.uint32), np.ones(2, np.float32), 1.0)
    with pytest.raises(lvn.CudaError):
        lvn.modularity(g, [0, 1])
    with pytest.raises(lvn.CudaError):
        lvn.louvain_compact(g)


def test_cpp_facade_builds_against_reference_headers():
    """include/louvain_gpu.hpp compiles with the reference's own headers and
    links against liblvn.so; without a GPU the call fails loudly (LVN_CUDA ->
    std::runtime_error), never falling back to a CPU path."""
    import subprocess
    import tempfile

    import torch

    ref_inc = "/root/reference/proj/core/include"
    if not os.path.isdir(ref_inc):
        pytest.skip("reference headers absent (GPU box)")
    prog = r'''
#include <cstdio>
#include "louvain/graph.hpp"
#include "louvain_gpu.hpp"
int main() {
  louvain::CsrGraph g;
  g.offsets = {0, 1, 2};
  g.targets = {1, 0};
  g.weights = {1.0f, 1.0f};
  g.total_weight = 1.0;
  try {
    const auto r = louvain::louvain_gpu(g);
    std::printf("ok %u %.6f\n", r.num_communities, r.modularity);
  } catch (const std::runtime_error& e) {
    std::printf("runtime_error %s\n", e.what());
  }
  return 0;
}'''
    lib = os.path.join(ROOT, "paper_2501_19004_b200", "lib")
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "facade.cpp")
        open(src, "w").write(prog)
        exe = os.path.join(d, "facade")
        subprocess.run(["/usr/bin/g++", "-std=c++20", "-I", ref_inc, "-I", os.path.join(ROOT, "include"), src,
                        "-L", lib, "-llvn", f"-Wl,-rpath,{lib}", "-o", exe], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    if torch.cuda.is_available():
        assert out.startswith("ok 1"), out
    else:
        assert out.startswith("runtime_error"), out
