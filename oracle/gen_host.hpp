// TEST INFRASTRUCTURE ONLY: host restatement of the GPU input generators
// (gen_host.cpp), compiled into oracle/_ref/libref.so.
#pragma once

#include <cstdint>

#include "louvain/graph.hpp"

namespace genhost {

using u32 = std::uint32_t;
using u64 = std::uint64_t;

// mirrors lvn_gen_params (include/lvn.h)
struct Spec {
  int kind = 0;  // 0 rmat, 1 sbm, 2 grid, 3 web, 4 uniform
  u64 n = 0, edges = 0;
  u32 scale = 0, blocks = 0;
  double a = 0.57, b = 0.19, c = 0.19, mu = 0.1, p = 0.6, avg_degree = 16.0;
  u64 seed = 1;
};

// canonical deduplicated unit-weight CSR of the spec's samples
void generate(Spec s, louvain::CsrGraph& g);

}  // namespace genhost
