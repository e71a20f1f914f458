// louvain_gpu.hpp — header-only C++ façade over include/lvn.h that keeps the
// reference's types, option structs and exceptions, so the reference CLI or
// tests can call the B200 engine where they call louvain_compact
// (louvain_compact.hpp:57-58). Include after the reference's headers.
#pragma once

#include <stdexcept>

#include "louvain/errors.hpp"
#include "louvain/louvain_compact.hpp"
#include "lvn.h"

namespace louvain {

inline void lvn_throw(int rc) {
  switch (rc) {
    case LVN_OK:
      return;
    case LVN_INVALID_ARGUMENT:
      throw std::invalid_argument(lvn_last_error());
    case LVN_DEGENERATE:
      throw DegenerateGraphError(lvn_last_error());
    case LVN_INTERNAL:
      throw InternalError(lvn_last_error());
    default:
      throw std::runtime_error(lvn_last_error());
  }
}

inline lvn_csr lvn_view(const CsrGraph& g) {
  return lvn_csr{g.num_vertices(), g.num_arcs(), g.offsets.data(), g.targets.data(),
                 g.weights.data(), g.total_weight, LVN_HOST};
}

inline lvn_params lvn_params_of(const LouvainParams& p, const CompactOptions& o) {
  lvn_params q;
  lvn_params_default(&q);
  q.max_passes = p.max_passes;
  q.max_iterations = p.max_iterations;
  q.initial_tolerance = p.initial_tolerance;
  q.tolerance_drop = p.tolerance_drop;
  q.aggregation_tolerance = p.aggregation_tolerance;
  q.thread_count = p.thread_count;
  q.chunk_size = p.chunk_size;
  q.prune = p.prune ? 1 : 0;
  q.pick_less_period = o.pick_less.period;
  q.switch_move = o.switch_degrees.move;
  q.switch_aggregate = o.switch_degrees.aggregate;
  q.probing = static_cast<int>(o.probing);
  q.value_bits = o.value_bits;
  return q;
}

// Drop-in for louvain_compact(g, params, options) on the B200.
inline LouvainResult louvain_gpu(const CsrGraph& g, const LouvainParams& params = {},
                                 const CompactOptions& options = {}) {
  const lvn_params q = lvn_params_of(params, options);
  const lvn_csr csr = lvn_view(g);
  lvn_result* r = nullptr;
  lvn_throw(lvn_louvain(&csr, &q, &r));
  LouvainResult out;
  out.membership.assign(r->membership, r->membership + r->num_vertices);
  out.num_communities = r->num_communities;
  out.modularity = r->modularity;
  out.passes = r->passes;
  out.aggregations = r->aggregations;
  out.iterations_per_pass.assign(r->iterations_per_pass, r->iterations_per_pass + r->passes);
  out.tolerance_per_pass.assign(r->tolerance_per_pass, r->tolerance_per_pass + r->passes);
  out.pass_seconds.assign(r->pass_seconds, r->pass_seconds + r->passes);
  out.phase.local_moving = r->local_moving;
  out.phase.aggregation = r->aggregation;
  out.phase.other = r->other;
  out.wall_seconds = r->wall_seconds;
  lvn_result_free(r);
  return out;
}

// Drop-in for modularity(g, membership) (quality.hpp:27), fp64 on the device.
inline double modularity_gpu(const CsrGraph& g, const Membership& membership) {
  const lvn_csr csr = lvn_view(g);
  double q = 0.0;
  lvn_throw(lvn_modularity(&csr, membership.data(), LVN_HOST, &q));
  return q;
}

// Drop-in for compact_aggregate(g, membership) (louvain_compact.hpp:76-77);
// rows come out sorted by target.
inline CsrGraph compact_aggregate_gpu(const CsrGraph& g, const Membership& membership,
                                      const LouvainParams& params = {},
                                      const CompactOptions& options = {}) {
  const lvn_params q = lvn_params_of(params, options);
  const lvn_csr csr = lvn_view(g);
  lvn_graph_out* o = nullptr;
  lvn_throw(lvn_aggregate(&csr, membership.data(), LVN_HOST, 1, &q, &o));
  CsrGraph out;
  out.offsets.assign(o->offsets, o->offsets + o->num_vertices + 1);
  out.targets.assign(o->targets, o->targets + o->num_arcs);
  out.weights.assign(o->weights, o->weights + o->num_arcs);
  out.total_weight = o->total_weight;
  lvn_graph_free(o);
  return out;
}

}  // namespace louvain
