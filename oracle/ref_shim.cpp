// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the UNMODIFIED reference library (/root/reference/proj/core,
// compiled from its sources where they lie by oracle/Makefile into
// oracle/_ref/libref.so). It lets the Python tests, the golden-fixture script
// and bench.py's CPU-baseline leg call the reference engines through ctypes:
//   louvain_mc           proj/core/src/louvain_mc.cpp:162
//   louvain_compact      proj/core/src/louvain_compact.cpp:406
//   sequential_louvain   proj/core/src/oracle.cpp:60
//   modularity           proj/core/src/quality.cpp:30
//   louvain_aggregate    proj/core/src/louvain_mc.cpp:104
//   compact_aggregate    proj/core/src/louvain_compact.cpp:454
//   renumber/lookup      proj/core/src/louvain_mc.cpp:125,145
//   compact_evaluate_move proj/core/src/louvain_compact.cpp:413
//   hashtable_*          proj/core/include/louvain/compact_hashtable.hpp:21-159
// Only the reference's public headers are used; no reference source is copied.

#include <cstdint>
#include <cstring>
#include <exception>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include <omp.h>

#include "louvain/compact_hashtable.hpp"
#include "louvain/errors.hpp"
#include "louvain/graph.hpp"
#include "louvain/louvain.hpp"
#include "louvain/louvain_compact.hpp"
#include "louvain/louvain_mc.hpp"
#include "louvain/oracle.hpp"
#include "louvain/prefix_sum.hpp"
#include "louvain/quality.hpp"
#include "louvain/synthetic.hpp"

#include "gen_host.hpp"

using namespace louvain;

namespace {

thread_local std::string g_err;

// 0 ok, 1 invalid_argument, 2 degenerate, 3 internal, 4 overflow, 5 other
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const DegenerateGraphError& e) {
    g_err = e.what();
    return 2;
  } catch (const InternalError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::overflow_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

struct ResultBox {
  LouvainResult r;
};

LouvainParams make_params(int max_passes, int max_iterations, double initial_tolerance,
                          double tolerance_drop, double aggregation_tolerance, int thread_count,
                          int chunk_size, int prune) {
  LouvainParams p;
  p.max_passes = max_passes;
  p.max_iterations = max_iterations;
  p.initial_tolerance = initial_tolerance;
  p.tolerance_drop = tolerance_drop;
  p.aggregation_tolerance = aggregation_tolerance;
  p.thread_count = thread_count;
  p.chunk_size = chunk_size;
  p.prune = prune != 0;
  return p;
}

CompactOptions make_options(int pl_period, std::uint64_t sw_move, std::uint64_t sw_agg,
                            int probing, int value_bits) {
  CompactOptions o;
  o.pick_less.period = pl_period;
  o.switch_degrees.move = sw_move;
  o.switch_degrees.aggregate = sw_agg;
  o.probing = static_cast<Probing>(probing);
  o.value_bits = value_bits;
  return o;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_max_threads() { return omp_get_max_threads(); }

// ---- graphs: opaque CsrGraph handles -------------------------------------

void* ref_graph_from_arrays(std::uint32_t n, const std::uint64_t* offsets,
                            const std::uint32_t* targets, const float* weights,
                            double total_weight) {
  auto* g = new (std::nothrow) CsrGraph;
  if (!g) return nullptr;
  const std::uint64_t arcs = offsets[n];
  g->offsets.assign(offsets, offsets + n + 1);
  g->targets.assign(targets, targets + arcs);
  g->weights.assign(weights, weights + arcs);
  g->total_weight = total_weight;
  return g;
}

void ref_graph_free(void* h) { delete static_cast<CsrGraph*>(h); }
std::uint32_t ref_graph_n(void* h) { return static_cast<CsrGraph*>(h)->num_vertices(); }
std::uint64_t ref_graph_arcs(void* h) { return static_cast<CsrGraph*>(h)->num_arcs(); }
double ref_graph_total_weight(void* h) { return static_cast<CsrGraph*>(h)->total_weight; }
void ref_graph_export(void* h, std::uint64_t* offsets, std::uint32_t* targets, float* weights) {
  const CsrGraph& g = *static_cast<CsrGraph*>(h);
  std::memcpy(offsets, g.offsets.data(), g.offsets.size() * sizeof(std::uint64_t));
  std::memcpy(targets, g.targets.data(), g.targets.size() * sizeof(std::uint32_t));
  std::memcpy(weights, g.weights.data(), g.weights.size() * sizeof(float));
}

// build_csr over caller triples (graph.cpp:15)
int ref_build_csr(std::uint32_t n, std::uint64_t ntriples, const std::uint32_t* src,
                  const std::uint32_t* dst, const double* w, int symmetrize, void** out) {
  return guard([&] {
    EdgeList el;
    el.num_vertices = n;
    el.triples.resize(ntriples);
    for (std::uint64_t i = 0; i < ntriples; ++i) el.triples[i] = {src[i], dst[i], w[i]};
    *out = new CsrGraph(build_csr(el, symmetrize != 0));
  });
}

// ---- the GPU engine's synthetic inputs, built on the host (gen_host.cpp) ----
// kind: 0 rmat(scale, edges), 1 sbm(n, blocks, edges, mu), 2 grid(side n, p),
// 3 web(n, avg_degree), 4 uniform(n, edges). Returns a CsrGraph handle.
int ref_generate(int kind, std::uint64_t n, std::uint64_t edges, std::uint32_t scale,
                 std::uint32_t blocks, double a, double b, double c, double mu, double p,
                 double avg_degree, std::uint64_t seed, void** out) {
  return guard([&] {
    genhost::Spec s;
    s.kind = kind, s.n = n, s.edges = edges, s.scale = scale, s.blocks = blocks;
    s.a = a, s.b = b, s.c = c, s.mu = mu, s.p = p, s.avg_degree = avg_degree, s.seed = seed;
    auto* g = new CsrGraph;
    try {
      genhost::generate(s, *g);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

// ---- generators (synthetic.cpp) as EdgeList handles ------------------------

void* ref_random_edges(std::uint32_t n, std::uint64_t edges, double wmin, double wmax,
                       std::uint64_t seed, int self_loops, int integer_weights) {
  try {
    return new EdgeList(random_edges(n, edges, wmin, wmax, seed, self_loops, integer_weights));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void* ref_planted_partition(std::uint32_t n, int blocks, double p_in, double p_out,
                            std::uint64_t seed) {
  try {
    return new EdgeList(planted_partition(n, blocks, p_in, p_out, seed));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

std::uint64_t ref_edgelist_size(void* h) { return static_cast<EdgeList*>(h)->triples.size(); }
void ref_edgelist_export(void* h, std::uint32_t* src, std::uint32_t* dst, double* w) {
  const EdgeList& el = *static_cast<EdgeList*>(h);
  for (std::size_t i = 0; i < el.triples.size(); ++i) {
    src[i] = el.triples[i].source;
    dst[i] = el.triples[i].target;
    w[i] = el.triples[i].weight;
  }
}
void ref_edgelist_free(void* h) { delete static_cast<EdgeList*>(h); }

int ref_random_membership(std::uint32_t n, std::uint32_t communities, std::uint64_t seed,
                          std::uint32_t* out) {
  return guard([&] {
    const Membership m = random_membership(n, communities, seed);
    std::memcpy(out, m.data(), n * sizeof(std::uint32_t));
  });
}

// ---- quality (quality.cpp) -------------------------------------------------

int ref_modularity(void* h, const std::uint32_t* memb, double* q) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    Membership m(memb, memb + g.num_vertices());
    *q = modularity(g, m);
  });
}

int ref_community_aggregates(void* h, const std::uint32_t* memb, double* sigma_total,
                             double* sigma_internal) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    Membership m(memb, memb + g.num_vertices());
    const CommunityAggregates a = community_aggregates(g, m);
    std::memcpy(sigma_total, a.sigma_total.data(), a.sigma_total.size() * sizeof(double));
    std::memcpy(sigma_internal, a.sigma_internal.data(), a.sigma_internal.size() * sizeof(double));
  });
}

double ref_delta_modularity(double k_i_to_c, double k_i_to_d, double k_i, double sigma_c,
                            double sigma_d, double m) {
  return delta_modularity(k_i_to_c, k_i_to_d, k_i, sigma_c, sigma_d, m);
}

std::uint32_t ref_count_communities(const std::uint32_t* memb, std::uint64_t n) {
  return count_communities(Membership(memb, memb + n));
}

int ref_vertex_weights(void* h, double* out) {
  return guard([&] {
    const auto k = vertex_weights(*static_cast<CsrGraph*>(h));
    std::memcpy(out, k.data(), k.size() * sizeof(double));
  });
}

// ---- renumber / lookup (louvain_mc.cpp:125-160) -----------------------------

int ref_renumber(std::uint32_t* memb, std::uint64_t n, int threads, std::uint32_t* count) {
  return guard([&] {
    Membership m(memb, memb + n);
    *count = renumber_communities(m, threads);
    std::memcpy(memb, m.data(), n * sizeof(std::uint32_t));
  });
}

int ref_lookup(std::uint32_t* memb, std::uint64_t n, const std::uint32_t* level,
               std::uint64_t nl) {
  return guard([&] {
    Membership m(memb, memb + n);
    lookup_dendrogram(m, Membership(level, level + nl), 1);
    std::memcpy(memb, m.data(), n * sizeof(std::uint32_t));
  });
}

int ref_exclusive_scan_u64(const std::uint64_t* in, std::uint64_t n, int threads,
                           std::uint64_t* out) {
  return guard([&] {
    const auto r = exclusive_scan(std::vector<std::uint64_t>(in, in + n), threads);
    std::memcpy(out, r.data(), r.size() * sizeof(std::uint64_t));
  });
}

// ---- aggregation -----------------------------------------------------------

int ref_louvain_aggregate(void* h, const std::uint32_t* memb, int threads, void** out) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    LouvainParams p;
    p.thread_count = threads;
    *out = new CsrGraph(louvain_aggregate(g, Membership(memb, memb + g.num_vertices()), p));
  });
}

int ref_compact_aggregate(void* h, const std::uint32_t* memb, int threads, int probing,
                          int value_bits, std::uint64_t sw_agg, void** out) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    LouvainParams p;
    p.thread_count = threads;
    CompactOptions o = make_options(4, 64, sw_agg, probing, value_bits);
    *out = new CsrGraph(compact_aggregate(g, Membership(memb, memb + g.num_vertices()), p, o));
  });
}

// ---- single-vertex decisions ------------------------------------------------

int ref_compact_evaluate_move(void* h, const std::uint32_t* memb, const double* kw,
                              const double* cw, double m, std::uint32_t u, int value_bits,
                              int probing, std::uint64_t sw_move, std::uint32_t* to,
                              double* gain) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    const std::size_t n = g.num_vertices();
    const Membership mb(memb, memb + n);
    const std::vector<double> k(kw, kw + n), c(cw, cw + n);
    CompactOptions o = make_options(4, sw_move, 128, probing, value_bits);
    std::pair<CommunityId, double> r;
    if (value_bits == 64) {
      CompactSlabs<double> slabs(g.num_arcs());
      r = compact_evaluate_move<double>(g, mb, k, c, m, u, o, slabs);
    } else {
      CompactSlabs<float> slabs(g.num_arcs());
      r = compact_evaluate_move<float>(g, mb, k, c, m, u, o, slabs);
    }
    *to = r.first;
    *gain = r.second;
  });
}

// Far-KV decision (louvain_mc.hpp:46-78)
int ref_best_community(void* h, const std::uint32_t* memb, const double* kw, const double* cw,
                       double m, std::uint32_t u, std::uint32_t* to, double* gain) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    const std::size_t n = g.num_vertices();
    const Membership mb(memb, memb + n);
    const std::vector<double> k(kw, kw + n), c(cw, cw + n);
    FarKvScratch s(n);
    scan_communities(s, g, mb, u, false);
    const auto r = best_community(s, u, mb[u], k, c, m);
    *to = r.first;
    *gain = r.second;
  });
}

int ref_check_delta(void* h, const std::uint32_t* memb, std::uint32_t i, std::uint32_t target,
                    double* formula, double* direct) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    const auto r = check_delta(g, Membership(memb, memb + g.num_vertices()), i, target);
    *formula = r.first;
    *direct = r.second;
  });
}

int ref_exhaustive_best_partition(void* h, std::uint32_t* memb, double* q) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    const BestPartition b = exhaustive_best_partition(g);
    std::memcpy(memb, b.membership.data(), b.membership.size() * sizeof(std::uint32_t));
    *q = b.modularity;
  });
}

// ---- full engines ------------------------------------------------------------

// engine: 0 louvain_mc, 1 louvain_compact, 2 sequential_louvain
int ref_louvain(void* h, int engine, int max_passes, int max_iterations, double initial_tolerance,
                double tolerance_drop, double aggregation_tolerance, int thread_count,
                int chunk_size, int prune, int pl_period, std::uint64_t sw_move,
                std::uint64_t sw_agg, int probing, int value_bits, void** out) {
  return guard([&] {
    const CsrGraph& g = *static_cast<CsrGraph*>(h);
    const LouvainParams p = make_params(max_passes, max_iterations, initial_tolerance,
                                        tolerance_drop, aggregation_tolerance, thread_count,
                                        chunk_size, prune);
    auto* box = new ResultBox;
    try {
      if (engine == 0)
        box->r = louvain_mc(g, p);
      else if (engine == 1)
        box->r = louvain_compact(g, p, make_options(pl_period, sw_move, sw_agg, probing, value_bits));
      else
        box->r = sequential_louvain(g, p);
    } catch (...) {
      delete box;
      throw;
    }
    *out = box;
  });
}

void ref_result_free(void* h) { delete static_cast<ResultBox*>(h); }

// scalar fields: [num_communities, passes, aggregations]
void ref_result_ints(void* h, std::int64_t* out) {
  const LouvainResult& r = static_cast<ResultBox*>(h)->r;
  out[0] = r.num_communities;
  out[1] = r.passes;
  out[2] = r.aggregations;
}
// [modularity, wall, local_moving, aggregation, other]
void ref_result_doubles(void* h, double* out) {
  const LouvainResult& r = static_cast<ResultBox*>(h)->r;
  out[0] = r.modularity;
  out[1] = r.wall_seconds;
  out[2] = r.phase.local_moving;
  out[3] = r.phase.aggregation;
  out[4] = r.phase.other;
}
void ref_result_membership(void* h, std::uint32_t* out) {
  const LouvainResult& r = static_cast<ResultBox*>(h)->r;
  std::memcpy(out, r.membership.data(), r.membership.size() * sizeof(std::uint32_t));
}
// per-pass arrays, each `passes` long
void ref_result_passes(void* h, std::int32_t* iterations, double* tolerance, double* seconds) {
  const LouvainResult& r = static_cast<ResultBox*>(h)->r;
  for (std::size_t i = 0; i < r.iterations_per_pass.size(); ++i) {
    iterations[i] = r.iterations_per_pass[i];
    tolerance[i] = r.tolerance_per_pass[i];
    seconds[i] = i < r.pass_seconds.size() ? r.pass_seconds[i] : 0.0;
  }
}

// ---- hashtable primitives over caller arrays (compact_hashtable.hpp) ------------

int ref_next_pow2(std::uint64_t x, std::uint64_t* out) {
  return guard([&] { *out = next_pow2(x); });
}

int ref_ht_accumulate(std::uint32_t* keys, double* values, std::uint64_t p1, int probing,
                      std::uint32_t key, double value) {
  return hashtable_accumulate(make_view(keys, values, p1), static_cast<Probing>(probing), key,
                              value, false)
             ? 1
             : 0;
}

double ref_ht_get(std::uint32_t* keys, double* values, std::uint64_t p1, int probing,
                  std::uint32_t key) {
  return hashtable_get(make_view(keys, values, p1), static_cast<Probing>(probing), key);
}

void ref_ht_max(std::uint32_t* keys, double* values, std::uint64_t p1, std::uint32_t* key,
                double* value) {
  const auto r = hashtable_max(make_view(keys, values, p1));
  *key = r.first;
  *value = r.second;
}

int ref_pick_less_active(int iteration, int period) {
  return pick_less_active(iteration, period) ? 1 : 0;
}

}  // extern "C"
