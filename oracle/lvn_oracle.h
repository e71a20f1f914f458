/* TEST INFRASTRUCTURE ONLY — the CPU checker for the CUDA path, never shipped.
 *
 * Plain-C restatement of the reference's Louvain hot path (arXiv 2501.19004
 * reference, /root/reference/proj). Each function cites the reference
 * file:line it follows. Parity is PINNED two ways (tests/test_oracle_*.py):
 * against the golden values the reference's own tests hold (tests/golden/) and
 * against the reference library itself compiled into oracle/_ref/libref.so.
 *
 * Graphs are CSR: offsets u64[n+1], targets u32[arcs], weights f32[arcs],
 * total_weight m (graph.hpp:38-54). Return codes: 0 ok, 1 invalid argument,
 * 2 degenerate graph (m == 0), 3 internal invariant, 4 overflow.
 */
#ifndef LVN_ORACLE_H
#define LVN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_EMPTY 0xFFFFFFFFu

/* compact_hashtable.hpp:13-18 */
enum { ORC_LINEAR = 0, ORC_QUADRATIC = 1, ORC_DOUBLE_HASH = 2, ORC_QUADRATIC_DOUBLE = 3 };

int orc_next_pow2(uint64_t x, uint64_t* out);
int orc_ht_accumulate(uint32_t* keys, double* values, uint64_t p1, int probing, uint32_t key,
                      double value);
double orc_ht_get(const uint32_t* keys, const double* values, uint64_t p1, int probing,
                  uint32_t key);
void orc_ht_max(const uint32_t* keys, const double* values, uint64_t p1, uint32_t* key,
                double* value);
int orc_pick_less_active(int iteration, int period);
double orc_delta_modularity(double k_i_to_c, double k_i_to_d, double k_i, double sigma_c,
                            double sigma_d, double m);

void orc_exclusive_scan_u64(const uint64_t* in, uint64_t n, uint64_t* out);
void orc_vertex_weights(uint32_t n, const uint64_t* off, const float* w, double* out);

int orc_community_aggregates(uint32_t n, const uint64_t* off, const uint32_t* tgt, const float* w,
                             const uint32_t* memb, double* sigma_total, double* sigma_internal);
int orc_modularity(uint32_t n, const uint64_t* off, const uint32_t* tgt, const float* w,
                   double total_weight, const uint32_t* memb, double* q);
uint32_t orc_count_communities(const uint32_t* memb, uint64_t n);
uint32_t orc_renumber(uint32_t* memb, uint64_t n);
int orc_lookup(uint32_t* memb, uint64_t n, const uint32_t* level, uint64_t nl);

int orc_community_csr(const uint32_t* memb, uint32_t n, uint32_t count, uint64_t* offsets,
                      uint32_t* members);
int orc_aggregate(uint32_t n, const uint64_t* off, const uint32_t* tgt, const float* w,
                  const uint32_t* memb, uint64_t* out_off, uint32_t* out_tgt, float* out_w,
                  double* out_total_weight, uint32_t* out_count);

int orc_evaluate_move(uint32_t n, const uint64_t* off, const uint32_t* tgt, const float* w,
                      const uint32_t* memb, const double* kw, const double* cw, double m,
                      uint32_t u, int value_bits, uint32_t* to, double* gain);

int orc_build_csr(uint32_t n, uint64_t ntriples, const uint32_t* src, const uint32_t* dst,
                  const double* w, int symmetrize, uint64_t* out_off, uint32_t* out_tgt,
                  float* out_w, double* out_total_weight);

typedef struct {
  int max_passes;
  int max_iterations;
  double initial_tolerance;
  double tolerance_drop;
  double aggregation_tolerance;
  int prune;
} orc_params;

int orc_sequential_louvain(uint32_t n, const uint64_t* off, const uint32_t* tgt, const float* w,
                           double total_weight, const orc_params* p, uint32_t* membership,
                           uint32_t* num_communities, double* modularity, int* passes,
                           int* aggregations, int* iterations_per_pass,
                           double* tolerance_per_pass);

/* deterministic test-graph sampler (splitmix64; not the reference's mt19937) */
void orc_random_triples(uint32_t n, uint64_t count, double wmin, double wmax, uint64_t seed,
                        int self_loops, int integer_weights, uint32_t* src, uint32_t* dst,
                        double* w);

#ifdef __cplusplus
}
#endif
#endif
