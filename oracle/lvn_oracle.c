/* TEST INFRASTRUCTURE ONLY — the CPU checker for the CUDA path, never shipped.
 *
 * Plain-C restatement of the reference's Louvain hot path; see lvn_oracle.h.
 * Every function names the reference file:line (under /root/reference/proj)
 * whose behaviour it restates. Accumulation orders follow the reference's
 * sequential definitions so integer-weight results are bit-identical and
 * float-weight results match the sequential reference code exactly.
 */
#include "lvn_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------
 * Hashtable (core/include/louvain/compact_hashtable.hpp)
 * ------------------------------------------------------------------------- */

/* next_pow2: smallest power of two strictly greater than x (hpp:21-24) */
int orc_next_pow2(uint64_t x, uint64_t* out) {
  if (x >= (UINT64_C(1) << 63)) return 4;
  uint64_t p = 1;
  while (p <= x) p <<= 1;
  *out = p;
  return 0;
}

/* probe_advance (hpp:60-82): configured walk for 2*p1 attempts, then linear */
static void probe_advance(int probing, uint64_t attempt, uint64_t p1, uint64_t kmod, uint64_t* i,
                          uint64_t* stride) {
  if (attempt + 1 >= 2 * p1) {
    *i += 1;
    return;
  }
  switch (probing) {
    case ORC_LINEAR:
      *i += 1;
      break;
    case ORC_QUADRATIC:
      *i += *stride;
      *stride *= 2;
      break;
    case ORC_DOUBLE_HASH:
      *i += kmod ? kmod : 1;
      break;
    default: /* ORC_QUADRATIC_DOUBLE */
      *i += *stride;
      *stride = 2 * *stride + kmod;
      break;
  }
}

/* hashtable_accumulate, non-shared path (hpp:91-122); p2 = 2*p1+1 (hpp:41-43) */
int orc_ht_accumulate(uint32_t* keys, double* values, uint64_t p1, int probing, uint32_t key,
                      double value) {
  uint64_t i = key, stride = 1;
  const uint64_t kmod = key % (2 * p1 + 1);
  for (uint64_t attempt = 0; attempt < 3 * p1; ++attempt) {
    const uint64_t s = i % p1;
    if (keys[s] == key) {
      values[s] += value;
      return 1;
    }
    if (keys[s] == ORC_EMPTY) {
      keys[s] = key;
      values[s] += value;
      return 1;
    }
    probe_advance(probing, attempt, p1, kmod, &i, &stride);
  }
  return 0;
}

/* hashtable_get (hpp:126-139) */
double orc_ht_get(const uint32_t* keys, const double* values, uint64_t p1, int probing,
                  uint32_t key) {
  uint64_t i = key, stride = 1;
  const uint64_t kmod = key % (2 * p1 + 1);
  for (uint64_t attempt = 0; attempt < 3 * p1; ++attempt) {
    const uint64_t s = i % p1;
    if (keys[s] == key) return values[s];
    if (keys[s] == ORC_EMPTY) return 0.0;
    probe_advance(probing, attempt, p1, kmod, &i, &stride);
  }
  return 0.0;
}

/* hashtable_max: greatest value, ties to the lowest key (hpp:143-159) */
void orc_ht_max(const uint32_t* keys, const double* values, uint64_t p1, uint32_t* key,
                double* value) {
  uint32_t best_key = ORC_EMPTY;
  double best = 0.0;
  int any = 0;
  for (uint64_t s = 0; s < p1; ++s) {
    const uint32_t k = keys[s];
    if (k == ORC_EMPTY) continue;
    const double v = values[s];
    if (!any || v > best || (v == best && k < best_key)) {
      any = 1;
      best_key = k;
      best = v;
    }
  }
  *key = best_key;
  *value = any ? best : 0.0;
}

/* pick_less_active (louvain_compact.hpp:22-24) */
int orc_pick_less_active(int iteration, int period) {
  return (iteration + period / 2) % period == 0;
}

/* delta_modularity, Eq. 2 (quality.hpp:34-37) */
double orc_delta_modularity(double k_i_to_c, double k_i_to_d, double k_i, double sigma_c,
                            double sigma_d, double m) {
  return (k_i_to_c - k_i_to_d) / m - k_i * (k_i + sigma_c - sigma_d) / (2.0 * m * m);
}

/* ---------------------------------------------------------------------------
 * Plumbing
 * ------------------------------------------------------------------------- */

/* exclusive_scan_sequential: out has n+1 entries (prefix_sum.hpp:12-23) */
void orc_exclusive_scan_u64(const uint64_t* in, uint64_t n, uint64_t* out) {
  uint64_t run = 0;
  for (uint64_t i = 0; i < n; ++i) {
    out[i] = run;
    run += in[i];
  }
  out[n] = run;
}

/* vertex_weights_into: K_u = sum of row weights in double (engine_detail.cpp:33-42) */
void orc_vertex_weights(uint32_t n, const uint64_t* off, const float* w, double* out) {
  for (uint32_t v = 0; v < n; ++v) {
    double s = 0.0;
    for (uint64_t a = off[v]; a < off[v + 1]; ++a) s += (double)w[a];
    out[v] = s;
  }
}

static uint32_t max_id(const uint32_t* memb, uint64_t n) {
  uint32_t mx = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (memb[i] > mx) mx = memb[i];
  return mx;
}

/* ---------------------------------------------------------------------------
 * Quality (core/src/quality.cpp)
 * ------------------------------------------------------------------------- */

/* community_aggregates (quality.cpp:9-28); arrays sized max id + 1 */
int orc_community_aggregates(uint32_t n, const uint64_t* off, const uint32_t* tgt, const float* w,
                             const uint32_t* memb, double* sigma_total, double* sigma_internal) {
  const uint64_t width = n ? (uint64_t)max_id(memb, n) + 1 : 0;
  memset(sigma_total, 0, width * sizeof(double));
  memset(sigma_internal, 0, width * sizeof(double));
  for (uint32_t v = 0; v < n; ++v) {
    const uint32_t c = memb[v];
    for (uint64_t a = off[v]; a < off[v + 1]; ++a) {
      const double x = (double)w[a];
      sigma_total[c] += x;
      if (memb[tgt[a]] == c) sigma_internal[c] += x;
    }
  }
  return 0;
}

/* modularity (quality.cpp:30-41) */
int orc_modularity(uint32_t n, const uint64_t* off, const uint32_t* tgt, const float* w,
                   double total_weight, const uint32_t* memb, double* q) {
  if (!(total_weight > 0.0)) return 2;
  const uint64_t width = n ? (uint64_t)max_id(memb, n) + 1 : 0;
  double* st = (double*)calloc(width ? width : 1, sizeof(double));
  double* si = (double*)calloc(width ? width : 1, sizeof(double));
  if (!st || !si) {
    free(st);
    free(si);
    return 5;
  }
  orc_community_aggregates(n, off, tgt, w, memb, st, si);
  const double two_m = 2.0 * total_weight;
  double acc = 0.0;
  for (uint64_t c = 0; c < width; ++c) {
    const double fraction = st[c] / two_m;
    acc += si[c] / two_m - fraction * fraction;
  }
  free(st);
  free(si);
  *q = acc;
  return 0;
}

/* count_communities (quality.cpp:43-56) */
uint32_t orc_count_communities(const uint32_t* memb, uint64_t n) {
  if (n == 0) return 0;
  const uint64_t width = (uint64_t)max_id(memb, n) + 1;
  uint8_t* seen = (uint8_t*)calloc(width, 1);
  uint32_t count = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (!seen[memb[i]]) {
      seen[memb[i]] = 1;
      ++count;
    }
  free(seen);
  return count;
}

/* renumber_communities: ascending old-id order (louvain_mc.cpp:125-143) */
uint32_t orc_renumber(uint32_t* memb, uint64_t n) {
  if (n == 0) return 0;
  const uint64_t width = (uint64_t)max_id(memb, n) + 1;
  uint32_t* rank = (uint32_t*)calloc(width + 1, sizeof(uint32_t));
  for (uint64_t i = 0; i < n; ++i) rank[memb[i]] = 1;
  uint32_t run = 0;
  for (uint64_t c = 0; c < width; ++c) {
    const uint32_t used = rank[c];
    rank[c] = run;
    run += used;
  }
  for (uint64_t i = 0; i < n; ++i) memb[i] = rank[memb[i]];
  free(rank);
  return run;
}

/* lookup_dendrogram: memb[i] <- level[memb[i]], range-checked (louvain_mc.cpp:145-160) */
int orc_lookup(uint32_t* memb, uint64_t n, const uint32_t* level, uint64_t nl) {
  int bad = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (memb[i] >= nl) {
      bad = 1;
      continue;
    }
    memb[i] = level[memb[i]];
  }
  return bad ? 3 : 0;
}

/* ---------------------------------------------------------------------------
 * Community CSR and aggregation
 * ------------------------------------------------------------------------- */

/* build_community_csr (engine_detail.cpp:44-64) with members in ascending
 * vertex order (the canonical form of the reference's atomic-cursor scatter) */
int orc_community_csr(const uint32_t* memb, uint32_t n, uint32_t count, uint64_t* offsets,
                      uint32_t* members) {
  uint64_t* counts = (uint64_t*)calloc((uint64_t)count + 1, sizeof(uint64_t));
  for (uint32_t v = 0; v < n; ++v) {
    if (memb[v] >= count) {
      free(counts);
      return 1;
    }
    ++counts[memb[v]];
  }
  orc_exclusive_scan_u64(counts, count, offsets);
  for (uint32_t c = 0; c < count; ++c) counts[c] = offsets[c];
  for (uint32_t v = 0; v < n; ++v) members[counts[memb[v]]++] = v;
  free(counts);
  return 0;
}

/* contiguity check shared by louvain_aggregate / compact_aggregate
 * (louvain_mc.cpp:106-112, louvain_compact.cpp:457-463) */
static int contiguous_count(const uint32_t* memb, uint32_t n, uint32_t* count) {
  uint32_t c = n ? max_id(memb, n) + 1 : 0;
  if (c != orc_count_communities(memb, n)) return 1;
  *count = c;
  return 0;
}

typedef struct {
  uint32_t row, key;
  uint64_t seq;
  double w;
} trip;

static int trip_cmp(const void* a, const void* b) {
  const trip* x = (const trip*)a;
  const trip* y = (const trip*)b;
  if (x->row != y->row) return x->row < y->row ? -1 : 1;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

/* Canonical super-graph: aggregate_map (oracle.cpp:32-56) — rows in ascending
 * target order, weights accumulated in double in vertex-then-arc order and
 * narrowed to f32 once; total_weight = (sum of narrowed weights)/2. Equal to
 * louvain_aggregate (louvain_mc.cpp:65-100) up to row order. out_off has
 * count+1 entries; out_tgt/out_w need room for n_arcs entries. */
int orc_aggregate(uint32_t n, const uint64_t* off, const uint32_t* tgt, const float* w,
                  const uint32_t* memb, uint64_t* out_off, uint32_t* out_tgt, float* out_w,
                  double* out_total_weight, uint32_t* out_count) {
  uint32_t count;
  if (contiguous_count(memb, n, &count)) return 1;
  const uint64_t arcs = off[n];
  trip* t = (trip*)malloc((arcs ? arcs : 1) * sizeof(trip));
  if (!t) return 5;
  for (uint32_t u = 0; u < n; ++u)
    for (uint64_t a = off[u]; a < off[u + 1]; ++a) {
      t[a].row = memb[u];
      t[a].key = memb[tgt[a]];
      t[a].seq = a;
      t[a].w = (double)w[a];
    }
  qsort(t, arcs, sizeof(trip), trip_cmp);
  memset(out_off, 0, ((uint64_t)count + 1) * sizeof(uint64_t));
  uint64_t k = 0, o = 0;
  double arc_weight = 0.0;
  while (k < arcs) {
    const uint32_t row = t[k].row, key = t[k].key;
    double s = 0.0;
    for (; k < arcs && t[k].row == row && t[k].key == key; ++k) s += t[k].w;
    out_tgt[o] = key;
    out_w[o] = (float)s;
    ++o;
    ++out_off[row + 1];
  }
  for (uint32_t c = 0; c < count; ++c) out_off[c + 1] += out_off[c];
  for (uint64_t a = 0; a < o; ++a) arc_weight += (double)out_w[a];
  free(t);
  *out_total_weight = arc_weight / 2.0;
  *out_count = count;
  return 0;
}

/* ---------------------------------------------------------------------------
 * Per-vertex move decision
 * ------------------------------------------------------------------------- */

/* compact_evaluate_move (louvain_compact.cpp:413-445) = scan_serial (37-49) +
 * decide_serial (54-68): K_{u->c} accumulated in row order over non-self arcs
 * (an entry per scanned arc, zero weights included), gains in double, stored
 * as V (f32 when value_bits == 32), maximum with ties to the lowest id; no move
 * unless to != from and gain > 0. With value_bits == 64 this is also the Far-KV
 * decision best_community (louvain_mc.hpp:60-78) for positive weights. */
int orc_evaluate_move(uint32_t n, const uint64_t* off, const uint32_t* tgt, const float* w,
                      const uint32_t* memb, const double* kw, const double* cw, double m,
                      uint32_t u, int value_bits, uint32_t* to, double* gain) {
  if (u >= n) return 1;
  if (value_bits != 32 && value_bits != 64) return 1;
  const uint32_t from = memb[u];
  const uint64_t deg = off[u + 1] - off[u];
  *to = from;
  *gain = 0.0;
  if (deg == 0) return 0;
  uint32_t* keys = (uint32_t*)malloc(deg * sizeof(uint32_t));
  double* vd = (double*)calloc(deg, sizeof(double));
  float* vf = (float*)calloc(deg, sizeof(float));
  uint64_t live = 0;
  for (uint64_t a = off[u]; a < off[u + 1]; ++a) {
    if (tgt[a] == u) continue;
    const uint32_t c = memb[tgt[a]];
    uint64_t s = 0;
    while (s < live && keys[s] != c) ++s;
    if (s == live) keys[live++] = c;
    if (value_bits == 64)
      vd[s] += (double)w[a];
    else
      vf[s] += w[a];
  }
  double own = 0.0;
  for (uint64_t s = 0; s < live; ++s)
    if (keys[s] == from) own = value_bits == 64 ? vd[s] : (double)vf[s];
  uint32_t best_key = ORC_EMPTY;
  double best = 0.0;
  for (uint64_t s = 0; s < live; ++s) {
    const uint32_t c = keys[s];
    const double k_to_c = value_bits == 64 ? vd[s] : (double)vf[s];
    double g = orc_delta_modularity(k_to_c, own, kw[u], cw[c], cw[from], m);
    if (value_bits == 32) g = (double)(float)g;
    if (best_key == ORC_EMPTY || g > best || (g == best && c < best_key)) {
      best_key = c;
      best = g;
    }
  }
  free(keys);
  free(vd);
  free(vf);
  if (best_key == ORC_EMPTY || best_key == from || best <= 0.0) return 0;
  *to = best_key;
  *gain = best;
  return 0;
}

/* ---------------------------------------------------------------------------
 * CSR build (core/src/graph.cpp:15-87)
 * ------------------------------------------------------------------------- */

typedef struct {
  uint32_t t;
  double w;
} arcw;

static int arcw_cmp(const void* a, const void* b) {
  const arcw* x = (const arcw*)a;
  const arcw* y = (const arcw*)b;
  if (x->t != y->t) return x->t < y->t ? -1 : 1;
  return x->w < y->w ? -1 : (x->w > y->w);
}

int orc_build_csr(uint32_t n, uint64_t ntriples, const uint32_t* src, const uint32_t* dst,
                  const double* w, int symmetrize, uint64_t* out_off, uint32_t* out_tgt,
                  float* out_w, double* out_total_weight) {
  if (n >= 0xFFFFFFFFu) return 1;
  uint64_t* counts = (uint64_t*)calloc((uint64_t)n + 1, sizeof(uint64_t));
  for (uint64_t i = 0; i < ntriples; ++i) {
    if (src[i] >= n || dst[i] >= n || !isfinite(w[i]) || w[i] < 0.0) {
      free(counts);
      return 1;
    }
    ++counts[src[i]];
    if (symmetrize && src[i] != dst[i]) ++counts[dst[i]];
  }
  uint64_t* raw_off = (uint64_t*)malloc(((uint64_t)n + 1) * sizeof(uint64_t));
  orc_exclusive_scan_u64(counts, n, raw_off);
  const uint64_t raw = raw_off[n];
  arcw* arcs = (arcw*)malloc((raw ? raw : 1) * sizeof(arcw));
  for (uint32_t v = 0; v < n; ++v) counts[v] = raw_off[v];
  for (uint64_t i = 0; i < ntriples; ++i) {
    arcs[counts[src[i]]++] = (arcw){dst[i], w[i]};
    if (symmetrize && src[i] != dst[i]) arcs[counts[dst[i]]++] = (arcw){src[i], w[i]};
  }
  /* sort each row by (target, weight), merge parallel arcs in double */
  uint64_t o = 0;
  out_off[0] = 0;
  for (uint32_t v = 0; v < n; ++v) {
    const uint64_t lo = raw_off[v], hi = raw_off[v + 1];
    qsort(arcs + lo, hi - lo, sizeof(arcw), arcw_cmp);
    for (uint64_t k = lo; k < hi;) {
      const uint32_t t = arcs[k].t;
      double s = 0.0;
      for (; k < hi && arcs[k].t == t; ++k) s += arcs[k].w;
      out_tgt[o] = t;
      out_w[o] = (float)s;
      ++o;
    }
    out_off[v + 1] = o;
  }
  double arc_weight = 0.0;
  for (uint64_t a = 0; a < o; ++a) arc_weight += (double)out_w[a];
  *out_total_weight = arc_weight / 2.0;
  free(arcs);
  free(raw_off);
  free(counts);
  return 0;
}

/* ---------------------------------------------------------------------------
 * Sequential Louvain (core/src/oracle.cpp:60-174)
 * ------------------------------------------------------------------------- */

typedef struct {
  uint32_t c;
  uint64_t seq;
  double w;
} link;

static int link_cmp(const void* a, const void* b) {
  const link* x = (const link*)a;
  const link* y = (const link*)b;
  if (x->c != y->c) return x->c < y->c ? -1 : 1;
  return x->seq < y->seq ? -1 : (x->seq > y->seq);
}

typedef struct {
  uint32_t n;
  uint64_t* off;
  uint32_t* tgt;
  float* w;
} owned_csr;

int orc_sequential_louvain(uint32_t n, const uint64_t* off0, const uint32_t* tgt0,
                           const float* w0, double total_weight, const orc_params* p,
                           uint32_t* global, uint32_t* num_communities, double* modularity,
                           int* passes, int* aggregations, int* iterations_per_pass,
                           double* tolerance_per_pass) {
  if (p->max_passes < 0 || p->max_iterations < 0 || !(p->tolerance_drop > 0.0) ||
      !(p->aggregation_tolerance > 0.0))
    return 1;
  if (!(total_weight > 0.0)) return 2;
  const double m = total_weight;
  for (uint32_t v = 0; v < n; ++v) global[v] = v;
  *passes = 0;
  *aggregations = 0;

  owned_csr owned = {0, NULL, NULL, NULL};
  uint32_t cn = n;
  const uint64_t* off = off0;
  const uint32_t* tgt = tgt0;
  const float* w = w0;
  double tolerance = p->initial_tolerance;

  double* kw = (double*)malloc(((uint64_t)n + 1) * sizeof(double));
  double* cw = (double*)malloc(((uint64_t)n + 1) * sizeof(double));
  uint32_t* local = (uint32_t*)malloc(((uint64_t)n + 1) * sizeof(uint32_t));
  uint8_t* unprocessed = (uint8_t*)malloc((uint64_t)n + 1);
  link* links = NULL;
  uint64_t links_cap = 0;

  for (int pass = 0; pass < p->max_passes; ++pass) {
    orc_vertex_weights(cn, off, w, kw); /* oracle.cpp:84-86 */
    memcpy(cw, kw, cn * sizeof(double));
    for (uint32_t v = 0; v < cn; ++v) local[v] = v;
    memset(unprocessed, 1, cn);

    int iterations = 0;
    for (int it = 0; it < p->max_iterations; ++it) { /* oracle.cpp:94-124 */
      double gain_total = 0.0;
      for (uint32_t u = 0; u < cn; ++u) {
        if (p->prune && !unprocessed[u]) continue;
        unprocessed[u] = 0;
        /* scan_map (oracle.cpp:20-30): ascending community order, sums in row order */
        const uint64_t deg = off[u + 1] - off[u];
        if (deg > links_cap) {
          links_cap = deg;
          links = (link*)realloc(links, links_cap * sizeof(link));
        }
        uint64_t nl = 0;
        for (uint64_t a = off[u]; a < off[u + 1]; ++a) {
          if (tgt[a] == u) continue;
          links[nl].c = local[tgt[a]];
          links[nl].seq = a;
          links[nl].w = (double)w[a];
          ++nl;
        }
        qsort(links, nl, sizeof(link), link_cmp);
        const uint32_t from = local[u];
        double to_own = 0.0;
        for (uint64_t k = 0; k < nl;) {
          const uint32_t c = links[k].c;
          double s = 0.0;
          for (; k < nl && links[k].c == c; ++k) s += links[k].w;
          if (c == from) to_own = s;
        }
        uint32_t best = from;
        double best_gain = 0.0;
        for (uint64_t k = 0; k < nl;) {
          const uint32_t c = links[k].c;
          double s = 0.0;
          for (; k < nl && links[k].c == c; ++k) s += links[k].w;
          if (c == from) continue;
          const double g = orc_delta_modularity(s, to_own, kw[u], cw[c], cw[from], m);
          if (g > best_gain) { /* ascending keys: first strict max has the lowest id */
            best = c;
            best_gain = g;
          }
        }
        if (best == from || best_gain <= 0.0) continue;
        cw[from] -= kw[u];
        cw[best] += kw[u];
        local[u] = best;
        gain_total += best_gain;
        if (p->prune)
          for (uint64_t a = off[u]; a < off[u + 1]; ++a) unprocessed[tgt[a]] = 1;
      }
      ++iterations;
      if (gain_total <= tolerance) break;
    }
    iterations_per_pass[*passes] = iterations;
    tolerance_per_pass[*passes] = tolerance;
    ++*passes;

    if (iterations <= 1) { /* oracle.cpp:134-138 */
      for (uint32_t v = 0; v < n; ++v) global[v] = local[global[v]];
      break;
    }
    const uint32_t count = orc_count_communities(local, cn);
    if ((double)count / cn > p->aggregation_tolerance) { /* oracle.cpp:141-145 */
      for (uint32_t v = 0; v < n; ++v) global[v] = local[global[v]];
      break;
    }
    orc_renumber(local, cn);
    for (uint32_t v = 0; v < n; ++v) global[v] = local[global[v]];

    /* aggregate_map (oracle.cpp:32-56) */
    owned_csr next;
    next.n = count;
    next.off = (uint64_t*)malloc(((uint64_t)count + 1) * sizeof(uint64_t));
    next.tgt = (uint32_t*)malloc((off[cn] ? off[cn] : 1) * sizeof(uint32_t));
    next.w = (float*)malloc((off[cn] ? off[cn] : 1) * sizeof(float));
    double tw;
    uint32_t cc;
    int rc = orc_aggregate(cn, off, tgt, w, local, next.off, next.tgt, next.w, &tw, &cc);
    free(owned.off);
    free(owned.tgt);
    free(owned.w);
    owned = next;
    if (rc) {
      free(kw), free(cw), free(local), free(unprocessed), free(links);
      free(owned.off), free(owned.tgt), free(owned.w);
      return 3;
    }
    cn = count;
    off = owned.off;
    tgt = owned.tgt;
    w = owned.w;
    ++*aggregations;
    tolerance /= p->tolerance_drop;
  }

  *num_communities = orc_renumber(global, n); /* oracle.cpp:160-166 */
  free(kw), free(cw), free(local), free(unprocessed), free(links);
  free(owned.off), free(owned.tgt), free(owned.w);
  return orc_modularity(n, off0, tgt0, w0, total_weight, global, modularity);
}

/* ---------------------------------------------------------------------------
 * Test-graph sampler (shape of synthetic.cpp:28-47 random_edges, different RNG)
 * ------------------------------------------------------------------------- */

static uint64_t splitmix64(uint64_t* s) {
  uint64_t z = (*s += UINT64_C(0x9E3779B97F4A7C15));
  z = (z ^ (z >> 30)) * UINT64_C(0xBF58476D1CE4E5B9);
  z = (z ^ (z >> 27)) * UINT64_C(0x94D049BB133111EB);
  return z ^ (z >> 31);
}

void orc_random_triples(uint32_t n, uint64_t count, double wmin, double wmax, uint64_t seed,
                        int self_loops, int integer_weights, uint32_t* src, uint32_t* dst,
                        double* w) {
  uint64_t s = seed;
  for (uint64_t e = 0; e < count; ++e) {
    uint32_t u = (uint32_t)(splitmix64(&s) % n);
    uint32_t v = (uint32_t)(splitmix64(&s) % n);
    while (!self_loops && u == v && n > 1) v = (uint32_t)(splitmix64(&s) % n);
    const double unit = (double)(splitmix64(&s) >> 11) * (1.0 / 9007199254740992.0);
    double x = wmin + (wmax - wmin) * (1.0 - unit);
    if (integer_weights) x = ceil(x);
    src[e] = u;
    dst[e] = v;
    w[e] = x;
  }
}
