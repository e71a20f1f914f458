// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Host (OpenMP) restatement of the synthetic input generators of the GPU
// engine (paper_2501_19004_b200/csrc/generate.cu; SURVEY.md 8(d) shapes C1-C5).
// It is compiled into oracle/_ref/libref.so next to the reference core so the
// reference arm of bench.py (`--impl reference`) builds its input graph with
// no product code mapped into its process, and so the GPU generator can be
// checked bit for bit against an independent implementation
// (tests/test_gpu_build.py).
//
// Same counter-based samples as the device kernels (splitmix64 hash of the
// sample index, 53-bit uniforms, 128-bit multiply-high ranges; only exact IEEE
// multiplies/adds feed integer decisions), same canonical CSR: both arcs of
// every non-loop sample, rows sorted by target, duplicates removed, unit
// weights, m = arcs / 2 -- the result of the reference's build_csr
// (proj/core/src/graph.cpp:15-87) on the deduplicated sample set.
//
// Build strategy (no global sort of 2E keys, which at C5 would need ~100 GB):
// count arcs per row, scan, regenerate and scatter with atomic row cursors,
// sort + unique each row, compact into the CsrGraph.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

#include <omp.h>

#include "gen_host.hpp"

namespace genhost {

inline u64 mix64(u64 z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline double unit(u64 x) { return double(x >> 11) * (1.0 / 9007199254740992.0); }
inline u64 below(u64 x, u64 n) { return u64((unsigned __int128)x * n >> 64); }

// web-shape constants (generate.cu kWeb*)
constexpr double kWebLocal = 0.92;
constexpr u64 kWebWindow = 64;
constexpr double kWebAlpha = 2.1;
constexpr u32 kWebKmax = 100000;
constexpr double kWebSamplesPerArc = 0.8615;

struct Web {
  std::vector<u32> lo, hi;
  std::vector<u64> eoff;  // samples of vertex u: [eoff[u], eoff[u+1])
};

void web_shape(const Spec& s, Web& w) {
  const u64 n = s.n;
  w.lo.resize(n);
  w.hi.resize(n);
  u64 state = s.seed * 0x2545F4914F6CDD1Dull + 1;
  auto rnd = [&]() {
    state ^= state >> 12, state ^= state << 25, state ^= state >> 27;
    return double((state * 0x2545F4914F6CDD1Dull) >> 11) * (1.0 / 9007199254740992.0);
  };
  for (u64 v = 0; v < n;) {
    const double x = rnd();
    u64 size = u64(10.0 / (1.0 - x * (1.0 - 10.0 / 1e6)));
    if (size > n - v) size = n - v;
    for (u64 k = v; k < v + size; ++k) w.lo[k] = u32(v), w.hi[k] = u32(v + size);
    v += size;
  }
  std::vector<double> cdf(kWebKmax);
  double total = 0.0, mean = 0.0;
  for (u32 k = 1; k <= kWebKmax; ++k) {
    const double pk = std::pow(double(k), -kWebAlpha);
    total += pk;
    cdf[k - 1] = total;
    mean += double(k) * pk;
  }
  mean /= total;
  std::vector<u64> thr(kWebKmax);
  for (u32 k = 0; k < kWebKmax; ++k) thr[k] = u64(cdf[k] / total * 9007199254740992.0);
  thr[kWebKmax - 1] = u64(1) << 53;
  const double scale = s.avg_degree * kWebSamplesPerArc / mean;
  w.eoff.assign(n + 1, 0);
#pragma omp parallel for schedule(static)
  for (u64 u = 0; u < n; ++u) {
    const u64 x = mix64((s.seed + 7) ^ mix64(u)) >> 11;
    const u64 k = u64(std::upper_bound(thr.begin(), thr.end(), x) - thr.begin());
    const double dd = double(k + 1) * scale;
    w.eoff[u + 1] = u64(dd < 1.0 ? 1.0 : dd);
  }
  for (u64 u = 0; u < n; ++u) w.eoff[u + 1] += w.eoff[u];
}

// Calls f(u, v) for every sample that is not dropped (u != v), in parallel.
template <class F>
void for_each_sample(const Spec& s, const Web* web, F&& f) {
  switch (s.kind) {
    case 0: {
#pragma omp parallel for schedule(static)
      for (u64 e = 0; e < s.edges; ++e) {
        u32 u = 0, v = 0;
        const u64 base = mix64(s.seed ^ mix64(e));
        for (u32 l = 0; l < s.scale; ++l) {
          const double r = unit(mix64(base + l));
          u32 bu = 0, bv = 0;
          if (r < s.a) {
          } else if (r < s.a + s.b) {
            bv = 1;
          } else if (r < s.a + s.b + s.c) {
            bu = 1;
          } else {
            bu = 1, bv = 1;
          }
          u = (u << 1) | bu;
          v = (v << 1) | bv;
        }
        if (u != v) f(u, v);
      }
      break;
    }
    case 1: {
      const u64 n = s.n, blocks = s.blocks, bsize = n / blocks;
#pragma omp parallel for schedule(static)
      for (u64 e = 0; e < s.edges; ++e) {
        const u64 r0 = mix64(s.seed ^ mix64(3 * e)), r1 = mix64(s.seed ^ mix64(3 * e + 1)),
                  r2 = mix64(s.seed ^ mix64(3 * e + 2));
        const u64 u = below(r0, n);
        u64 v;
        if (unit(r1) < s.mu) {
          v = below(r2, n);
        } else {
          u64 blk = u / bsize;
          if (blk >= blocks) blk = blocks - 1;
          const u64 lo = blk * bsize, hi = (blk == blocks - 1) ? n : lo + bsize;
          v = lo + below(r2, hi - lo);
        }
        if (u != v) f(u32(u), u32(v));
      }
      break;
    }
    case 2: {
      const u64 side = s.n, horiz = side * (side - 1), edges = 2 * horiz;
#pragma omp parallel for schedule(static)
      for (u64 e = 0; e < edges; ++e) {
        u64 u, v;
        if (e < horiz) {
          const u64 r = e / (side - 1), c = e % (side - 1);
          u = r * side + c;
          v = u + 1;
        } else {
          u = e - horiz;
          v = u + side;
        }
        if (unit(mix64(s.seed ^ mix64(e))) < s.p) f(u32(u), u32(v));
      }
      break;
    }
    case 3: {
      const u64 n = s.n;
#pragma omp parallel for schedule(dynamic, 4096)
      for (u64 u = 0; u < n; ++u) {
        const u64 e0 = web->eoff[u], e1 = web->eoff[u + 1];
        const u64 lo = web->lo[u], hi = web->hi[u];
        const u64 d = e1 - e0;
        const u64 w = d * 2 > kWebWindow ? d * 2 : kWebWindow;
        for (u64 e = e0; e < e1; ++e) {
          const u64 r0 = mix64(s.seed ^ mix64(2 * e)), r1 = mix64(s.seed ^ mix64(2 * e + 1));
          u64 v;
          if (unit(r0) < kWebLocal) {
            const u64 a = u > lo + w ? u - w : lo;
            const u64 b = u + w + 1 < hi ? u + w + 1 : hi;
            v = a + below(r1, b - a);
          } else {
            const double x = unit(r1);
            const double x2 = x * x;
            const double x5 = (x2 * x2) * x;
            v = u64(double(n) * x5);
            if (v >= n) v = n - 1;
          }
          if (u != v) f(u32(u), u32(v));
        }
      }
      break;
    }
    case 4: {
#pragma omp parallel for schedule(static)
      for (u64 e = 0; e < s.edges; ++e) {
        const u64 u = below(mix64(s.seed ^ mix64(2 * e)), s.n), v = below(mix64(s.seed ^ mix64(2 * e + 1)), s.n);
        if (u != v) f(u32(u), u32(v));
      }
      break;
    }
    default:
      throw std::invalid_argument("unknown generator kind");
  }
}

void generate(Spec s, louvain::CsrGraph& g) {
  Web web;
  switch (s.kind) {
    case 0:
      if (s.scale == 0 || s.scale > 31) throw std::invalid_argument("rmat scale must be in 1..31");
      s.n = u64(1) << s.scale;
      break;
    case 1:
      if (!s.n || !s.blocks || s.blocks > s.n) throw std::invalid_argument("sbm needs 1 <= blocks <= n");
      break;
    case 2:
      if (s.n < 2) throw std::invalid_argument("grid side must be >= 2");
      break;
    case 3:
      if (s.n < 16) throw std::invalid_argument("web graph needs n >= 16");
      web_shape(s, web);
      break;
    case 4:
      if (s.n < 2) throw std::invalid_argument("uniform graph needs n >= 2");
      break;
    default:
      throw std::invalid_argument("unknown generator kind");
  }
  const u64 n = s.kind == 2 ? s.n * s.n : s.n;
  if (n >= 0xFFFFFFFFull) throw std::invalid_argument("vertex count collides with the reserved sentinel id");

  // 1. raw arcs per row (both directions of every kept sample)
  std::vector<u64> cur(n + 1, 0);
  for_each_sample(s, &web, [&](u32 u, u32 v) {
    __atomic_fetch_add(&cur[u], 1, __ATOMIC_RELAXED);
    __atomic_fetch_add(&cur[v], 1, __ATOMIC_RELAXED);
  });
  std::vector<u64> raw(n + 1, 0);
  for (u64 u = 0; u < n; ++u) raw[u + 1] = raw[u] + cur[u];
  // 2. scatter with atomic row cursors
  std::vector<u32> tmp(raw[n]);
#pragma omp parallel for schedule(static)
  for (u64 u = 0; u < n; ++u) cur[u] = raw[u];
  for_each_sample(s, &web, [&](u32 u, u32 v) {
    tmp[__atomic_fetch_add(&cur[u], 1, __ATOMIC_RELAXED)] = v;
    tmp[__atomic_fetch_add(&cur[v], 1, __ATOMIC_RELAXED)] = u;
  });
  // 3. sort + unique per row
#pragma omp parallel for schedule(dynamic, 1024)
  for (u64 u = 0; u < n; ++u) {
    u32* b = tmp.data() + raw[u];
    u32* e = tmp.data() + raw[u + 1];
    std::sort(b, e);
    cur[u] = u64(std::unique(b, e) - b);
  }
  // 4. compact into the CSR
  g.offsets.assign(n + 1, 0);
  for (u64 u = 0; u < n; ++u) g.offsets[u + 1] = g.offsets[u] + cur[u];
  const u64 arcs = g.offsets[n];
  g.targets.resize(arcs);
#pragma omp parallel for schedule(dynamic, 1024)
  for (u64 u = 0; u < n; ++u)
    std::copy(tmp.data() + raw[u], tmp.data() + raw[u] + cur[u], g.targets.data() + g.offsets[u]);
  std::vector<u32>().swap(tmp);
  g.weights.resize(arcs);
#pragma omp parallel for schedule(static)
  for (u64 i = 0; i < arcs; ++i) g.weights[i] = 1.0f;
  g.total_weight = double(arcs) / 2.0;
}

}  // namespace genhost
