// Device-side synthetic graph construction (SURVEY 8(d) C1-C5 shapes; the
// device replacement of build_csr, graph.cpp:15-87, for unit-weight inputs):
// sample undirected edges with a counter-based hash RNG, emit both arcs as
// 64-bit (source<<32 | target) keys, drop self-loops, sort, deduplicate, and
// build the CSR (rows sorted by target, unit weights, m = arcs / 2).
//
// This is input plumbing, not the timed hot path; the key sort uses CUB's
// radix sort (library code, like cuBLAS for a plain GEMM).
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>

#include <cmath>
#include <vector>

#include "kernels.cuh"

namespace lvn {

namespace {

constexpr ull kDrop = ~0ull;

__device__ __forceinline__ u64 mix64(u64 z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double unit(u64 x) { return double(x >> 11) * (1.0 / 9007199254740992.0); }
__device__ __forceinline__ u64 below(u64 x, u64 n) {  // uniform in [0, n) from 64 random bits
  return u64((unsigned __int128)x * n >> 64);
}

__device__ __forceinline__ void emit(ull* keys, u64 e, u32 u, u32 v) {
  if (u == v) {
    keys[2 * e] = kDrop;
    keys[2 * e + 1] = kDrop;
  } else {
    keys[2 * e] = (ull(u) << 32) | v;
    keys[2 * e + 1] = (ull(v) << 32) | u;
  }
}

// Graph500 R-MAT: 2^scale vertices, quadrant (a, b, c, d) per level
__global__ void gen_rmat(ull* keys, u64 edges, u32 scale, double a, double b, double c, u64 seed) {
  for (u64 e = blockIdx.x * u64(blockDim.x) + threadIdx.x; e < edges;
       e += u64(gridDim.x) * blockDim.x) {
    u32 u = 0, v = 0;
    const u64 base = mix64(seed ^ mix64(e));
    for (u32 l = 0; l < scale; ++l) {
      const double r = unit(mix64(base + l));
      u32 bu = 0, bv = 0;
      if (r < a) {
      } else if (r < a + b) {
        bv = 1;
      } else if (r < a + b + c) {
        bu = 1;
      } else {
        bu = 1, bv = 1;
      }
      u = (u << 1) | bu;
      v = (v << 1) | bv;
    }
    emit(keys, e, u, v);
  }
}

// planted partition: u ~ U(n); v ~ U(block(u)) with probability 1 - mu, else U(n)
__global__ void gen_sbm(ull* keys, u64 edges, u64 n, u64 blocks, double mu, u64 seed) {
  const u64 bsize = n / blocks;
  for (u64 e = blockIdx.x * u64(blockDim.x) + threadIdx.x; e < edges;
       e += u64(gridDim.x) * blockDim.x) {
    const u64 r0 = mix64(seed ^ mix64(3 * e)), r1 = mix64(seed ^ mix64(3 * e + 1)),
              r2 = mix64(seed ^ mix64(3 * e + 2));
    const u64 u = below(r0, n);
    u64 v;
    if (unit(r1) < mu) {
      v = below(r2, n);
    } else {
      u64 blk = u / bsize;
      if (blk >= blocks) blk = blocks - 1;
      const u64 lo = blk * bsize, hi = (blk == blocks - 1) ? n : lo + bsize;
      v = lo + below(r2, hi - lo);
    }
    emit(keys, e, u32(u), u32(v));
  }
}

// 2-D lattice side x side, each lattice edge kept with probability p
__global__ void gen_grid(ull* keys, u64 side, double p, u64 seed) {
  const u64 horiz = side * (side - 1);
  const u64 edges = 2 * horiz;
  for (u64 e = blockIdx.x * u64(blockDim.x) + threadIdx.x; e < edges;
       e += u64(gridDim.x) * blockDim.x) {
    u64 u, v;
    if (e < horiz) {  // (r, c) - (r, c+1)
      const u64 r = e / (side - 1), c = e % (side - 1);
      u = r * side + c;
      v = u + 1;
    } else {  // (r, c) - (r+1, c)
      const u64 k = e - horiz;
      u = k;
      v = k + side;
    }
    if (unit(mix64(seed ^ mix64(e))) < p)
      emit(keys, e, u32(u), u32(v));
    else
      keys[2 * e] = keys[2 * e + 1] = kDrop;
  }
}

__global__ void gen_uniform(ull* keys, u64 edges, u64 n, u64 seed) {
  for (u64 e = blockIdx.x * u64(blockDim.x) + threadIdx.x; e < edges;
       e += u64(gridDim.x) * blockDim.x) {
    const u64 u = below(mix64(seed ^ mix64(2 * e)), n), v = below(mix64(seed ^ mix64(2 * e + 1)), n);
    emit(keys, e, u32(u), u32(v));
  }
}

// Web-crawl shape: hosts are contiguous id ranges; vertex u emits deg(u)
// (truncated power law) edges, most inside its host within a locality window
// of +-2 deg(u) ids (clipped to the host, so small hosts saturate towards
// cliques, as navigation-linked web hosts do), the rest to global
// preferential-attachment targets (low ids). Only exact IEEE operations feed
// the integer decisions (no pow/exp: the host restatement in
// oracle/gen_host.cpp reproduces every sample bit for bit).
__global__ void gen_web(ull* keys, const u64* __restrict__ eoff, u64 n, const u32* __restrict__ host_lo,
                        const u32* __restrict__ host_hi, double p_local, u64 window, u64 seed) {
  for (u64 u = blockIdx.x * u64(blockDim.x) + threadIdx.x; u < n;
       u += u64(gridDim.x) * blockDim.x) {
    const u64 e0 = eoff[u], e1 = eoff[u + 1];
    const u64 lo = host_lo[u], hi = host_hi[u];
    const u64 d = e1 - e0;
    const u64 w = d * 2 > window ? d * 2 : window;
    const double pl = p_local;
    for (u64 e = e0; e < e1; ++e) {
      const u64 r0 = mix64(seed ^ mix64(2 * e)), r1 = mix64(seed ^ mix64(2 * e + 1));
      u64 v;
      if (unit(r0) < pl) {
        const u64 a = u > lo + w ? u - w : lo;
        const u64 b = u + w + 1 < hi ? u + w + 1 : hi;
        v = a + below(r1, b - a);
      } else {
        // preferential attachment: v = n x^5, P(v) ~ v^(-0.8) over the id space
        const double x = unit(r1);
        const double x2 = __dmul_rn(x, x);
        const double x5 = __dmul_rn(__dmul_rn(x2, x2), x);
        v = u64(__dmul_rn(double(n), x5));
        if (v >= n) v = n - 1;
      }
      emit(keys, e, u32(u), u32(v));
    }
  }
}

// out-degree: inverse CDF of a discrete power law over k = 1..K by binary
// search on 53-bit integer thresholds, scaled to the requested mean
__global__ void web_degrees(u64* __restrict__ deg, u64 n, const u64* __restrict__ thr, u32 kmax,
                            double scale, u64 seed) {
  for (u64 u = blockIdx.x * u64(blockDim.x) + threadIdx.x; u < n;
       u += u64(gridDim.x) * blockDim.x) {
    const u64 x = mix64(seed ^ mix64(u)) >> 11;
    u32 lo = 0, hi = kmax - 1;  // smallest k with x < thr[k]
    while (lo < hi) {
      const u32 mid = (lo + hi) >> 1;
      if (x < thr[mid]) hi = mid; else lo = mid + 1;
    }
    const double dd = __dmul_rn(double(lo + 1), scale);
    deg[u] = u64(dd < 1.0 ? 1.0 : dd);
  }
}

// unique compaction of sorted keys in tiles of kTile keys: pass 1 counts the
// kept keys per tile, pass 2 re-derives the flags, block-scans them and places
// targets (no per-key position array, which at 4e9 keys would cost 32 GB)
constexpr int kTileT = 256, kTileI = 16;
constexpr u64 kTile = u64(kTileT) * kTileI;

__device__ __forceinline__ bool kept(const ull* keys, u64 i) {
  const ull k = keys[i];
  return k != kDrop && (i == 0 || k != keys[i - 1]);
}

__global__ void __launch_bounds__(kTileT) tile_counts(const ull* __restrict__ keys, u64 m, u32* __restrict__ cnt) {
  using Scan = cub::BlockScan<u32, kTileT>;
  __shared__ typename Scan::TempStorage tmp;
  const u64 base = u64(blockIdx.x) * kTile + u64(threadIdx.x) * kTileI;
  u32 c = 0;
#pragma unroll
  for (int j = 0; j < kTileI; ++j)
    if (base + j < m && kept(keys, base + j)) ++c;
  u32 total;
  Scan(tmp).ExclusiveSum(c, c, total);
  if (threadIdx.x == 0) cnt[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kTileT) tile_place(const ull* __restrict__ keys, u64 m,
                                                     const u64* __restrict__ toff, u32* __restrict__ tgt,
                                                     u32* __restrict__ deg) {
  using Scan = cub::BlockScan<u32, kTileT>;
  __shared__ typename Scan::TempStorage tmp;
  const u64 base = u64(blockIdx.x) * kTile + u64(threadIdx.x) * kTileI;
  u32 c = 0;
#pragma unroll
  for (int j = 0; j < kTileI; ++j)
    if (base + j < m && kept(keys, base + j)) ++c;
  u32 pos;
  Scan(tmp).ExclusiveSum(c, pos);
  u64 out = toff[blockIdx.x] + pos;
#pragma unroll
  for (int j = 0; j < kTileI; ++j) {
    if (base + j < m && kept(keys, base + j)) {
      const ull k = keys[base + j];
      tgt[out++] = u32(k);
      atomicAdd(&deg[u32(k >> 32)], 1u);
    }
  }
}

__global__ void fill_ones(float* w, u64 n) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
    w[i] = 1.0f;
}

constexpr double kWebLocal = 0.92;  // fraction of in-host (windowed) endpoints
constexpr u64 kWebWindow = 64;       // minimum half-width of the locality window
constexpr double kWebAlpha = 2.1;    // out-degree power-law exponent
constexpr u32 kWebKmax = 100000;     // largest raw out-degree
// undirected samples per vertex for a requested mean arc degree (absorbs the
// loss to self-loops and duplicates; C5: 50.6 M vertices -> 3.80 G arcs)
constexpr double kWebSamplesPerArc = 0.8615;

struct WebShape {
  std::vector<u32> host_lo, host_hi;
  std::vector<u64> thresholds;  // thresholds[k-1] = floor(2^53 P(deg <= k))
  double scale = 1.0;
};

// Host-side shape of the web graph, shared by every sample: Zipf host sizes in
// [10, 1e6] (P(size >= x) ~ 1/x) from a seeded xorshift, the discrete
// power-law CDF of the raw out-degree and its scale to the requested mean.
void web_shape(u64 n, double avg_degree, u64 seed, WebShape& ws) {
  ws.host_lo.resize(n);
  ws.host_hi.resize(n);
  u64 state = seed * 0x2545F4914F6CDD1Dull + 1;
  auto rnd = [&]() {
    state ^= state >> 12, state ^= state << 25, state ^= state >> 27;
    return double((state * 0x2545F4914F6CDD1Dull) >> 11) * (1.0 / 9007199254740992.0);
  };
  for (u64 v = 0; v < n;) {
    const double x = rnd();
    u64 size = u64(10.0 / (1.0 - x * (1.0 - 10.0 / 1e6)));
    if (size > n - v) size = n - v;
    for (u64 k = v; k < v + size; ++k) ws.host_lo[k] = u32(v), ws.host_hi[k] = u32(v + size);
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
  ws.thresholds.resize(kWebKmax);
  for (u32 k = 0; k < kWebKmax; ++k) ws.thresholds[k] = u64(cdf[k] / total * 9007199254740992.0);
  ws.thresholds[kWebKmax - 1] = u64(1) << 53;
  ws.scale = avg_degree * kWebSamplesPerArc / mean;
}

unsigned grid(u64 n) {
  return unsigned(std::max<u64>(1, std::min<u64>((n + 255) / 256, u64(sm_count()) * 32)));
}

}  // namespace

// keys: 2 * edges arc keys (some kDrop) -> CSR over n vertices
void keys_to_csr(DBuf<ull>& keys, u64 nkeys, u64 n, OwnedCsr& out, cudaStream_t s) {
  DBuf<ull> sorted(nkeys);
  const int end_bit = 32 + int(ceil_log2_u64(n ? n : 1));
  size_t tmp_bytes = 0;
  // valid keys have no bits at or above end_bit; the drop marker has all bits
  // set, so it still sorts last
  LVN_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, keys.p, sorted.p, nkeys, 0, end_bit, s));
  {
    DBuf<unsigned char> tmp(tmp_bytes);
    LVN_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, keys.p, sorted.p, nkeys, 0, end_bit, s));
    LVN_CUDA(cudaStreamSynchronize(s));
  }
  keys.release();
  const u64 tiles = (nkeys + kTile - 1) / kTile;
  DBuf<u32> cnt(tiles ? tiles : 1);
  DBuf<u64> toff(tiles + 1);
  if (tiles) {
    tile_counts<<<unsigned(tiles), kTileT, 0, s>>>(sorted.p, nkeys, cnt.p);
    LVN_LAUNCH();
  }
  exclusive_scan_u32_to_u64(cnt.p, toff.p, tiles, s);
  u64 arcs = 0;
  LVN_CUDA(cudaMemcpyAsync(&arcs, toff.p + tiles, sizeof(u64), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  out.n = u32(n);
  out.arcs = arcs;
  out.tgt.alloc(arcs ? arcs : 1);
  out.w.alloc(arcs ? arcs : 1);
  out.off.alloc(n + 1);
  DBuf<u32> deg(n ? n : 1);
  LVN_CUDA(cudaMemsetAsync(deg.p, 0, (n ? n : 1) * sizeof(u32), s));
  if (tiles) {
    tile_place<<<unsigned(tiles), kTileT, 0, s>>>(sorted.p, nkeys, toff.p, out.tgt.p, deg.p);
    LVN_LAUNCH();
  }
  sorted.release();
  exclusive_scan_u32_to_u64(deg.p, out.off.p, n, s);
  fill_ones<<<grid(arcs), 256, 0, s>>>(out.w.p, arcs);
  LVN_LAUNCH();
  out.total_weight = double(arcs) / 2.0;
  LVN_CUDA(cudaStreamSynchronize(s));
}

void generate(const GenSpec& g, OwnedCsr& out, cudaStream_t s) {
  u64 n = g.n, edges = g.edges;
  DBuf<ull> keys;
  switch (g.kind) {
    case 0: {  // RMAT
      if (g.scale == 0 || g.scale > 31) fail(kInvalid, "rmat scale must be in 1..31");
      n = u64(1) << g.scale;
      keys.alloc(2 * edges);
      gen_rmat<<<grid(edges), 256, 0, s>>>(keys.p, edges, g.scale, g.a, g.b, g.c, g.seed);
      break;
    }
    case 1: {  // SBM
      if (!n || !g.blocks || g.blocks > n) fail(kInvalid, "sbm needs 1 <= blocks <= n");
      keys.alloc(2 * edges);
      gen_sbm<<<grid(edges), 256, 0, s>>>(keys.p, edges, n, g.blocks, g.mu, g.seed);
      break;
    }
    case 2: {  // grid
      const u64 side = g.n;
      if (side < 2) fail(kInvalid, "grid side must be >= 2");
      n = side * side;
      edges = 2 * side * (side - 1);
      keys.alloc(2 * edges);
      gen_grid<<<grid(edges), 256, 0, s>>>(keys.p, side, g.p, g.seed);
      break;
    }
    case 3: {  // web
      if (n < 16) fail(kInvalid, "web graph needs n >= 16");
      WebShape ws;
      web_shape(n, g.avg_degree, g.seed, ws);
      DBuf<u32> dlo(n), dhi(n);
      DBuf<u64> thr(ws.thresholds.size());
      LVN_CUDA(cudaMemcpyAsync(dlo.p, ws.host_lo.data(), n * 4, cudaMemcpyHostToDevice, s));
      LVN_CUDA(cudaMemcpyAsync(dhi.p, ws.host_hi.data(), n * 4, cudaMemcpyHostToDevice, s));
      LVN_CUDA(cudaMemcpyAsync(thr.p, ws.thresholds.data(), ws.thresholds.size() * 8, cudaMemcpyHostToDevice, s));
      DBuf<u64> deg(n), eoff(n + 1);
      web_degrees<<<grid(n), 256, 0, s>>>(deg.p, n, thr.p, u32(ws.thresholds.size()), ws.scale, g.seed + 7);
      LVN_LAUNCH();
      exclusive_scan_u64(deg.p, eoff.p, n, s);
      LVN_CUDA(cudaMemcpyAsync(&edges, eoff.p + n, sizeof(u64), cudaMemcpyDeviceToHost, s));
      LVN_CUDA(cudaStreamSynchronize(s));
      keys.alloc(2 * edges);
      gen_web<<<grid(n), 256, 0, s>>>(keys.p, eoff.p, n, dlo.p, dhi.p, kWebLocal, kWebWindow, g.seed);
      LVN_LAUNCH();
      LVN_CUDA(cudaStreamSynchronize(s));
      break;
    }
    case 4: {  // uniform
      if (n < 2) fail(kInvalid, "uniform graph needs n >= 2");
      keys.alloc(2 * edges);
      gen_uniform<<<grid(edges), 256, 0, s>>>(keys.p, edges, n, g.seed);
      break;
    }
    default:
      fail(kInvalid, "unknown generator kind");
  }
  LVN_LAUNCH();
  if (n >= kEmpty) fail(kInvalid, "vertex count collides with the reserved sentinel id");
  keys_to_csr(keys, 2 * edges, n, out, s);
}

}  // namespace lvn
