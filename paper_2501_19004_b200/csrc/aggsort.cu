// Aggregation of a uniform integer-weight pass by its external arcs
// (compact_aggregate_into, louvain_compact.cpp:214-310, for the case of every
// unweighted input's first pass).
//
// With every arc weight equal to an integer w, a super-row needs only counts:
// the self-loop of community c is w x (its member arcs - its external arcs),
// and the weight to community d != c is w x (arcs from c's members into d).
// So one row pass gathers C[t] for every arc (as the external-arc count of
// the hash path does anyway), counts c's external arcs and appends each one's
// key (c, d) to a buffer; the keys are radix-sorted (2 x ceil(log2 count)
// bits) and run-length encoded, and the runs ARE the super-graph's off-diagonal
// entries, already in canonical (row, target) order; the self-loops are
// inserted at their sorted position. On a web graph after its first pass
// about a quarter of the arcs cross communities (C5: 0.95 G of 3.79 G), so
// the merge touches a fraction of the arcs and no hash table at all. Each
// warp stages its keys in shared memory and reserves global space for them
// with one atomic per ~224 keys (a single global counter per key ran at
// 95 ms on C5; 30 ms staged).
//
// Integer counts times an integer weight are exact in fp64, so every entry is
// the fp64 sum of the reference (louvain_mc.cpp:95) before the one narrowing:
// bit-exact. The path is taken when a sample says at most 40 % of the arcs
// are external (else the hash aggregation is cheaper) and falls back to it when the
// buffer overflows (the counts it made are reused for the row capacities).
#include <chrono>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>

#include <cstdio>
#include <cstdlib>

#include "kernels.cuh"

namespace lvn {
namespace {

unsigned grid_for(u64 n, int threads, int per_sm) {
  return unsigned(std::max<u64>(1, std::min<u64>((n + threads - 1) / threads, u64(sm_count()) * per_sm)));
}

// every `stride`-th arc: is it external? (its row by binary search)
__global__ void ext_sample_k(DGraph g, const u32* __restrict__ C, u64 stride, ull* __restrict__ hits) {
  ull h = 0;
  for (u64 j = blockIdx.x * u64(blockDim.x) + threadIdx.x; j * stride < g.arcs; j += u64(gridDim.x) * blockDim.x) {
    const u64 a = j * stride;
    u32 lo = 0, hi = g.n;  // last row with off[row] <= a
    while (hi - lo > 1) {
      const u32 mid = lo + (hi - lo) / 2;
      if (g.off[mid] <= a) lo = mid; else hi = mid;
    }
    h += C[g.tgt[a]] != C[lo];
  }
  h = warp_sum(h);
  if ((threadIdx.x & 31) == 0 && h) atomicAdd(hits, h);
}

// A row's arcs, G threads per row (32: a warp, kBlock: a block): count the
// external arcs into ext[c] and append their keys (c << kb | d) at *n_out
// (keys past cap are dropped; *n_out still counts them). Each warp gathers
// its keys in a shared-memory buffer and reserves global space once per
// ~224 keys: one global counter took an atomic per 32-arc round from every
// warp of the GPU and serialised the pass (C5: 95 ms)
constexpr u32 kWarpBuf = 256;

template <int G>
__global__ void __launch_bounds__(G < 256 ? 256 : G) ext_emit_k(DGraph g, const u32* __restrict__ list, u64 count,
                                                                const u32* __restrict__ C, ull* __restrict__ ext,
                                                                ull* __restrict__ keys, u64 cap, ull* __restrict__ n_out,
                                                                u32 kb) {
  constexpr int T = G < 256 ? 256 : G;
  __shared__ ull buf[T / 32][kWarpBuf];
  const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  ull* wb = buf[wid];
  u32 nb = 0;  // keys in this warp's buffer (warp-uniform)
  auto flush = [&]() {
    ull base = 0;
    if (lane == 0) base = atomicAdd(n_out, ull(nb));
    base = __shfl_sync(0xffffffffu, base, 0);
    __syncwarp();
    for (u32 j = lane; j < nb; j += 32)
      if (base + j < cap) keys[base + j] = wb[j];
    __syncwarp();
    nb = 0;
  };
  const u64 groups = u64(gridDim.x) * (blockDim.x / G);
  for (u64 i = (blockIdx.x * u64(blockDim.x) + threadIdx.x) / G; i < count; i += groups) {
    const u32 u = list[i];
    const u32 c = C[u];
    const u64 lo = g.off[u], hi = g.off[u + 1];
    ull mine = 0;
    // the trip count is uniform across each warp (ballots need every lane)
    for (u64 b0 = lo + (threadIdx.x % G) - lane; b0 < hi; b0 += G) {
      const u64 a = b0 + lane;
      u32 d = c;
      if (a < hi) d = C[__ldcs(g.tgt + a)];
      const bool x = d != c;
      const u32 m = __ballot_sync(0xffffffffu, x);
      if (!m) continue;
      if (x) wb[nb + __popc(m & ((1u << lane) - 1u))] = (ull(c) << kb) | d;
      nb += __popc(m);
      mine += __popc(m);
      if (nb > kWarpBuf - 32) flush();
    }
    if (lane == 0 && mine) atomicAdd(&ext[c], mine);
  }
  if (nb) flush();
}

__global__ void run_rows_k(const ull* __restrict__ ukeys, const u32* __restrict__ nruns_p, u32 kb, u32* __restrict__ cnt) {
  const u64 nruns = *nruns_p;
  for (u64 j = blockIdx.x * u64(blockDim.x) + threadIdx.x; j < nruns; j += u64(gridDim.x) * blockDim.x)
    atomicAdd(&cnt[u32(ukeys[j] >> kb)], 1u);
}

// row length = distinct external targets + the self-loop when c has internal arcs
__global__ void row_len_k(const u32* __restrict__ cnt, const u64* __restrict__ budget, const ull* __restrict__ ext,
                          u32 count, u32* __restrict__ len) {
  for (u64 c = blockIdx.x * u64(blockDim.x) + threadIdx.x; c < count; c += u64(gridDim.x) * blockDim.x)
    len[c] = cnt[c] + (budget[c] > ext[c] ? 1u : 0u);
}

__device__ __forceinline__ float narrow_count(double v, u32* inexact) {
  const float f = float(v);
  if (inexact && double(f) != v) *inexact = 1u;
  return f;
}

__global__ void place_runs_k(const ull* __restrict__ ukeys, const u32* __restrict__ counts,
                             const u32* __restrict__ nruns_p, u32 kb, const u64* __restrict__ off,
                             const u64* __restrict__ uoff, const u64* __restrict__ budget,
                             const ull* __restrict__ ext, float uw, u32* __restrict__ tgt, float* __restrict__ w,
                             u32* inexact) {
  const u64 nruns = *nruns_p;
  const ull mask = (ull(1) << kb) - 1;
  for (u64 j = blockIdx.x * u64(blockDim.x) + threadIdx.x; j < nruns; j += u64(gridDim.x) * blockDim.x) {
    const u32 c = u32(ukeys[j] >> kb), d = u32(ukeys[j] & mask);
    const u64 pos = off[c] + (j - uoff[c]) + ((d > c && budget[c] > ext[c]) ? 1 : 0);
    tgt[pos] = d;
    w[pos] = narrow_count(double(counts[j]) * double(uw), inexact);
  }
}

__global__ void place_self_k(const ull* __restrict__ ukeys, u32 kb, u32 count, const u64* __restrict__ off,
                             const u64* __restrict__ uoff, const u64* __restrict__ budget, const ull* __restrict__ ext,
                             float uw, u32* __restrict__ tgt, float* __restrict__ w, double* __restrict__ self64) {
  const ull mask = (ull(1) << kb) - 1;
  for (u64 c = blockIdx.x * u64(blockDim.x) + threadIdx.x; c < count; c += u64(gridDim.x) * blockDim.x) {
    const u64 internal = budget[c] - ext[c];
    if (self64) self64[c] = double(internal) * double(uw);
    if (!internal) continue;
    u64 lo = uoff[c], hi = uoff[c + 1];  // first unique entry of row c with target > c
    while (lo < hi) {
      const u64 mid = lo + (hi - lo) / 2;
      if (u32(ukeys[mid] & mask) < c) lo = mid + 1; else hi = mid;
    }
    const u64 pos = off[c] + (lo - uoff[c]);
    tgt[pos] = u32(c);
    w[pos] = float(double(internal) * double(uw));  // the self-loop keeps its fp64 value in self64
  }
}

__global__ void sum_weights_k(const float* __restrict__ w, u64 n, double* __restrict__ tw) {
  double acc = 0.0;
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
    acc += double(w[i]);
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc != 0.0) atomicAdd(tw, acc);
}

template <class T>
T read_one(const T* dev, cudaStream_t s) {
  T h;
  LVN_CUDA(cudaMemcpyAsync(&h, dev, sizeof(T), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  return h;
}

}  // namespace

bool external_arcs_few(const DGraph& g, const u32* C, double max_frac, cudaStream_t s, double* sampled) {
  if (!g.arcs) return false;
  const u64 stride = 61;  // ~1.6 % of the arcs, coprime to the usual row lengths
  DBuf<ull> hits(1);
  LVN_CUDA(cudaMemsetAsync(hits.p, 0, sizeof(ull), s));
  ext_sample_k<<<grid_for(g.arcs / stride + 1, 256, 8), 256, 0, s>>>(g, C, stride, hits.p);
  LVN_LAUNCH();
  const double frac = double(read_one(hits.p, s)) / double(g.arcs / stride + 1);
  if (const char* e = std::getenv("LVN_VERBOSE"); e && *e && *e != '0')
    std::fprintf(stderr, "[lvn] aggregate: sampled external-arc fraction %.3f (by external arcs when <= %.2f)\n", frac,
                 max_frac);
  if (sampled) *sampled = frac;
  return frac <= max_frac;
}

bool aggregate_by_external_arcs(const DGraph& g, const Bins& b, const u32* C, u32 count, const u64* budget,
                                u64* ext, u64 cap, OwnedCsr& out, u32* inexact, double* self64, cudaStream_t s) {
  const u32 kb = std::max(1u, ceil_log2_u64(u64(count) + 1));
  const bool trace = [] {
    const char* v = std::getenv("LVN_VERBOSE");
    return v && *v && *v != '0';
  }();
  const auto t0 = std::chrono::steady_clock::now();
  auto ms = [&] {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  LVN_CUDA(cudaMemsetAsync(ext, 0, size_t(count ? count : 1) * sizeof(u64), s));
  DBuf<ull> keys(cap ? cap : 1), nout(1);
  LVN_CUDA(cudaMemsetAsync(nout.p, 0, sizeof(ull), s));
  ull* e = reinterpret_cast<ull*>(ext);
  // rows of <= 1024 arcs (adjacent bins, thread .. block-short): a warp each;
  // longer rows: a block each
  const u64 small = b.start[kBinBlock] - b.start[kBinThread];
  if (small)
    ext_emit_k<32><<<grid_for(small * 32, 256, 8), 256, 0, s>>>(g, b.of(kBinThread), small, C, e, keys.p, cap,
                                                                 nout.p, kb);
  LVN_LAUNCH();
  const u64 big = b.count(kBinBlock) + b.count(kBinGlobal);
  if (big)
    ext_emit_k<512><<<unsigned(std::min<u64>(big, u64(sm_count()) * 4)), 512, 0, s>>>(g, b.of(kBinBlock), big, C, e,
                                                                                       keys.p, cap, nout.p, kb);
  LVN_LAUNCH();
  const u64 n = read_one(nout.p, s);
  if (trace)
    std::fprintf(stderr, "[lvn] aggregate by external arcs: %llu keys (cap %llu) emitted at %.1f ms\n",
                 (unsigned long long)n, (unsigned long long)cap, ms());
  if (n > cap) return false;  // the hash path takes over (ext is complete)
  // sort + run-length encode the keys: the distinct off-diagonal entries.
  // The sort ping-pongs between the key buffer and one n-key buffer (small
  // CUB scratch); the run-length encoding writes into whichever is free.
  DBuf<ull> alt(n ? n : 1);
  DBuf<u32> rcounts(n ? n : 1), nruns(1);
  LVN_CUDA(cudaMemsetAsync(nruns.p, 0, sizeof(u32), s));
  ull* ukeys = alt.p;
  if (n) {
    cub::DoubleBuffer<ull> db(keys.p, alt.p);
    size_t b1 = 0, b2 = 0;
    LVN_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b1, db, n, 0, int(2 * kb), s));
    LVN_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, b2, db.Current(), db.Alternate(), rcounts.p, nruns.p, n, s));
    DBuf<unsigned char> tmp(std::max(b1, b2));
    LVN_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, b1, db, n, 0, int(2 * kb), s));
    ukeys = db.Alternate();
    LVN_CUDA(cub::DeviceRunLengthEncode::Encode(tmp.p, b2, db.Current(), ukeys, rcounts.p, nruns.p, n, s));
    g_launches += 4;
  }
  if (ukeys == alt.p)
    keys.release();
  else
    alt.release();
  DBuf<u32> cnt(count ? count : 1), len(count ? count : 1);
  LVN_CUDA(cudaMemsetAsync(cnt.p, 0, size_t(count ? count : 1) * sizeof(u32), s));
  run_rows_k<<<grid_for(n + 1, 256, 8), 256, 0, s>>>(ukeys, nruns.p, kb, cnt.p);
  LVN_LAUNCH();
  row_len_k<<<grid_for(count, 256, 8), 256, 0, s>>>(cnt.p, budget, e, count, len.p);
  LVN_LAUNCH();
  DBuf<u64> uoff(u64(count) + 1);
  out.off.alloc(u64(count) + 1);
  exclusive_scan_u32_to_u64(len.p, out.off.p, count, s);
  exclusive_scan_u32_to_u64(cnt.p, uoff.p, count, s);
  const u64 A = read_one(out.off.p + count, s);
  const u32 runs = read_one(nruns.p, s);
  out.n = count;
  out.arcs = A;
  out.tgt.alloc(A ? A : 1);
  out.w.alloc(A ? A : 1);
  if (runs)
    place_runs_k<<<grid_for(runs, 256, 8), 256, 0, s>>>(ukeys, rcounts.p, nruns.p, kb, out.off.p, uoff.p, budget, e,
                                                        g.uw, out.tgt.p, out.w.p, inexact);
  LVN_LAUNCH();
  place_self_k<<<grid_for(count, 256, 8), 256, 0, s>>>(ukeys, kb, count, out.off.p, uoff.p, budget, e, g.uw,
                                                       out.tgt.p, out.w.p, self64);
  LVN_LAUNCH();
  DBuf<double> tw(1);
  LVN_CUDA(cudaMemsetAsync(tw.p, 0, sizeof(double), s));
  if (A) {
    sum_weights_k<<<grid_for(A, 256, 8), 256, 0, s>>>(out.w.p, A, tw.p);
    LVN_LAUNCH();
  }
  out.total_weight = read_one(tw.p, s) / 2.0;
  if (trace) std::fprintf(stderr, "[lvn] aggregate by external arcs: %u runs, done at %.1f ms\n", runs, ms());
  return true;
}

}  // namespace lvn
