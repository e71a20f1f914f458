// Degree binning (stable multi-way partition of the rows by degree class) and
// the pass reset of compact_impl (louvain_compact.cpp:357-360 +
// engine_detail.cpp:26-42): K_u = fp64 row sum, Sigma = K, C = identity,
// flags = 1 for rows with arcs (rows with none are never visited,
// louvain_compact.cpp:138-141).
//
// Bytes: reset = 4 B x arcs + 29 B x vertices.
#include "kernels.cuh"

namespace lvn {
namespace {

constexpr int kT = 256;     // threads per tile

// uniform-weight detection folded into the reset's row reads: any arc weight
// differing from the first arc's clears *uni (one atomic per warp at most)
__device__ __forceinline__ void uni_flush(u32* uni, bool differs) {
  if (uni && __any_sync(__activemask(), differs) && (threadIdx.x & 31) == (__ffs(__activemask()) - 1))
    atomicAnd(uni, 0u);
}
constexpr int kRounds = 8;  // vertices per thread per tile
constexpr int kTileV = kT * kRounds;

__device__ __forceinline__ int bin_of(u64 deg, const BinEdges& e) {
  if (deg == 0) return kBinIso;
  if (deg <= e.thread_max) return kBinThread;
  if (deg <= e.group_max) {
    if (deg <= 8) return kBinSort8;
    if (deg <= 16) return kBinSort16;
    if (deg <= 32) return kBinSort32;
    if (deg <= 64) return kBinSort64;
    if (deg <= 128) return kBinSort128;
    return kBinSort256;
  }
  if (deg <= e.warp_max) return kBinWarp;
  if (deg <= e.block_max) return deg <= kBlockSplitDeg / 2 ? kBinBlockT : deg <= kBlockSplitDeg ? kBinBlockS : kBinBlock;
  return kBinGlobal;
}

__global__ void __launch_bounds__(kT) bin_count(const u64* __restrict__ off, u32 n, BinEdges e,
                                                u64 cap, u64* __restrict__ counts, u32 nblocks,
                                                ull* max_deg) {
  __shared__ u32 cnt[kBins];
  if (threadIdx.x < kBins) cnt[threadIdx.x] = 0;
  __syncthreads();
  const u64 base = u64(blockIdx.x) * kTileV;
  const int lane = threadIdx.x & 31;
  u64 mx = 0;
  for (int r = 0; r < kRounds; ++r) {
    const u64 v = base + u64(r) * kT + threadIdx.x;
    int b = -1;
    if (v < n) {
      u64 d = off[v + 1] - off[v];
      mx = d > mx ? d : mx;
      d = d < cap ? d : cap;
      b = bin_of(d, e);
    }
#pragma unroll
    for (int k = 0; k < kBins; ++k) {
      const u32 bal = __ballot_sync(0xffffffffu, b == k);
      if (lane == 0 && bal) atomicAdd(&cnt[k], __popc(bal));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 y = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = y > mx ? y : mx;
  }
  if (lane == 0 && mx) atomicMax(max_deg, ull(mx));
  __syncthreads();
  if (threadIdx.x < kBins) counts[u64(threadIdx.x) * nblocks + blockIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(kT) bin_scatter(const u64* __restrict__ off, u32 n, BinEdges e,
                                                  u64 cap, const u64* __restrict__ pos,
                                                  u32 nblocks, u32* __restrict__ list, u32 id_base) {
  __shared__ u32 wc[kT / 32][kBins];
  __shared__ u64 run[kBins];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x < kBins) run[threadIdx.x] = pos[u64(threadIdx.x) * nblocks + blockIdx.x];
  const u64 base = u64(blockIdx.x) * kTileV;
  const u32 lt = (1u << lane) - 1u;
  for (int r = 0; r < kRounds; ++r) {
    const u64 v = base + u64(r) * kT + threadIdx.x;
    int b = -1;
    if (v < n) {
      u64 d = off[v + 1] - off[v];
      d = d < cap ? d : cap;
      b = bin_of(d, e);
    }
    u32 my_rank = 0;
#pragma unroll
    for (int k = 0; k < kBins; ++k) {
      const u32 bal = __ballot_sync(0xffffffffu, b == k);
      if (lane == 0) wc[wid][k] = __popc(bal);
      if (b == k) my_rank = __popc(bal & lt);
    }
    __syncthreads();
    if (b >= 0) {
      u64 o = run[b];
      for (int w = 0; w < wid; ++w) o += wc[w][b];
      list[o + my_rank] = u32(v) + id_base;
    }
    __syncthreads();
    if (threadIdx.x < kBins) {
      u64 t = 0;
      for (int w = 0; w < kT / 32; ++w) t += wc[w][threadIdx.x];
      run[threadIdx.x] += t;
    }
    __syncthreads();
  }
}

__global__ void gather_starts(const u64* pos, u32 nblocks, const ull* max_deg, u64* out) {
  if (threadIdx.x < kBins) out[threadIdx.x] = pos[u64(threadIdx.x) * nblocks];
  if (threadIdx.x == kBins) out[kBins] = *max_deg;
}

// thread per vertex: identity, flags, and the sequential fp64 row sum for
// short rows (same summation order as the reference)
__global__ void reset_thread(DGraph g, u32 short_max, double* __restrict__ K,
                             double* __restrict__ sigma, u32* __restrict__ C,
                             u8* __restrict__ flags, u32* uni) {
  const float wref = g.arcs ? g.w[0] : 0.f;
  bool differs = false;
  for (u64 v = blockIdx.x * u64(blockDim.x) + threadIdx.x; v < g.n;
       v += u64(gridDim.x) * blockDim.x) {
    const u64 lo = g.off[v], hi = g.off[v + 1];
    if (C) C[v] = u32(v);
    if (flags) flags[v] = hi > lo ? 1 : 0;
    if (hi - lo <= short_max) {
      double s = 0.0;
      for (u64 a = lo; a < hi; ++a) {
        const float w = g.w[a];
        differs = differs || w != wref;
        s += double(w);
      }
      K[v] = s;
      if (sigma) sigma[v] = s;
    }
  }
  uni_flush(uni, differs);
}

// rows of the register-sort bins above 32 arcs: a warp per row, K arcs per
// lane, two rows in flight per warp
template <int K>
__global__ void __launch_bounds__(256) reset_group(DGraph g, const u32* __restrict__ list, u64 count,
                                                   double* __restrict__ K_out, double* __restrict__ sigma,
                                                   u32* uni) {
  const float wref = g.arcs ? g.w[0] : 0.f;
  bool differs = false;
  const u32 lane = threadIdx.x & 31;
  const u64 wi = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5;
  const u64 warps = u64(gridDim.x) * (blockDim.x >> 5);
  for (u64 i = wi; i < count; i += 2 * warps) {
    u32 v[2];
    float w[2][K];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const u64 ij = i + u64(j) * warps;
      v[j] = ij < count ? list[ij] : 0u;
      const u64 lo = ij < count ? g.off[v[j]] : 0, hi = ij < count ? g.off[v[j] + 1] : 0;
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const u64 a = lo + u64(r) * 32 + lane;
        w[j][r] = a < hi ? __ldcs(g.w + a) : 0.f;
        differs = differs || (a < hi && w[j][r] != wref);
      }
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      double k = 0.0;
#pragma unroll
      for (int r = 0; r < K; ++r) {
        k += double(w[j][r]);
      }
      k = warp_sum(k);
      if (lane == 0 && i + u64(j) * warps < count) {
        K_out[v[j]] = k;
        if (sigma) sigma[v[j]] = k;
      }
    }
  }
  uni_flush(uni, differs);
}

__global__ void reset_warp(DGraph g, const u32* __restrict__ list, u64 count,
                           double* __restrict__ K, double* __restrict__ sigma, u32* uni) {
  const float wref = g.arcs ? g.w[0] : 0.f;
  bool differs = false;
  const int lane = threadIdx.x & 31;
  const u64 warps = u64(gridDim.x) * (blockDim.x >> 5);
  for (u64 i = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5; i < count; i += warps) {
    const u32 v = list[i];
    const u64 lo = g.off[v], hi = g.off[v + 1];
    // four loads in flight per lane (rows of up to 1024 arcs)
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    u64 a = lo + lane;
    for (; a + 96 < hi; a += 128) {
      const float w0 = __ldcs(g.w + a), w1 = __ldcs(g.w + a + 32), w2 = __ldcs(g.w + a + 64),
                  w3 = __ldcs(g.w + a + 96);
      differs = differs || w0 != wref || w1 != wref || w2 != wref || w3 != wref;
      s0 += double(w0), s1 += double(w1), s2 += double(w2), s3 += double(w3);
    }
    for (; a < hi; a += 32) {
      const float w = __ldcs(g.w + a);
      differs = differs || w != wref;
      s0 += double(w);
    }
    double s = warp_sum((s0 + s1) + (s2 + s3));
    if (lane == 0) {
      K[v] = s;
      if (sigma) sigma[v] = s;
    }
  }
  uni_flush(uni, differs);
}

__global__ void __launch_bounds__(512) reset_block(DGraph g, const u32* __restrict__ list,
                                                   u64 count, double* __restrict__ K,
                                                   double* __restrict__ sigma, u32* uni) {
  __shared__ double ws[16];
  const float wref = g.arcs ? g.w[0] : 0.f;
  bool differs = false;
  for (u64 i = blockIdx.x; i < count; i += gridDim.x) {
    const u32 v = list[i];
    const u64 lo = g.off[v], hi = g.off[v + 1];
    // four loads in flight per thread
    const u64 st = blockDim.x;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    u64 a = lo + threadIdx.x;
    for (; a + 3 * st < hi; a += 4 * st) {
      const float w0 = __ldcs(g.w + a), w1 = __ldcs(g.w + a + st), w2 = __ldcs(g.w + a + 2 * st),
                  w3 = __ldcs(g.w + a + 3 * st);
      differs = differs || w0 != wref || w1 != wref || w2 != wref || w3 != wref;
      s0 += double(w0), s1 += double(w1), s2 += double(w2), s3 += double(w3);
    }
    for (; a < hi; a += st) {
      const float w = __ldcs(g.w + a);
      differs = differs || w != wref;
      s0 += double(w);
    }
    double s = warp_sum((s0 + s1) + (s2 + s3));
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < int(blockDim.x >> 5); ++w) t += ws[w];
      K[v] = t;
      if (sigma) sigma[v] = t;
    }
    __syncthreads();
  }
  uni_flush(uni, differs);
}

void reset_impl(const DGraph& g, const Bins& b, double* K, double* sigma, u32* C, u8* flags,
                cudaStream_t s, u32* uni = nullptr) {
  if (g.n == 0) return;
  const int sms = sm_count();
  const u64 tb = std::min<u64>((g.n + 255) / 256, u64(sms) * 16);
  // rows of <= 32 arcs: one thread, sequential sum (the reference's order)
  reset_thread<<<unsigned(tb), 256, 0, s>>>(g, 32u, K, sigma, C, flags, uni);
  LVN_LAUNCH();
  // 32 < deg <= 256 in the register-sort bins: a warp per row, K arcs per lane
  auto grp = [&](int bin, auto kernel) {
    if (!b.count(bin)) return;
    const u64 wb = std::min<u64>((b.count(bin) + 7) / 8, u64(sms) * 8);
    kernel<<<unsigned(wb), 256, 0, s>>>(g, b.of(bin), b.count(bin), K, sigma, uni);
    LVN_LAUNCH();
  };
  grp(kBinSort64, reset_group<2>);
  grp(kBinSort128, reset_group<4>);
  grp(kBinSort256, reset_group<8>);
  // the warp bin and the short block rows (<= 1024 arcs, adjacent in the
  // list): one warp per row; a block only for the longer rows
  const u64 mid = b.count(kBinWarp) + b.count(kBinBlockT) + b.count(kBinBlockS);
  if (mid) {
    const u64 wb = std::min<u64>((mid + 7) / 8, u64(sms) * 16);
    reset_warp<<<unsigned(wb), 256, 0, s>>>(g, b.of(kBinWarp), mid, K, sigma, uni);
    LVN_LAUNCH();
  }
  const u64 big = b.count(kBinBlock) + b.count(kBinGlobal);
  if (big) {
    const u64 bb = std::min<u64>(big, u64(sms) * 4);
    reset_block<<<unsigned(bb), 512, 0, s>>>(g, b.of(kBinBlock), big, K, sigma, uni);
    LVN_LAUNCH();
  }
}

// active vertices of every bin segment, packed at the front of the segment
// Tiles of 1024 list entries per block: warp-aggregated shared counters per
// bin, then ONE global reservation per (tile, bin) instead of one per warp
// (a lattice pass puts every vertex in one bin: 24 M / 32 same-address
// atomics per iteration made this the third-largest kernel on C4).
constexpr int kCompactItems = 4;
__global__ void __launch_bounds__(256) compact_active_k(const u32* __restrict__ list, u64 n, BinView v,
                                                        const u8* __restrict__ flags, u32* __restrict__ out,
                                                        ull* __restrict__ counts) {
  __shared__ u32 cnt[kBins];
  __shared__ ull base[kBins];
  constexpr u64 kTile = 256 * kCompactItems;
  const int lane = threadIdx.x & 31;
  for (u64 t0 = blockIdx.x * kTile; t0 < n; t0 += u64(gridDim.x) * kTile) {
    if (threadIdx.x < kBins) cnt[threadIdx.x] = 0;
    __syncthreads();
    u32 u[kCompactItems], pos[kCompactItems];
    int bin[kCompactItems];
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k) {
      const u64 i = t0 + u64(k) * 256 + threadIdx.x;
      u[k] = i < n ? list[i] : 0u;
      int b = kBins - 1;
      while (b > 0 && i < v.off[b]) --b;
      const bool on = i < n && b != kBinIso && flags[u[k]];
      bin[k] = on ? b : -1;
      const u32 peers = __match_any_sync(0xffffffffu, on ? u32(b) : 0xFFFFFFFFu);
      const int leader = __ffs(peers) - 1;
      u32 wb = 0;
      if (on && lane == leader) wb = atomicAdd(&cnt[b], u32(__popc(peers)));
      wb = __shfl_sync(0xffffffffu, wb, leader);
      pos[k] = wb + __popc(peers & ((1u << lane) - 1u));
    }
    __syncthreads();
    if (threadIdx.x < kBins && cnt[threadIdx.x]) base[threadIdx.x] = atomicAdd(&counts[threadIdx.x], ull(cnt[threadIdx.x]));
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k)
      if (bin[k] >= 0) out[v.off[bin[k]] + base[bin[k]] + pos[k]] = u[k];
    __syncthreads();
  }
}

}  // namespace

void compact_active(const Bins& b, const u8* flags, u32* out_list, ull* counts, cudaStream_t s) {
  LVN_CUDA(cudaMemsetAsync(counts, 0, kBins * sizeof(ull), s));
  const u64 n = b.start[kBins];
  if (!n) return;
  const u64 blocks = std::min<u64>((n + 1023) / 1024, u64(sm_count()) * 8);
  compact_active_k<<<unsigned(blocks), 256, 0, s>>>(b.list.p, n, b.view(), flags, out_list, counts);
  LVN_LAUNCH();
}

void compute_bins(const u64* off, u32 n, const BinEdges& e, Bins& out, cudaStream_t s, u64 cap,
                  u32 id_base) {
  out.edges = e;
  out.list.ensure(n ? n : 1);
  if (n == 0) {
    for (int b = 0; b <= kBins; ++b) out.start[b] = 0;
    out.max_degree = 0;
    return;
  }
  const u32 nblocks = u32((u64(n) + kTileV - 1) / kTileV);
  const u64 ncnt = u64(kBins) * nblocks;
  DBuf<u64> counts(ncnt), pos(ncnt + 1), small(kBins + 1);
  DBuf<ull> mx(1);
  LVN_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(ull), s));
  bin_count<<<nblocks, kT, 0, s>>>(off, n, e, cap, counts.p, nblocks, mx.p);
  LVN_LAUNCH();
  exclusive_scan_u64(counts.p, pos.p, ncnt, s);
  bin_scatter<<<nblocks, kT, 0, s>>>(off, n, e, cap, pos.p, nblocks, out.list.p, id_base);
  LVN_LAUNCH();
  gather_starts<<<1, 32, 0, s>>>(pos.p, nblocks, mx.p, small.p);
  LVN_LAUNCH();
  u64* h = ctx().pinned;
  LVN_CUDA(cudaMemcpyAsync(h, small.p, (kBins + 1) * sizeof(u64), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < kBins; ++b) out.start[b] = h[b];
  out.start[kBins] = n;
  out.max_degree = h[kBins];
}

void pass_reset(const DGraph& g, const Bins& b, double* K, double* sigma, u32* C, u8* flags,
                cudaStream_t s, u32* uniform) {
  if (uniform) LVN_CUDA(cudaMemsetAsync(uniform, 0xFF, sizeof(u32), s));
  reset_impl(g, b, K, sigma, C, flags, s, uniform);
}

void vertex_weights(const DGraph& g, const Bins& b, double* K, cudaStream_t s) {
  reset_impl(g, b, K, nullptr, nullptr, nullptr, s);
}

}  // namespace lvn
