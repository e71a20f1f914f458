// fp64 modularity (quality.cpp:9-41): Q = sum_c [sigma_c/2m - (Sigma_c/2m)^2],
// sigma_c = weight of arcs with both ends in c (a self-loop once), Sigma_c =
// sum of member arc weights. One row pass computes, per vertex, its row sum K_u
// and its internal weight; internal weights are reduced to one scalar and K_u
// is added to tot[C[u]] with fp64 L2 reductions (warp-aggregated per
// community); a second pass forms sum_c (tot_c / 2m)^2.
//
// Bytes: 12 B x arcs + 12 B x vertices.
#include "kernels.cuh"

namespace lvn {
namespace {

// one fp64 contribution per vertex into tot[c], aggregated across equal c in a warp
__device__ __forceinline__ void add_tot(double* tot, u32 c, double k) {
  const u32 act = __activemask();
  const u32 peers = __match_any_sync(act, c);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(peers) - 1;
  double s = 0.0;
  for (u32 rest = peers; rest; rest &= rest - 1) s += __shfl_sync(peers, k, __ffs(rest) - 1);
  if (lane == leader) atomicAdd(&tot[c], s);
}

// one count per vertex into ext[c] (arcs to other communities), warp-aggregated
__device__ __forceinline__ void add_ext(ull* ext, u32 c, ull n) {
  const u32 act = __activemask();
  const u32 peers = __match_any_sync(act, c);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(peers) - 1;
  ull s = 0;
  for (u32 rest = peers; rest; rest &= rest - 1) s += __shfl_sync(peers, n, __ffs(rest) - 1);
  if (lane == leader && s) atomicAdd(&ext[c], s);
}

// X (ext-only): count each row's arcs to other communities into ext[C[u]]
// instead of the modularity terms (aggregation capacities, aggregate.cu)
template <bool X>
__global__ void mod_thread(DGraph g, const u32* __restrict__ list, u64 count,
                           const u32* __restrict__ C, double* __restrict__ tot, double* sums, ull* ext) {
  double internal = 0.0;
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < count;
       i += u64(gridDim.x) * blockDim.x) {
    const u32 v = list[i];
    const u32 c = C[v];
    double k = 0.0, in = 0.0;
    ull out = 0;
    for (u64 a = g.off[v]; a < g.off[v + 1]; ++a) {
      if (X) {
        out += C[g.tgt[a]] != c;
        continue;
      }
      const double w = double(arc_w(g, a));
      k += w;
      if (C[g.tgt[a]] == c) in += w;
    }
    if (X) {
      add_ext(ext, c, out);
    } else {
      internal += in;
      add_tot(tot, c, k);
    }
  }
  if (X) return;
  internal = warp_sum(internal);
  if ((threadIdx.x & 31) == 0 && internal != 0.0) atomicAdd(&sums[0], internal);
}

// Rows of the register-sort bins: a G-lane group per row, K arcs per lane
// (arc r*G + lane, coalesced), two rows per group in flight so each lane has
// 2K independent gathers of C[t] outstanding. The thread-per-row kernel above
// reads 32 different rows per warp load (one L1TEX line per lane per arc).
template <int G, int K, bool X>
__global__ void __launch_bounds__(256) mod_group(DGraph g, const u32* __restrict__ list, u64 count,
                                                 const u32* __restrict__ C, double* __restrict__ tot,
                                                 double* sums, ull* ext) {
  constexpr int GPB = 256 / G;
  const u32 lane = threadIdx.x & (G - 1);
  const u64 gi = (blockIdx.x * u64(blockDim.x) + threadIdx.x) / G;
  const u64 groups = u64(gridDim.x) * GPB;
  double internal = 0.0;
  for (u64 i = gi; i < count; i += 2 * groups) {
    u32 v[2], c[2], t[2][K];
    u64 lo[2], hi[2];
    float w[2][K];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const u64 ij = i + u64(j) * groups;
      v[j] = ij < count ? list[ij] : 0u;
      lo[j] = ij < count ? g.off[v[j]] : 0;
      hi[j] = ij < count ? g.off[v[j] + 1] : 0;
      c[j] = ij < count ? C[v[j]] : kEmpty;
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const u64 a = lo[j] + u64(r) * G + lane;
        t[j][r] = a < hi[j] ? __ldcs(g.tgt + a) : kEmpty;
        w[j][r] = X ? 0.f : a < hi[j] ? arc_w(g, a) : 0.f;
      }
    }
    u32 ct[2][K];
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int r = 0; r < K; ++r) ct[j][r] = t[j][r] != kEmpty ? C[t[j][r]] : kEmpty;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (X) {
        u32 out = 0;
#pragma unroll
        for (int r = 0; r < K; ++r) out += ct[j][r] != kEmpty && ct[j][r] != c[j];
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) out += __shfl_xor_sync(0xffffffffu, out, o, G);
        if (lane == 0 && c[j] != kEmpty && out) atomicAdd(&ext[c[j]], ull(out));
        continue;
      }
      double k = 0.0;
#pragma unroll
      for (int r = 0; r < K; ++r) {
        k += double(w[j][r]);
        if (ct[j][r] == c[j]) internal += double(w[j][r]);
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o, G);
      if (lane == 0 && c[j] != kEmpty && k != 0.0) atomicAdd(&tot[c[j]], k);
    }
  }
  if (X) return;
  internal = warp_sum(internal);
  if ((threadIdx.x & 31) == 0 && internal != 0.0) atomicAdd(&sums[0], internal);
}

template <bool X>
__global__ void mod_warp(DGraph g, const u32* __restrict__ list, u64 count,
                         const u32* __restrict__ C, double* __restrict__ tot, double* sums, ull* ext) {
  const int lane = threadIdx.x & 31;
  const u64 warps = u64(gridDim.x) * (blockDim.x >> 5);
  double internal = 0.0;
  for (u64 i = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5; i < count; i += warps) {
    const u32 v = list[i];
    const u32 c = C[v];
    double k = 0.0, in = 0.0;
    if (X) {
      u32 out = 0;
      for (u64 a = g.off[v] + lane; a < g.off[v + 1]; a += 32) out += C[g.tgt[a]] != c;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) out += __shfl_xor_sync(0xffffffffu, out, o);
      if (lane == 0 && out) atomicAdd(&ext[c], ull(out));
    } else {
      for (u64 a = g.off[v] + lane; a < g.off[v + 1]; a += 32) {
        const double w = double(arc_w(g, a));
        k += w;
        if (C[g.tgt[a]] == c) in += w;
      }
    }
    if (X) continue;
    k = warp_sum(k);
    internal += in;
    if (lane == 0) atomicAdd(&tot[c], k);
  }
  if (X) return;
  internal = warp_sum(internal);
  if (lane == 0 && internal != 0.0) atomicAdd(&sums[0], internal);
}

template <bool X>
__global__ void __launch_bounds__(512) mod_block(DGraph g, const u32* __restrict__ list, u64 count,
                                                 const u32* __restrict__ C,
                                                 double* __restrict__ tot, double* sums, ull* ext) {
  __shared__ double ws[16];
  double internal = 0.0;
  for (u64 i = blockIdx.x; i < count; i += gridDim.x) {
    const u32 v = list[i];
    const u32 c = C[v];
    if (X) {
      u32 out = 0;
      for (u64 a = g.off[v] + threadIdx.x; a < g.off[v + 1]; a += blockDim.x) out += C[__ldcs(g.tgt + a)] != c;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) out += __shfl_xor_sync(0xffffffffu, out, o);
      if ((threadIdx.x & 31) == 0 && out) atomicAdd(&ext[c], ull(out));
      continue;
    }
    double k = 0.0;
    for (u64 a = g.off[v] + threadIdx.x; a < g.off[v + 1]; a += blockDim.x) {
      const double w = double(arc_w(g, a));
      k += w;
      if (C[g.tgt[a]] == c) internal += w;
    }
    k = warp_sum(k);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = k;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < int(blockDim.x >> 5); ++w) t += ws[w];
      atomicAdd(&tot[c], t);
    }
    __syncthreads();
  }
  if (X) return;
  internal = warp_sum(internal);
  if ((threadIdx.x & 31) == 0 && internal != 0.0) atomicAdd(&sums[0], internal);
}

__global__ void sum_squares(const double* __restrict__ tot, u64 width, double two_m, double* sums) {
  double acc = 0.0;
  for (u64 c = blockIdx.x * u64(blockDim.x) + threadIdx.x; c < width;
       c += u64(gridDim.x) * blockDim.x) {
    const double f = tot[c] / two_m;
    acc += f * f;
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc != 0.0) atomicAdd(&sums[1], acc);
}


template <bool X>
void row_pass(const DGraph& g, const Bins& b, const u32* C, double* tot, double* sums, ull* ext, cudaStream_t s) {
  const int sms = sm_count();
  // rows in the register-sort bins: a lane group per row (the bin fixes the
  // row length bound); isolated vertices contribute nothing
  auto grp = [&](int bin, auto kernel, int G) {
    if (!b.count(bin)) return;
    const u64 per_block = 256 / G;
    const u64 blocks = std::min<u64>((b.count(bin) + per_block - 1) / per_block, u64(sms) * 8);
    kernel<<<unsigned(blocks), 256, 0, s>>>(g, b.of(bin), b.count(bin), C, tot, sums, ext);
    LVN_LAUNCH();
  };
  // rows of <= 16 arcs (thread, sort8 and sort16 bins, adjacent in the list): a thread each
  const u64 small = b.start[kBinSort32] - b.start[kBinThread];
  if (small) {
    const u64 blocks = std::min<u64>((small + 255) / 256, u64(sms) * 8);
    mod_thread<X><<<unsigned(blocks), 256, 0, s>>>(g, b.of(kBinThread), small, C, tot, sums, ext);
    LVN_LAUNCH();
  }
  grp(kBinSort32, mod_group<32, 1, X>, 32);
  grp(kBinSort64, mod_group<32, 2, X>, 32);
  grp(kBinSort128, mod_group<32, 4, X>, 32);
  grp(kBinSort256, mod_group<32, 8, X>, 32);
  const u64 mid = b.count(kBinWarp);
  if (mid) {
    const u64 blocks = std::min<u64>((mid + 7) / 8, u64(sms) * 8);
    mod_warp<X><<<unsigned(blocks), 256, 0, s>>>(g, b.of(kBinWarp), mid, C, tot, sums, ext);
    LVN_LAUNCH();
  }
  const u64 big = b.count(kBinBlockT) + b.count(kBinBlockS) + b.count(kBinBlock) + b.count(kBinGlobal);
  if (big) {
    const u64 blocks = std::min<u64>(big, u64(sms) * 4);
    mod_block<X><<<unsigned(blocks), 512, 0, s>>>(g, b.of(kBinBlockT), big, C, tot, sums, ext);
    LVN_LAUNCH();
  }
}

}  // namespace

void modularity_rows(const DGraph& g, const Bins& b, const u32* C, double* tot, u64 width, double* sums,
                     cudaStream_t s) {
  LVN_CUDA(cudaMemsetAsync(tot, 0, width * sizeof(double), s));
  LVN_CUDA(cudaMemsetAsync(sums, 0, 2 * sizeof(double), s));
  row_pass<false>(g, b, C, tot, sums, nullptr, s);
}

void modularity_squares(const double* tot, u64 width, double two_m, double* sums, cudaStream_t s) {
  if (!width) return;
  const int sms = sm_count();
  const u64 blocks = std::min<u64>((width + 255) / 256, u64(sms) * 8);
  sum_squares<<<unsigned(blocks), 256, 0, s>>>(tot, width, two_m, sums);
  LVN_LAUNCH();
}

void modularity_terms(const DGraph& g, const Bins& b, const u32* C, double* tot, u64 width,
                      double* sums, cudaStream_t s, double two_m) {
  modularity_rows(g, b, C, tot, width, sums, s);
  modularity_squares(tot, width, two_m, sums, s);
}

// Q of the last super-graph with exact per-vertex terms: internal weight =
// the fp64 self-loop self64[v] + the arcs to other members of v's community,
// total degree Kx[v] (fp64); a warp per vertex
__global__ void mod_exact_k(DGraph g, const u32* __restrict__ C, const double* __restrict__ kx,
                            const double* __restrict__ self64, double* __restrict__ tot, double* __restrict__ sums) {
  const u32 lane = threadIdx.x & 31;
  const u64 warps = u64(gridDim.x) * (blockDim.x >> 5);
  double internal = 0.0;
  for (u64 v = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5; v < g.n; v += warps) {
    const u32 c = C[v];
    double in = 0.0;
    for (u64 a = g.off[v] + lane; a < g.off[v + 1]; a += 32) {
      const u32 t = g.tgt[a];
      if (t != v && C[t] == c) in += double(arc_w(g, a));
    }
    in = warp_sum(in);
    if (lane == 0) {
      internal += in + self64[v];
      if (kx[v] != 0.0) atomicAdd(&tot[c], kx[v]);
    }
  }
  internal = warp_sum(internal);
  if (lane == 0 && internal != 0.0) atomicAdd(&sums[0], internal);
}

void modularity_exact(const DGraph& g, const u32* C, const double* kx, const double* self64, double* tot, u64 width,
                      double* sums, cudaStream_t s, double two_m) {
  LVN_CUDA(cudaMemsetAsync(tot, 0, (width ? width : 1) * sizeof(double), s));
  LVN_CUDA(cudaMemsetAsync(sums, 0, 2 * sizeof(double), s));
  if (g.n) {
    const u64 blocks = std::min<u64>((u64(g.n) + 7) / 8, u64(sm_count()) * 8);
    mod_exact_k<<<unsigned(blocks), 256, 0, s>>>(g, C, kx, self64, tot, sums);
    LVN_LAUNCH();
  }
  modularity_squares(tot, width, two_m, sums, s);
}

void external_arcs(const DGraph& g, const Bins& b, const u32* C, u64* ext, u64 width, cudaStream_t s) {
  LVN_CUDA(cudaMemsetAsync(ext, 0, width * sizeof(u64), s));
  row_pass<true>(g, b, C, nullptr, nullptr, reinterpret_cast<ull*>(ext), s);
}

}  // namespace lvn
