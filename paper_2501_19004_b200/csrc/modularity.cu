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

__global__ void mod_thread(DGraph g, const u32* __restrict__ list, u64 count,
                           const u32* __restrict__ C, double* __restrict__ tot, double* sums) {
  double internal = 0.0;
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < count;
       i += u64(gridDim.x) * blockDim.x) {
    const u32 v = list[i];
    const u32 c = C[v];
    double k = 0.0, in = 0.0;
    for (u64 a = g.off[v]; a < g.off[v + 1]; ++a) {
      const double w = double(g.w[a]);
      k += w;
      if (C[g.tgt[a]] == c) in += w;
    }
    internal += in;
    add_tot(tot, c, k);
  }
  internal = warp_sum(internal);
  if ((threadIdx.x & 31) == 0 && internal != 0.0) atomicAdd(&sums[0], internal);
}

__global__ void mod_warp(DGraph g, const u32* __restrict__ list, u64 count,
                         const u32* __restrict__ C, double* __restrict__ tot, double* sums) {
  const int lane = threadIdx.x & 31;
  const u64 warps = u64(gridDim.x) * (blockDim.x >> 5);
  double internal = 0.0;
  for (u64 i = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5; i < count; i += warps) {
    const u32 v = list[i];
    const u32 c = C[v];
    double k = 0.0, in = 0.0;
    for (u64 a = g.off[v] + lane; a < g.off[v + 1]; a += 32) {
      const double w = double(g.w[a]);
      k += w;
      if (C[g.tgt[a]] == c) in += w;
    }
    k = warp_sum(k);
    internal += in;
    if (lane == 0) atomicAdd(&tot[c], k);
  }
  internal = warp_sum(internal);
  if (lane == 0 && internal != 0.0) atomicAdd(&sums[0], internal);
}

__global__ void __launch_bounds__(512) mod_block(DGraph g, const u32* __restrict__ list, u64 count,
                                                 const u32* __restrict__ C,
                                                 double* __restrict__ tot, double* sums) {
  __shared__ double ws[16];
  double internal = 0.0;
  for (u64 i = blockIdx.x; i < count; i += gridDim.x) {
    const u32 v = list[i];
    const u32 c = C[v];
    double k = 0.0;
    for (u64 a = g.off[v] + threadIdx.x; a < g.off[v + 1]; a += blockDim.x) {
      const double w = double(g.w[a]);
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

}  // namespace

void modularity_terms(const DGraph& g, const Bins& b, const u32* C, double* tot, u64 width,
                      double* sums, cudaStream_t s, double two_m) {
  LVN_CUDA(cudaMemsetAsync(tot, 0, width * sizeof(double), s));
  LVN_CUDA(cudaMemsetAsync(sums, 0, 2 * sizeof(double), s));
  const int sms = sm_count();
  const u64 small = b.start[kBinSort64] - b.start[kBinIso];  // rows of <= 32 arcs
  if (small) {
    const u64 blocks = std::min<u64>((small + 255) / 256, u64(sms) * 8);
    mod_thread<<<unsigned(blocks), 256, 0, s>>>(g, b.of(kBinIso), small, C, tot, sums);
    LVN_LAUNCH();
  }
  const u64 mid = b.start[kBinBlock] - b.start[kBinSort64];
  if (mid) {
    const u64 blocks = std::min<u64>((mid + 7) / 8, u64(sms) * 8);
    mod_warp<<<unsigned(blocks), 256, 0, s>>>(g, b.of(kBinSort64), mid, C, tot, sums);
    LVN_LAUNCH();
  }
  const u64 big = b.count(kBinBlock) + b.count(kBinGlobal);
  if (big) {
    const u64 blocks = std::min<u64>(big, u64(sms) * 4);
    mod_block<<<unsigned(blocks), 512, 0, s>>>(g, b.of(kBinBlock), big, C, tot, sums);
    LVN_LAUNCH();
  }
  if (width) {
    const u64 blocks = std::min<u64>((width + 255) / 256, u64(sms) * 8);
    sum_squares<<<unsigned(blocks), 256, 0, s>>>(tot, width, two_m, sums);
    LVN_LAUNCH();
  }
}

}  // namespace lvn
