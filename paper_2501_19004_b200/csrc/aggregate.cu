// Aggregation phase: compact_aggregate_into (louvain_compact.cpp:214-310).
// For every community c (renumbered, contiguous) all arcs of all members are
// merged by target community C[t] into an open-addressing table, INCLUDING
// self-loops (aggregation wants them: louvain_mc.hpp:46-54 include_self); the
// entries become row c of the super-graph, written into a holey row of
// capacity min(total member degree, #communities) (engine_detail.cpp:66-75)
// and compacted afterwards (compact_holey_into, engine_detail.cpp:77-94).
//
// Values accumulate in fp64 and are narrowed to f32 once (louvain_mc.cpp:95),
// so integer-weight super-graphs are bit-exact against the reference. The
// intra-community weight (key == c, the super-vertex self-loop) is kept
// privately per lane and reduced once: it is the dominant, most contended key.
//
// Binned by total member degree (the community's budget): budgets <= 256 use
// the register-sort kernels (ag_sort: the member arcs' (C[t], w) pairs are
// sorted by target community across a lane group and reduced per run, which
// also emits each row already in canonical target order); larger budgets use
// smem/global hash tables (warp: ag_group, block: ag_block).
// Bytes: 12 B x A_in + 16 B x V_in + 8 B x A_out + 8 B x (count+1).
#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>

#include "kernels.cuh"
#include "sortnet.cuh"
#include "tables.cuh"

namespace cg = cooperative_groups;

namespace lvn {
namespace {

constexpr int kWarpCapLog = 9;
constexpr int kBlockCapLog = 13;
constexpr int kBlockThreads = 512;
using Tab = SplitF64;

// Communities with budget <= N = G*K: element e = r*G + lane of the
// community's member arcs (members in CSR order) is loaded into register r.
template <int G, int K>
__global__ void __launch_bounds__(256) ag_sort(AggArgs x, const u32* __restrict__ list, u64 count) {
  constexpr int GPB = 256 / G;
  const u32 lane = threadIdx.x & (G - 1);
  const u32 gi = threadIdx.x / G;
  for (u64 i0 = u64(blockIdx.x) * GPB; i0 < count; i0 += u64(gridDim.x) * GPB) {
    const u64 i = i0 + gi;
    const bool have = i < count;
    const u32 c = have ? list[i] : 0;
    u32 key[K];
    double val[K];
#pragma unroll
    for (int r = 0; r < K; ++r) key[r] = kEmpty, val[r] = 0.0;
    u64 mlo = 0, mhi = 0;
    if (have) mlo = x.coff[c], mhi = x.coff[c + 1];
    u64 base = 0;
    for (u64 k = mlo; k < mhi; ++k) {
      const u32 v = x.members[k];
      const u64 lo = x.g.off[v], d = x.g.off[v + 1] - lo;
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const u64 e = u64(r) * G + lane;
        if (e >= base && e < base + d) {
          const u64 a = lo + (e - base);
          key[r] = x.C[__ldcs(x.g.tgt + a)];
          val[r] = double(__ldcs(x.g.w + a));
        }
      }
      base += d;
    }
    bitonic_sort<G, K, double>(key, val, lane);
    bool tail[K];
    segmented_runs<G, K, double>(key, val, tail, lane);
    u32 mine = 0;
#pragma unroll
    for (int r = 0; r < K; ++r) mine += (tail[r] && key[r] != kEmpty) ? 1u : 0u;
    u32 total;
    u32 pos = group_exclusive<G>(mine, lane, total);
    if (have) {
      const u64 hbase = x.hoff[c], hcap = x.hoff[c + 1] - hbase;
      if (total > hcap) {
        if (lane == 0) atomicOr(x.err, u32(kErrTable));
      } else {
#pragma unroll
        for (int r = 0; r < K; ++r) {
          if (tail[r] && key[r] != kEmpty) {
            x.htgt[hbase + pos] = key[r];
            x.hw[hbase + pos] = float(val[r]);  // fp64 sum narrowed once
            ++pos;
          }
        }
        if (lane == 0) x.fill[c] = total;
      }
    }
  }
}

// merge one member's arcs into the table
__device__ __forceinline__ void merge_row(const AggArgs& x, const Tab& tab, u32 lg, u32 c, u32 v,
                                          u32 lane, u32 stride, double& own, u32& own_seen) {
  const u64 lo = x.g.off[v], hi = x.g.off[v + 1];
  for (u64 a = lo + lane; a < hi; a += stride) {
    const u32 key = x.C[x.g.tgt[a]];
    const double w = double(x.g.w[a]);
    if (key == c) {
      own += w;
      own_seen = 1;
    } else {
      tab.insert(lg, key, w);
    }
  }
}

template <int G, int CAPLOG, int THREADS>
__global__ void __launch_bounds__(THREADS) ag_group(AggArgs x, const u32* __restrict__ list,
                                                    u64 count) {
  constexpr int GPB = THREADS / G;
  constexpr u32 CAP = 1u << CAPLOG;
  constexpr u32 MINLOG = G == 8 ? 3 : 5;
  extern __shared__ __align__(16) unsigned char smem[];
  const auto tile = cg::tiled_partition<G>(cg::this_thread_block());
  const int gi = threadIdx.x / G;
  const u32 lane = tile.thread_rank();
  const Tab tab(smem + size_t(gi) * CAP * Tab::kSlotBytes, CAP);
  for (u64 i = blockIdx.x * u64(GPB) + gi; i < count; i += u64(gridDim.x) * GPB) {
    const u32 c = list[i];
    const u64 mlo = x.coff[c], mhi = x.coff[c + 1];
    const u64 hbase = x.hoff[c], hcap = x.hoff[c + 1] - hbase;
    const u64 budget = x.boff[c + 1] - x.boff[c];
    const u32 lg = table_log(hcap, MINLOG);
    const u32 S = 1u << lg;
    for (u32 s = lane; s < S; s += G) tab.clear(s);
    tile.sync();
    double own = 0.0;
    u32 own_seen = 0;
    if (budget >= (mhi - mlo) * G) {  // long member rows: lanes across each row
      for (u64 k = mlo; k < mhi; ++k) merge_row(x, tab, lg, c, x.members[k], lane, G, own, own_seen);
    } else {  // short rows: one member per lane
      for (u64 k = mlo + lane; k < mhi; k += G) merge_row(x, tab, lg, c, x.members[k], 0, 1, own, own_seen);
    }
    own = cg::reduce(tile, own, cg::plus<double>());
    own_seen = tile.any(own_seen);
    tile.sync();
    u64 pos = 0;
    for (u32 s0 = 0; s0 < S; s0 += G) {
      u32 key;
      double val;
      const bool live = tab.read(s0 + lane, key, val);
      const u32 bal = tile.ballot(live);
      if (live) {
        const u64 o = hbase + pos + __popc(bal & ((1u << lane) - 1u));
        x.htgt[o] = key;
        x.hw[o] = float(val);
      }
      pos += __popc(bal);
    }
    if (lane == 0) {
      if (own_seen) {
        x.htgt[hbase + pos] = c;
        x.hw[hbase + pos] = float(own);
        ++pos;
      }
      if (pos > hcap) atomicOr(x.err, u32(kErrTable));
      x.fill[c] = u32(pos);
    }
    tile.sync();
  }
}

template <bool GLOBAL>
__device__ void ag_block_one(const AggArgs& x, const Tab& tab, u32 c, u32 lg, double* red,
                             u32* red_seen, u32* cursor) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int W = kBlockThreads / 32;
  const u64 mlo = x.coff[c], mhi = x.coff[c + 1];
  const u64 hbase = x.hoff[c], hcap = x.hoff[c + 1] - hbase;
  const u64 budget = x.boff[c + 1] - x.boff[c];
  const u32 S = 1u << lg;
  for (u32 s = threadIdx.x; s < S; s += kBlockThreads) tab.clear(s);
  if (threadIdx.x == 0) *cursor = 0;
  __syncthreads();
  double own = 0.0;
  u32 own_seen = 0;
  if (budget >= (mhi - mlo) * 16) {  // warp per member
    for (u64 k = mlo + wid; k < mhi; k += W) merge_row(x, tab, lg, c, x.members[k], lane, 32, own, own_seen);
  } else {  // thread per member
    for (u64 k = mlo + threadIdx.x; k < mhi; k += kBlockThreads)
      merge_row(x, tab, lg, c, x.members[k], 0, 1, own, own_seen);
  }
  own = warp_sum(own);
  own_seen = __any_sync(0xffffffffu, own_seen);
  if (lane == 0) red[wid] = own, red_seen[wid] = own_seen;
  __syncthreads();
  for (u32 s = threadIdx.x; s < S; s += kBlockThreads) {
    u32 key;
    double val;
    if (tab.read(s, key, val)) {
      const u32 o = atomicAdd(cursor, 1u);
      x.htgt[hbase + o] = key;
      x.hw[hbase + o] = float(val);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    u32 seen = 0;
    for (int k = 0; k < W; ++k) t += red[k], seen |= red_seen[k];
    u64 pos = *cursor;
    if (seen) {
      x.htgt[hbase + pos] = c;
      x.hw[hbase + pos] = float(t);
      ++pos;
    }
    if (pos > hcap) atomicOr(x.err, u32(kErrTable));
    x.fill[c] = u32(pos);
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kBlockThreads) ag_block(AggArgs x, const u32* __restrict__ list,
                                                          u64 count) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[kBlockThreads / 32];
  __shared__ u32 red_seen[kBlockThreads / 32];
  __shared__ u32 cursor;
  const Tab stab(smem, u64(1) << kBlockCapLog);
  for (u64 i = blockIdx.x; i < count; i += gridDim.x) {
    const u32 c = list[i];
    const u64 hcap = x.hoff[c + 1] - x.hoff[c];
    const u32 lg = table_log(hcap, 5);
    if (lg <= u32(kBlockCapLog)) {
      ag_block_one<false>(x, stab, c, lg, red, red_seen, &cursor);
    } else if (!x.table || (u64(1) << lg) > x.table_slots) {
      if (threadIdx.x == 0) atomicOr(x.err, u32(kErrTable));
    } else {
      const Tab gtab(x.table + blockIdx.x * x.table_slots * Tab::kSlotBytes / 8, x.table_slots);
      ag_block_one<true>(x, gtab, c, lg, red, red_seen, &cursor);
    }
  }
}

__global__ void compact_k(const u64* __restrict__ hoff, const u32* __restrict__ htgt,
                          const float* __restrict__ hw, const u32* __restrict__ fill,
                          const u64* __restrict__ noff, u32 count, u32* __restrict__ otgt,
                          float* __restrict__ ow, double* tw) {
  const int lane = threadIdx.x & 31;
  const u64 warps = u64(gridDim.x) * (blockDim.x >> 5);
  double acc = 0.0;
  for (u64 c = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5; c < count; c += warps) {
    const u64 src = hoff[c], dst = noff[c];
    const u32 k = fill[c];
    for (u32 j = lane; j < k; j += 32) {
      otgt[dst + j] = htgt[src + j];
      const float w = hw[src + j];
      ow[dst + j] = w;
      acc += double(w);
    }
  }
  acc = warp_sum(acc);
  if (lane == 0 && acc != 0.0) atomicAdd(tw, acc);
}

template <class K>
int occupancy(K kernel, int threads, size_t smem) {
  if (smem > 48 * 1024)
    LVN_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int b = 0;
  LVN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem));
  return b > 0 ? b : 1;
}

}  // namespace

size_t aggregate_table_bytes(u64 max_slots, int* blocks) {
  if (blocks) *blocks = sm_count();
  return size_t(max_slots) * Tab::kSlotBytes * size_t(sm_count());
}

void aggregate_rows(const AggArgs& a, const Bins& b, cudaStream_t s) {
  const int sms = sm_count();
  if (b.edges.thread_max > 8 || b.edges.group_max > 256 || b.edges.warp_max > 256 ||
      b.edges.block_max > 4096)
    fail(kInvalid, "aggregation bin edges exceed the device table capacities");
  // budgets <= 256: register sort, N = G*K elements per community
  auto sort_bin = [&](int bin, auto kernel, int G) {
    if (!b.count(bin)) return;
    const int occ = occupancy(kernel, 256, 0);
    const u64 blocks = std::min<u64>((b.count(bin) + 256 / G - 1) / (256 / G), u64(sms) * occ);
    kernel<<<unsigned(blocks), 256, 0, s>>>(a, b.of(bin), b.count(bin));
    LVN_LAUNCH();
  };
  sort_bin(kBinThread, ag_sort<8, 1>, 8);
  sort_bin(kBinSort8, ag_sort<8, 1>, 8);
  sort_bin(kBinSort16, ag_sort<16, 1>, 16);
  sort_bin(kBinSort32, ag_sort<32, 1>, 32);
  sort_bin(kBinSort64, ag_sort<32, 2>, 32);
  sort_bin(kBinSort128, ag_sort<32, 4>, 32);
  sort_bin(kBinSort256, ag_sort<32, 8>, 32);
  if (b.count(kBinWarp)) {
    constexpr int T = 256;
    auto k = ag_group<32, kWarpCapLog, T>;
    const size_t smem = size_t(T / 32) * (1u << kWarpCapLog) * Tab::kSlotBytes;
    static const int occ = occupancy(k, T, smem);
    const u64 blocks = std::min<u64>((b.count(kBinWarp) + T / 32 - 1) / (T / 32), u64(sms) * occ);
    k<<<unsigned(blocks), T, smem, s>>>(a, b.of(kBinWarp), b.count(kBinWarp));
    LVN_LAUNCH();
  }
  const u64 big = b.count(kBinBlock) + b.count(kBinGlobal);
  if (big) {
    const size_t smem = (size_t(1) << kBlockCapLog) * Tab::kSlotBytes;
    static const int occ = occupancy(ag_block, kBlockThreads, smem);
    const u64 blocks = std::min<u64>(big, u64(sms) * (a.table ? 1 : occ));
    ag_block<<<unsigned(blocks), kBlockThreads, smem, s>>>(a, b.of(kBinBlock), big);
    LVN_LAUNCH();
  }
}

void compact_rows(const u64* hoff, const u32* htgt, const float* hw, const u32* fill,
                  const u64* noff, u32 count, u32* otgt, float* ow, double* tw, cudaStream_t s) {
  LVN_CUDA(cudaMemsetAsync(tw, 0, sizeof(double), s));
  if (!count) return;
  const u64 blocks = std::min<u64>((u64(count) + 7) / 8, u64(sm_count()) * 16);
  compact_k<<<unsigned(blocks), 256, 0, s>>>(hoff, htgt, hw, fill, noff, count, otgt, ow, tw);
  LVN_LAUNCH();
}

}  // namespace lvn
