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
// smem hash tables (warp: ag_group, block: ag_block) and, beyond block_max,
// per-community HBM tables filled arc-parallel (ag_big_*).
// Bytes: 12 B x A_in + 16 B x V_in + 8 B x A_out + 8 B x (count+1).
#include <cooperative_groups.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <cooperative_groups/reduce.h>

#include "kernels.cuh"
#include "psort.cuh"
#include "sortnet.cuh"
#include "tables.cuh"

namespace cg = cooperative_groups;

namespace lvn {
namespace {

constexpr int kWarpCapLog = 9;
constexpr int kBlockCapLog = 13;
constexpr int kBlockThreads = 512;
using Tab = SplitF64;

// fp64 sum -> f32 super-graph weight (narrowed once, louvain_mc.cpp:95); a
// narrowing that loses bits raises *x.inexact (then the engine computes the
// final modularity on the input graph instead of the last super-graph)
__device__ __forceinline__ float narrow(const AggArgs& x, u32 key, u32 c, double v) {
  const float f = float(v);
  if (key == c) {
    // the super-vertex self-loop (its internal weight) keeps its fp64 sum
    if (x.self64) x.self64[c] = v;
  } else if (x.inexact && double(f) != v) {
    *x.inexact = 1u;
  }
  return f;
}
// weight of a super-row entry: narrowed into hw, or (partial rows of a
// sharded aggregation, hw64 set) kept in fp64 for the owner's merge
__device__ __forceinline__ void put_w(const AggArgs& x, u64 i, u32 key, u32 c, double v) {
  if (x.hw64) x.hw64[i] = v;
  else x.hw[i] = narrow(x, key, c, v);
}

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
          val[r] = double(arc_w(x.g, a));
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
            put_w(x, hbase + pos, key[r], c, val[r]);  // fp64 sum narrowed once
            ++pos;
          }
        }
        if (lane == 0) x.fill[c] = total;
      }
    }
  }
}

// Packed-key variant (psort.cuh): keys (C[t] << LB) | position, the f32
// weights staged per group in smem and fetched by position after the sort,
// runs summed in fp64 (sequence starts from a ballot). Needs count < 2^(32-LB).
template <int G, int K>
__global__ void __launch_bounds__(256) ag_psort(AggArgs x, const u32* __restrict__ list, u64 count) {
  constexpr int GPB = 256 / G;
  constexpr int N = G * K;
  constexpr int LB = ilog2<N>();
  constexpr u32 FULL = 0xffffffffu;
  __shared__ float wbuf[256 * K];
  const u32 lane = threadIdx.x & (G - 1);
  const u32 gi = threadIdx.x / G;
  const u32 gshift = (threadIdx.x & 31u) & ~u32(G - 1);
  float* gw = wbuf + gi * N;
  const ull dirs = psort_dirs<G, K>(lane);
  for (u64 i0 = u64(blockIdx.x) * GPB; i0 < count; i0 += u64(gridDim.x) * GPB) {
    const u64 i = i0 + gi;
    const bool have = i < count;
    const u32 c = have ? list[i] : 0;
    u32 key[K];
#pragma unroll
    for (int r = 0; r < K; ++r) key[r] = kNoKey;
    u64 mlo = 0, mhi = 0;
    if (have) mlo = x.coff[c], mhi = x.coff[c + 1];
    __syncwarp();
    const u64 nm = mhi - mlo;
    if (__all_sync(FULL, nm <= u64(G))) {
      // lane j holds member j's row: an inclusive scan of the row lengths
      // maps every element to its member (shuffle search), so all K arcs per
      // lane are loaded at once instead of one member row after another
      u64 mlo_j = 0, md_j = 0;
      if (lane < nm) {
        const u32 v = x.members[mlo + lane];
        mlo_j = x.g.off[v];
        md_j = x.g.off[v + 1] - mlo_j;
      }
      u64 end_j = md_j;  // inclusive prefix of the row lengths
#pragma unroll
      for (int o = 1; o < G; o <<= 1) {
        const u64 y = __shfl_up_sync(FULL, end_j, o, G);
        if (lane >= u32(o)) end_j += y;
      }
      const u64 total = __shfl_sync(FULL, end_j, G - 1, G);
#pragma unroll
      for (int r = 0; r < K; ++r) {
        const u64 e = u64(r) * G + lane;
        u32 j = 0;  // first member whose inclusive end exceeds e
#pragma unroll
        for (u32 step = G / 2; step; step >>= 1) {
          const u64 en = __shfl_sync(FULL, end_j, j + step - 1, G);
          if (en <= e) j += step;
        }
        const u64 lo_j = __shfl_sync(FULL, mlo_j, j, G);
        const u64 st_j = __shfl_sync(FULL, end_j - md_j, j, G);
        if (e < total) {
          const u64 a = lo_j + (e - st_j);
          key[r] = (x.C[__ldcs(x.g.tgt + a)] << LB) | u32(e);
          gw[e] = arc_w(x.g, a);
        }
      }
    } else {
      u64 base = 0;
      for (u64 k = mlo; k < mhi; ++k) {
        const u32 v = x.members[k];
        const u64 lo = x.g.off[v], d = x.g.off[v + 1] - lo;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const u64 e = u64(r) * G + lane;
          if (e >= base && e < base + d) {
            const u64 a = lo + (e - base);
            key[r] = (x.C[__ldcs(x.g.tgt + a)] << LB) | u32(e);
            gw[e] = arc_w(x.g, a);
          }
        }
        base += d;
      }
    }
    __syncwarp();
    psort<G, K>(key, dirs);
    u32 ck[K];
    double val[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      ck[r] = key[r] == kNoKey ? kEmpty : key[r] >> LB;
      val[r] = key[r] == kNoKey ? 0.0 : double(gw[key[r] & u32(N - 1)]);
    }
    bool tail[K];
    prun_sums<G, K, double>(ck, val, tail, lane, gshift);
    u32 mine = 0;
#pragma unroll
    for (int r = 0; r < K; ++r) mine += (tail[r] && ck[r] != kEmpty) ? 1u : 0u;
    u32 total;
    u32 pos = group_exclusive<G>(mine, lane, total);
    if (have) {
      const u64 hbase = x.hoff[c], hcap = x.hoff[c + 1] - hbase;
      if (total > hcap) {
        if (lane == 0) atomicOr(x.err, u32(kErrTable));
      } else {
#pragma unroll
        for (int r = 0; r < K; ++r) {
          if (tail[r] && ck[r] != kEmpty) {
            x.htgt[hbase + pos] = ck[r];
            put_w(x, hbase + pos, ck[r], c, val[r]);  // fp64 sum narrowed once
            ++pos;
          }
        }
        if (lane == 0) x.fill[c] = total;
      }
    }
    (void)FULL;
  }
}

// merge one member's arcs into the table
__device__ __forceinline__ void merge_row(const AggArgs& x, const Tab& tab, u32 lg, u32 c, u32 v,
                                          u32 lane, u32 stride, double& own, u32& own_seen) {
  const u64 lo = x.g.off[v], hi = x.g.off[v + 1];
  for (u64 a = lo + lane; a < hi; a += stride) {
    const u32 key = x.C[x.g.tgt[a]];
    const double w = double(arc_w(x.g, a));
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
        put_w(x, o, key, c, val);
      }
      pos += __popc(bal);
    }
    if (lane == 0) {
      if (own_seen) {
        x.htgt[hbase + pos] = c;
        put_w(x, hbase + pos, c, c, own);
        ++pos;
      }
      if (pos > hcap) atomicOr(x.err, u32(kErrTable));
      x.fill[c] = u32(pos);
    }
    tile.sync();
  }
}

// One arc per lane per round (kEmpty when the lane has none): the weight to
// the community itself is summed privately, the rest is pre-combined across
// the warp and inserted once per distinct key.
__device__ __forceinline__ void ag_merge_round(const Tab& tab, u32 lg, u32 c, u32 key, double w, u32 lane,
                                               double& own, u32& own_seen) {
  if (key == c) {
    own += w;
    own_seen = 1;
    key = kEmpty;
  }
  if (warp_combine(key, w, lane)) tab.insert(lg, key, w);
}

// Block per community (budget <= block_max): the community's member arcs are
// enumerated flat, thread t taking arcs t, t + 512, ... of the concatenated
// member rows (member found by binary search in an smem prefix of member
// degrees), so a hub member is spread over the whole block instead of one
// warp while the others wait at the barrier. Communities with more members
// than the prefix holds (many arc-less members) take the member loops.
constexpr u32 kPrefixCap = 4096;

__device__ void ag_block_one(const AggArgs& x, const Tab& tab, u32* pre, u32 c, u32 lg, double* red,
                             u32* red_seen, u32* cursor) {
  const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int W = kBlockThreads / 32;
  const u64 mlo = x.coff[c], mhi = x.coff[c + 1], nm = mhi - mlo;
  const u64 hbase = x.hoff[c], hcap = x.hoff[c + 1] - hbase;
  const u32 S = 1u << lg;
  for (u32 s = threadIdx.x; s < S; s += kBlockThreads) tab.clear(s);
  if (threadIdx.x == 0) *cursor = 0;
  double own = 0.0;
  u32 own_seen = 0;
  if (nm <= kPrefixCap) {
    // pre[k] = arcs of members [0, k): block-wide exclusive scan in chunks
    u32 run = 0;
    for (u64 k0 = 0; k0 < nm; k0 += kBlockThreads) {
      const u64 k = k0 + threadIdx.x;
      u32 d = 0;
      if (k < nm) {
        const u32 v = x.members[mlo + k];
        d = u32(x.g.off[v + 1] - x.g.off[v]);
      }
      u32 inc = d;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= u32(o)) inc += y;
      }
      if (lane == 31) red_seen[wid] = inc;
      __syncthreads();
      u32 before = run;
      for (u32 w = 0; w < wid; ++w) before += red_seen[w];
      if (k < nm) pre[k] = before + inc - d;
      u32 tot = 0;
      for (int w = 0; w < W; ++w) tot += red_seen[w];
      run += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) pre[nm] = run;
    __syncthreads();
    const u32 E = run;
    // uniform trip count over the block: every warp runs every round
    for (u32 e0 = 0; e0 < E; e0 += kBlockThreads) {
      const u32 e = e0 + threadIdx.x;
      u32 key = kEmpty;
      double w = 0.0;
      if (e < E) {
        u32 lo = 0, hi = u32(nm);  // last k with pre[k] <= e
        while (hi - lo > 1) {
          const u32 mid = (lo + hi) >> 1;
          if (pre[mid] <= e) lo = mid; else hi = mid;
        }
        const u32 v = x.members[mlo + lo];
        const u64 a = x.g.off[v] + (e - pre[lo]);
        key = x.C[__ldcs(x.g.tgt + a)];
        w = double(arc_w(x.g, a));
      }
      ag_merge_round(tab, lg, c, key, w, lane, own, own_seen);
    }
  } else {
    __syncthreads();
    // rows of >= 32 arcs: a warp across each row; shorter rows: a lane each
    for (u64 k = mlo + wid; k < mhi; k += W) {
      const u32 v = x.members[k];
      const u64 lo = x.g.off[v], hi = x.g.off[v + 1];
      if (hi - lo < 32) continue;
      for (u64 a0 = lo; a0 < hi; a0 += 32) {
        const u64 a = a0 + lane;
        const u32 key = a < hi ? x.C[__ldcs(x.g.tgt + a)] : kEmpty;
        const double w = a < hi ? double(arc_w(x.g, a)) : 0.0;
        ag_merge_round(tab, lg, c, key, w, lane, own, own_seen);
      }
    }
    for (u64 k0 = mlo + u64(wid) * 32; k0 < mhi; k0 += u64(W) * 32) {
      const u64 k = k0 + lane;
      u64 a = 0, hi = 0;
      if (k < mhi) {
        const u32 v = x.members[k];
        a = x.g.off[v], hi = x.g.off[v + 1];
        if (hi - a >= 32) hi = a;  // taken by the warp loop above
      }
      for (; __any_sync(0xffffffffu, a < hi); ++a) {
        const u32 key = a < hi ? x.C[x.g.tgt[a]] : kEmpty;
        const double w = a < hi ? double(arc_w(x.g, a)) : 0.0;
        ag_merge_round(tab, lg, c, key, w, lane, own, own_seen);
      }
    }
  }
  own = warp_sum(own);
  own_seen = __any_sync(0xffffffffu, own_seen);
  __syncthreads();  // red_seen doubled as scan scratch
  if (lane == 0) red[wid] = own, red_seen[wid] = own_seen;
  __syncthreads();
  for (u32 s = threadIdx.x; s < S; s += kBlockThreads) {
    u32 key;
    double val;
    if (tab.read(s, key, val)) {
      const u32 o = atomicAdd(cursor, 1u);
      x.htgt[hbase + o] = key;
      put_w(x, hbase + o, key, c, val);
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
      put_w(x, hbase + pos, c, c, t);
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
  u32* pre = reinterpret_cast<u32*>(smem + (size_t(1) << kBlockCapLog) * Tab::kSlotBytes);
  for (u64 i = blockIdx.x; i < count; i += gridDim.x) {
    const u32 c = list[i];
    const u64 hcap = x.hoff[c + 1] - x.hoff[c];
    const u32 lg = table_log(hcap, 5);
    if (lg > u32(kBlockCapLog)) {  // the Block bin has budgets <= 4096
      if (threadIdx.x == 0) atomicOr(x.err, u32(kErrTable));
      continue;
    }
    ag_block_one(x, stab, pre, c, lg, red, red_seen, &cursor);
  }
}

// ---- communities with budget > block_max: arc-parallel ---------------------------
// The members of the big communities (grouped by community, vertices without
// arcs dropped) form a list L whose arcs are cut into tiles (ag_big_arcs): a
// hub row is split across many blocks and the blocks of one community run
// together, so its HBM region stays hot in L2. The weight to the community
// itself (the super-vertex self-loop, usually the dominant key) is summed per
// lane while the lane stays in one community and added once per run; the
// other arcs are pre-combined across the warp and merged into the
// community's region:
//   hash  : 16-byte slots {key, fp64 value} (one sector per probe), claimed by
//           CAS (one L2 round trip per probe), fp64 L2 reductions, a live list;
//   dense : when the hash table would outgrow a dense fp64 array over all
//           `count` target communities, the array itself (no keys, no probing:
//           one reduction per arc; present entries are the ones no longer -0.0).
// Then one block per community emits the row.
//
// Region sizes: a region holds the community's holey capacity min(ext + 1,
// count) keys (ext: its arcs to other communities, counted by external_arcs),
// which bounds its distinct targets, at load <= 1/2. Inserts still check for
// a full region (live list full, or a probe sequence wrapping): a flagged
// community stops inserting and is redone in a second round sized by the arcs
// it counted there (a guard: with exact capacities it does not trigger).
constexpr ull kDenseEmpty = 0x8000000000000000ull;  // -0.0: never produced by adding a weight

struct BigSlot {
  u32 key;
  u32 pad;
  double val;
};

// slots of a hash region for `keys` expected keys (load <= 1/2), or 0 for dense
__device__ __forceinline__ u64 big_region_slots(u64 keys, u32 count, int mode) {
  const u32 l = ceil_log2_u64(2 * (keys ? keys : 1));
  const u64 slots = u64(1) << (l > 5 ? l : 5);
  const bool dense = mode ? mode == 2 : slots * sizeof(BigSlot) >= u64(count) * sizeof(double);
  return dense ? 0 : slots;
}
__device__ __forceinline__ u64 big_region_bytes(u64 slots, u32 count) {
  if (!slots) return (u64(count) * sizeof(double) + 15) & ~u64(15);
  return (slots * sizeof(BigSlot) + slots / 2 * 4 + 15) & ~u64(15);
}
// claim-or-find by CAS (one round trip per probe); returns the slot and
// whether this call claimed it, or ~0u when the probe sequence wraps (full)
// Giant-community regions probe linearly whatever lvn_params.probing says:
// they are a device structure with no counterpart among the reference's
// slab tables, and a linear step stays within the 64-byte DRAM burst of the
// 16-byte slot just missed (the probing modes cost 11 % of C5's aggregation
// here: 40 -> 48 registers in ag_big_arcs)
__device__ __forceinline__ u32 big_insert(BigSlot* t, u64 slots, u32 key, double w, bool& fresh) {
  const u32 lg = ceil_log2_u64(slots);
  const u32 mask = u32(slots - 1);
  u32 h = slot_hash(key, lg);
  for (u64 probe = 0; probe < slots; ++probe) {
    const u32 cur = atomicCAS(&t[h].key, kEmpty, key);
    if (cur == kEmpty || cur == key) {
      atomicAdd(&t[h].val, w);
      fresh = cur == kEmpty;
      return h;
    }
    h = (h + 1) & mask;
  }
  fresh = false;
  return ~0u;
}
// largest i in [0, n) with p[i] <= x (p ascending, p[0] <= x)
__device__ __forceinline__ u64 last_le(const u64* __restrict__ p, u64 n, u64 x) {
  u64 lo = 0, hi = n;
  while (hi - lo > 1) {
    const u64 mid = (lo + hi) >> 1;
    if (p[mid] <= x) lo = mid; else hi = mid;
  }
  return lo;
}

// round 1 (ext_c == nullptr): estimated region sizes; round 2: sized by the
// community's arcs to other communities counted in round 1 (>= its keys)
__global__ void ag_big_plan(const u32* __restrict__ big, u64 nbig, u32 count, int mode,
                            const u64* __restrict__ ext_c, const u64* __restrict__ hoff,
                            const u64* __restrict__ boff, const u64* __restrict__ coff, u32* __restrict__ index,
                            u64* __restrict__ rslots, u64* __restrict__ bytes, u32* __restrict__ mcount) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < nbig; i += u64(gridDim.x) * blockDim.x) {
    const u32 c = big[i];
    index[c] = u32(i);
    const u64 hcap = hoff[c + 1] - hoff[c];
    const u64 sl = big_region_slots(ext_c ? min(hcap, ext_c[c] + 1) : hcap, count, mode);
    rslots[i] = sl;
    bytes[i] = big_region_bytes(sl, count);
    mcount[i] = u32(coff[c + 1] - coff[c]);
  }
}

__global__ void ag_big_clear(u64 nbig, u32 count, const u64* __restrict__ rslots,
                             const u64* __restrict__ tab_off, unsigned char* tables) {
  for (u64 i = blockIdx.x; i < nbig; i += gridDim.x) {
    unsigned char* base = tables + tab_off[i];
    const u64 slots = rslots[i];
    if (!slots) {
      ull* d = reinterpret_cast<ull*>(base);
      for (u64 j = threadIdx.x; j < count; j += blockDim.x) d[j] = kDenseEmpty;
    } else {
      BigSlot* t = reinterpret_cast<BigSlot*>(base);
      for (u64 j = threadIdx.x; j < slots; j += blockDim.x) t[j] = BigSlot{kEmpty, 0u, 0.0};
    }
  }
}

// j-th member of the big communities (j < M): vertex and whether it has arcs
__global__ void ag_big_keep(AggArgs x, const u32* __restrict__ big, u64 nbig, const u64* __restrict__ moff,
                            u64 M, u32* __restrict__ vert, u32* __restrict__ keep) {
  for (u64 j = blockIdx.x * u64(blockDim.x) + threadIdx.x; j < M; j += u64(gridDim.x) * blockDim.x) {
    const u64 pi = last_le(moff, nbig, j);
    const u32 v = x.members[x.coff[big[pi]] + (j - moff[pi])];
    vert[j] = v;
    keep[j] = x.g.off[v + 1] > x.g.off[v] ? 1u : 0u;
  }
}

__global__ void ag_big_list(const DGraph g, const u32* __restrict__ vert, const u32* __restrict__ keep,
                            const u32* __restrict__ kpos, u64 M, u32* __restrict__ L, u32* __restrict__ D) {
  for (u64 j = blockIdx.x * u64(blockDim.x) + threadIdx.x; j < M; j += u64(gridDim.x) * blockDim.x) {
    if (!keep[j]) continue;
    const u32 v = vert[j];
    L[kpos[j]] = v;
    D[kpos[j]] = u32(g.off[v + 1] - g.off[v]);
  }
}

// Per-round state of the big path, indexed by the position of a community in
// the round's list.
struct BigState {
  const u32* index;     // community -> position
  const u64* rslots;    // position -> hash slots (0: dense region)
  const u64* tab_off;   // position -> byte offset of its region
  unsigned char* tables;
  u32* live_n;          // live entries (hash) / emitted entries (dense)
  double* own_sum;      // weight to the community itself
  u32* own_seen;
  u32* ovf;             // region overflowed: redone in round 2
  u64* ext;             // arcs to other communities (round 2 sizes regions by it)
};

// P: exclusive scan of the arc counts of L (nL + 1 entries, P[nL] = all arcs).
//
// The flat arc space [0, P[nL]) is cut into tiles of kBigTile arcs; tile t's
// first owner (last i with P[i] <= t kBigTile) comes from big_tile_owner. A
// block takes one tile at a time:
//   1. owner metadata of the tile (<= kBigTile members: vertex, community,
//      region, row base) into smem, one thread per owner, all loads in flight;
//   2. owner of every arc: head marks + block max-scan over the tile;
//   3. the tile's targets and weights staged into smem with cp.async
//      (LDGSTS, 4 B per arc, every copy of the tile in flight before one wait):
//      the neighbour lists of the members are contiguous CSR segments;
//   4. C[t] gathers for all staged targets (8 per thread in flight), then per
//      warp batch of 32 consecutive arcs: own-community weight summed per
//      lane, the rest pre-combined across the warp and merged into the
//      community's region (dense fp64 reductions or the 16-byte-slot table).
// The dependent chain owner -> vertex -> row -> target -> community is paid
// once per tile instead of once per 32 arcs.
constexpr u32 kBigTile = 2048;
constexpr u32 kBigThreads = 256;
constexpr u32 kBigPer = kBigTile / kBigThreads;
constexpr size_t kBigSmem = size_t(kBigTile) * (8 + 4 + 4 + 4 + 4 + 2);

__global__ void big_tile_owner(const u64* __restrict__ P, const u32* __restrict__ nL_p, u32* __restrict__ first) {
  const u64 nL = *nL_p;
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < nL; i += u64(gridDim.x) * blockDim.x) {
    const u64 p0 = P[i], p1 = P[i + 1];
    // tiles whose start t * kBigTile falls in [p0, p1): owner i
    for (u64 t = (p0 + kBigTile - 1) / kBigTile; t * kBigTile < p1; ++t) first[t] = u32(i);
  }
}

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

__global__ void __launch_bounds__(kBigThreads) ag_big_arcs(AggArgs x, BigState st, const u32* __restrict__ L,
                                                           const u64* __restrict__ P, const u32* __restrict__ nL_p,
                                                           const u32* __restrict__ tile_first, u64 a_lo, u64 a_hi) {
  extern __shared__ __align__(16) unsigned char big_smem[];
  u64* s_base = reinterpret_cast<u64*>(big_smem);        // owner -> row start - P[i]
  u32* s_tgt = reinterpret_cast<u32*>(s_base + kBigTile);  // staged targets
  float* s_w = reinterpret_cast<float*>(s_tgt + kBigTile); // staged weights
  u32* s_c = reinterpret_cast<u32*>(s_w + kBigTile);       // owner -> community
  u32* s_pi = s_c + kBigTile;                              // owner -> region index
  u16* s_own = reinterpret_cast<u16*>(s_pi + kBigTile);    // tile-local owner of each arc
  __shared__ u32 s_scan[kBigThreads];
  const u32 tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u64 nL = *nL_p;
  if (!nL) return;
  const u64 E = min(P[nL], a_hi);
  if (a_lo >= E) return;
  const u64 t_lo = a_lo / kBigTile, t_hi = (E + kBigTile - 1) / kBigTile;
  u32 own_pi = ~0u, seen = 0;  // per-lane run of the own-community weight
  double own = 0.0;
  for (u64 t = t_lo + blockIdx.x; t < t_hi; t += gridDim.x) {
    const u64 lo = max(t * kBigTile, a_lo), hi = min((t + 1) * kBigTile, E);
    const u32 nA = u32(hi - lo);
    // owner of lo: the tile's first owner, or (first tile of a batch) within
    // the next kBigTile owners (every owner has at least one arc)
    u64 i0 = tile_first[t];
    if (lo != t * kBigTile) i0 += last_le(P + i0, min(nL - i0, u64(kBigTile) + 1), lo);
    // 1. owners: i0 + j while P[i0 + j] < hi
    for (u32 j = tid; j < kBigTile; j += kBigThreads) s_own[j] = 0;
    __syncthreads();
    for (u32 j = tid; j < nA; j += kBigThreads) {
      const u64 i = i0 + j;
      if (i >= nL) break;
      const u64 p = P[i];
      if (p >= hi) break;
      const u32 v = L[i];
      const u32 c = x.C[v];
      s_c[j] = c;
      s_pi[j] = st.index[c];
      s_base[j] = x.g.off[v] - p;
      s_own[p > lo ? u32(p - lo) : 0u] = u16(j);
    }
    __syncthreads();
    // 2. owner of each arc: inclusive max-scan of the head marks
    {
      u32 run = 0;
      u16 loc[kBigPer];
#pragma unroll
      for (u32 k = 0; k < kBigPer; ++k) {
        run = max(run, u32(s_own[tid * kBigPer + k]));
        loc[k] = u16(run);
      }
      u32 incl = run;
#pragma unroll
      for (u32 d = 1; d < 32; d <<= 1) {
        const u32 o = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl = max(incl, o);
      }
      if (lane == 31) s_scan[wid] = incl;
      __syncthreads();
      u32 carry = 0;
      for (u32 w = 0; w < wid; ++w) carry = max(carry, s_scan[w]);
      const u32 prev = __shfl_up_sync(0xffffffffu, incl, 1);
      carry = max(carry, lane ? prev : 0u);
#pragma unroll
      for (u32 k = 0; k < kBigPer; ++k) s_own[tid * kBigPer + k] = u16(max(carry, u32(loc[k])));
    }
    __syncthreads();
    // 3. stage targets and weights (cp.async, every copy in flight)
#pragma unroll
    for (u32 k = 0; k < kBigPer; ++k) {
      const u32 e = k * kBigThreads + tid;
      if (e < nA) {
        const u64 ga = s_base[s_own[e]] + lo + e;
        cp_async4(&s_tgt[e], x.g.tgt + ga);
        if (!x.g.uniform) cp_async4(&s_w[e], x.g.w + ga);
      }
    }
    cp_async_wait_all();
    __syncthreads();
    // 4. communities of the targets, then merge per warp batch
    u32 key[kBigPer];
#pragma unroll
    for (u32 k = 0; k < kBigPer; ++k) {
      const u32 e = k * kBigThreads + wid * 32 + lane;
      key[k] = e < nA ? x.C[s_tgt[e]] : kEmpty;
    }
#pragma unroll
    for (u32 k = 0; k < kBigPer; ++k) {
      const u32 e = k * kBigThreads + wid * 32 + lane;
      u32 kk = key[k], c = 0, pi = 0;
      double wt = 0.0;
      if (e < nA) {
        const u32 o = s_own[e];
        c = s_c[o];
        pi = s_pi[o];
        wt = x.g.uniform ? double(x.g.uw) : double(s_w[e]);
        if (kk == c) {
          if (pi != own_pi) {
            if (seen) atomicAdd(&st.own_sum[own_pi], own), st.own_seen[own_pi] = 1;
            own_pi = pi, own = 0.0;
          }
          own += wt;
          seen = 1;
          kk = kEmpty;
        }
      }
      // a batch inside one community (the usual case): one merge per distinct key
      const u32 phi = __reduce_max_sync(0xffffffffu, kk != kEmpty ? pi : 0u);
      const u32 plo = __reduce_min_sync(0xffffffffu, kk != kEmpty ? pi : ~0u);
      if (phi == plo) {
        const u32 next = __popc(__ballot_sync(0xffffffffu, kk != kEmpty));
        if (lane == 0 && next) atomicAdd(reinterpret_cast<ull*>(&st.ext[phi]), ull(next));
        if (!warp_combine(kk, wt, lane)) continue;
        pi = phi;
      } else if (kk == kEmpty) {
        continue;
      } else {
        atomicAdd(reinterpret_cast<ull*>(&st.ext[pi]), 1ull);
      }
      unsigned char* base = st.tables + st.tab_off[pi];
      const u64 slots = st.rslots[pi];
      if (!slots) {
        atomicAdd(reinterpret_cast<double*>(base) + kk, wt);
      } else if (!*reinterpret_cast<volatile u32*>(&st.ovf[pi])) {
        bool fresh;
        const u32 sl = big_insert(reinterpret_cast<BigSlot*>(base), slots, kk, wt, fresh);
        if (sl == ~0u) {
          st.ovf[pi] = 1;
        } else if (fresh) {
          const u32 at = atomicAdd(&st.live_n[pi], 1u);
          if (at < slots / 2) reinterpret_cast<u32*>(base + slots * sizeof(BigSlot))[at] = sl;
          else st.ovf[pi] = 1;
        }
      }
    }
    __syncthreads();  // the stage is rewritten by the next tile
  }
  if (seen) atomicAdd(&st.own_sum[own_pi], own), st.own_seen[own_pi] = 1;
}

// present entries of the dense regions, all regions' chunks spread over the
// whole grid (one block per region left most SMs idle on few giant
// communities): warp-compacted appends to the region's row (live_n counts)
constexpr u64 kDenseChunk = 16384;
__global__ void __launch_bounds__(256) ag_dense_scan(AggArgs x, BigState st, const u32* __restrict__ big,
                                                     u64 nbig) {
  const u64 cpc = (u64(x.count) + kDenseChunk - 1) / kDenseChunk;
  const u32 lane = threadIdx.x & 31;
  for (u64 q = blockIdx.x; q < nbig * cpc; q += gridDim.x) {
    const u64 i = q / cpc, j0 = (q % cpc) * kDenseChunk;
    if (st.rslots[i]) continue;
    const u32 c = big[i];
    const u64 hbase = x.hoff[c], hcap = x.hoff[c + 1] - hbase;
    const ull* d = reinterpret_cast<const ull*>(st.tables + st.tab_off[i]);
    const u64 j1 = min(j0 + kDenseChunk, u64(x.count));
    for (u64 b = j0; b < j1; b += blockDim.x) {
      const u64 j = b + threadIdx.x;
      const ull bits = j < j1 ? d[j] : kDenseEmpty;
      const bool live = bits != kDenseEmpty;
      const u32 bal = __ballot_sync(0xffffffffu, live);
      u32 wbase = 0;
      if (lane == 0 && bal) wbase = atomicAdd(&st.live_n[i], __popc(bal));
      wbase = __shfl_sync(0xffffffffu, wbase, 0);
      if (live) {
        const u32 o = wbase + __popc(bal & ((1u << lane) - 1u));
        if (o < hcap) {
          x.htgt[hbase + o] = u32(j);
          put_w(x, hbase + o, u32(j), c, __longlong_as_double((long long)bits));  // fp64 sum narrowed once
        }
      }
    }
  }
}

// rows of the regions that did not overflow (the others are redone in round 2)
__global__ void __launch_bounds__(kBlockThreads) ag_big_emit(AggArgs x, BigState st, const u32* __restrict__ big,
                                                             u64 nbig) {
  for (u64 i = blockIdx.x; i < nbig; i += gridDim.x) {
    if (st.ovf[i]) continue;
    const u32 c = big[i];
    const u64 hbase = x.hoff[c], hcap = x.hoff[c + 1] - hbase;
    unsigned char* base = st.tables + st.tab_off[i];
    const u32 self = st.own_seen[i] ? 1u : 0u;
    const u64 slots = st.rslots[i];
    const u32 n = st.live_n[i];  // dense: entries already emitted by ag_dense_scan
    if (slots) {
      const BigSlot* t = reinterpret_cast<const BigSlot*>(base);
      const u32* live = reinterpret_cast<const u32*>(base + slots * sizeof(BigSlot));
      for (u32 j = threadIdx.x; j < n && j < hcap; j += kBlockThreads) {
        const BigSlot e = t[live[j]];
        x.htgt[hbase + j] = e.key;
        put_w(x, hbase + j, e.key, c, e.val);  // fp64 sum narrowed once
      }
    }
    if (threadIdx.x == 0) {
      if (n + self > hcap) {
        atomicOr(x.err, u32(kErrTable));
      } else {
        if (self) {
          x.htgt[hbase + n] = c;
          put_w(x, hbase + n, c, c, st.own_sum[i]);
        }
        x.fill[c] = n + self;
      }
    }
  }
}

// communities of the list whose region overflowed, compacted (round 2 input)
__global__ void ag_big_redo(const u32* __restrict__ big, u64 nbig, const u32* __restrict__ ovf,
                            const u64* __restrict__ ext, u32* __restrict__ out, u32* __restrict__ nout,
                            u64* __restrict__ ext_c) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < nbig; i += u64(gridDim.x) * blockDim.x)
    if (ovf[i]) {
      out[atomicAdd(nout, 1u)] = big[i];
      ext_c[big[i]] = ext[i];
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


// One round of the big path over `big` (nbig communities): region plan,
// batches sized to the free memory, member arc list, tiles, merge, emit.
// Round 1 (ext_c == nullptr) uses estimated region sizes and appends the
// communities whose regions overflowed to redo[*nredo], with their counted
// arcs to other communities in ext_out[c]; round 2 sizes regions by those.
void big_round(const AggArgs& a, const u32* big, u64 nbig, const u64* ext_c, u32* redo, u32* nredo, u64* ext_out,
               cudaStream_t s) {
  const bool exact = ext_c != nullptr;
  const int sms = sm_count();
  DBuf<u32> index(a.count), live_n(nbig), own_seen(nbig), mcount(nbig), ovf(nbig);
  DBuf<u64> bytes(nbig), rslots(nbig), tab_off(nbig + 1), moff(nbig + 1), ext(nbig);
  DBuf<double> own(nbig);
  LVN_CUDA(cudaMemsetAsync(ext.p, 0, nbig * sizeof(u64), s));
  LVN_CUDA(cudaMemsetAsync(live_n.p, 0, nbig * sizeof(u32), s));
  LVN_CUDA(cudaMemsetAsync(own_seen.p, 0, nbig * sizeof(u32), s));
  LVN_CUDA(cudaMemsetAsync(ovf.p, 0, nbig * sizeof(u32), s));
  LVN_CUDA(cudaMemsetAsync(own.p, 0, nbig * sizeof(double), s));
  const unsigned pg = unsigned(std::min<u64>((nbig + 255) / 256, u64(sms) * 4));
  ag_big_plan<<<pg, 256, 0, s>>>(big, nbig, a.count, a.big_mode, ext_c, a.hoff, a.boff, a.coff, index.p,
                                 rslots.p, bytes.p, mcount.p);
  LVN_LAUNCH();
  exclusive_scan_u64(bytes.p, tab_off.p, nbig, s);
  exclusive_scan_u32_to_u64(mcount.p, moff.p, nbig, s);
  // host copies of the region offsets and member offsets (batch planning)
  std::vector<u64> h_tab(nbig + 1), h_moff(nbig + 1);
  LVN_CUDA(cudaMemcpyAsync(h_tab.data(), tab_off.p, (nbig + 1) * sizeof(u64), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaMemcpyAsync(h_moff.data(), moff.p, (nbig + 1) * sizeof(u64), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  const u64 M = h_moff[nbig];
  // The regions can exceed device memory; communities are processed in
  // batches whose regions fit a budget of a quarter of the free memory (at
  // least the largest single region).
  const size_t free_b = ctx().pool.available();
  u64 largest = 0;
  for (u64 i = 0; i < nbig; ++i) largest = std::max(largest, h_tab[i + 1] - h_tab[i]);
  u64 budget = std::min<u64>(h_tab[nbig], u64(free_b / 4));
  if (const char* e = std::getenv("LVN_BIG_TABLE_BUDGET")) budget = std::strtoull(e, nullptr, 10);  // tests
  budget = std::max<u64>(budget, largest);
  std::vector<u64> cuts{0};
  for (u64 i = 0; i < nbig; ++i)
    if (h_tab[i + 1] - h_tab[cuts.back()] > budget) cuts.push_back(i);
  cuts.push_back(nbig);
  if (const char* e = std::getenv("LVN_VERBOSE"); e && *e && *e != '0')
    std::fprintf(stderr, "[lvn] aggregate round %d: %llu giant communities, %llu members, regions %.2f GB in %zu "
                 "batches (budget %.2f GB, free %.2f GB)\n", exact ? 2 : 1, (unsigned long long)nbig,
                 (unsigned long long)M, h_tab[nbig] / 1e9, cuts.size() - 1, budget / 1e9, free_b / 1e9);
  DBuf<unsigned char> tables(budget ? budget : 16);
  // L = members of the big communities with arcs, P = scan of their degrees
  DBuf<u32> vert(M ? M : 1), keep(M + 1), kpos(M + 1), L(M ? M : 1), D(M ? M : 1);
  DBuf<u64> P(M + 1);
  const unsigned mg = unsigned(std::min<u64>((M + 255) / 256 + 1, u64(sms) * 8));
  ag_big_keep<<<mg, 256, 0, s>>>(a, big, nbig, moff.p, M, vert.p, keep.p);
  LVN_LAUNCH();
  exclusive_scan_u32(keep.p, kpos.p, M, s);
  // D past nL = kpos[M] stays 0, so P[nL..M] all hold the arc total
  LVN_CUDA(cudaMemsetAsync(D.p, 0, (M ? M : 1) * sizeof(u32), s));
  ag_big_list<<<mg, 256, 0, s>>>(a.g, vert.p, keep.p, kpos.p, M, L.p, D.p);
  LVN_LAUNCH();
  exclusive_scan_u32_to_u64(D.p, P.p, M, s);
  // first owner of every kBigTile-arc tile of the flat arc space
  u32 nL32 = 0;
  LVN_CUDA(cudaMemcpyAsync(&nL32, kpos.p + M, sizeof(u32), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  u64 total_arcs = 0;
  LVN_CUDA(cudaMemcpyAsync(&total_arcs, P.p + nL32, sizeof(u64), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  const u64 nL = nL32;
  const u64 ntiles = total_arcs / kBigTile + 1;
  DBuf<u32> tile_first(ntiles);
  LVN_CUDA(cudaMemsetAsync(tile_first.p, 0, ntiles * sizeof(u32), s));
  big_tile_owner<<<unsigned(std::min<u64>((nL + 255) / 256 + 1, u64(sms) * 8)), 256, 0, s>>>(P.p, kpos.p + M,
                                                                                             tile_first.p);
  LVN_LAUNCH();
  static const int occ = occupancy(ag_big_arcs, kBigThreads, kBigSmem);
  for (size_t bi = 0; bi + 1 < cuts.size(); ++bi) {
    const u64 b0 = cuts[bi], b1 = cuts[bi + 1], nb = b1 - b0;
    if (!nb) continue;
    // regions of this batch start at the buffer's base
    BigState st{index.p, rslots.p, tab_off.p, tables.p - h_tab[b0], live_n.p, own.p, own_seen.p, ovf.p, ext.p};
    ag_big_clear<<<unsigned(std::min<u64>(nb, u64(sms) * 4)), 256, 0, s>>>(nb, a.count, rslots.p + b0,
                                                                            tab_off.p + b0, st.tables);
    LVN_LAUNCH();
    // arc range of the batch: members [moff[b0], moff[b1]) -> kept L entries -> P
    u64 arc_lo = 0, arc_hi = ~u64(0);
    if (cuts.size() > 2) {
      u32 k[2] = {0, 0};
      LVN_CUDA(cudaMemcpyAsync(&k[0], kpos.p + h_moff[b0], sizeof(u32), cudaMemcpyDeviceToHost, s));
      LVN_CUDA(cudaMemcpyAsync(&k[1], kpos.p + h_moff[b1], sizeof(u32), cudaMemcpyDeviceToHost, s));
      LVN_CUDA(cudaStreamSynchronize(s));
      LVN_CUDA(cudaMemcpyAsync(&arc_lo, P.p + k[0], sizeof(u64), cudaMemcpyDeviceToHost, s));
      LVN_CUDA(cudaMemcpyAsync(&arc_hi, P.p + k[1], sizeof(u64), cudaMemcpyDeviceToHost, s));
      LVN_CUDA(cudaStreamSynchronize(s));
    }
    ag_big_arcs<<<unsigned(u64(sms) * occ), kBigThreads, kBigSmem, s>>>(a, st, L.p, P.p, kpos.p + M, tile_first.p,
                                                                       arc_lo, arc_hi);
    LVN_LAUNCH();
    BigState sb = st;  // views starting at the batch's first community
    sb.rslots += b0, sb.tab_off += b0, sb.live_n += b0, sb.own_sum += b0, sb.own_seen += b0, sb.ovf += b0;
    sb.ext += b0;
    ag_dense_scan<<<unsigned(u64(sms) * 8), 256, 0, s>>>(a, sb, big + b0, nb);
    LVN_LAUNCH();
    ag_big_emit<<<unsigned(std::min<u64>(nb, u64(sms) * 4)), kBlockThreads, 0, s>>>(a, sb, big + b0, nb);
    LVN_LAUNCH();
  }
  if (redo) {
    ag_big_redo<<<pg, 256, 0, s>>>(big, nbig, ovf.p, ext.p, redo, nredo, ext_out);
    LVN_LAUNCH();
  }
}

void aggregate_rows(const AggArgs& a0, const Bins& b, cudaStream_t s) {
  const int sms = sm_count();
  AggArgs a = a0;
  if (const char* e = std::getenv("LVN_BIG_MODE")) a.big_mode = std::string(e) == "hash" ? 1 : std::string(e) == "dense" ? 2 : 0;
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
  // packed keys when the community ids leave room for the row position
  const bool pk = !std::getenv("LVN_AGG_UNPACKED");
  auto fits = [&](int lb) { return pk && u64(a.count) < (u64(1) << (32 - lb)); };
  if (fits(3)) sort_bin(kBinThread, ag_psort<8, 1>, 8); else sort_bin(kBinThread, ag_sort<8, 1>, 8);
  if (fits(3)) sort_bin(kBinSort8, ag_psort<8, 1>, 8); else sort_bin(kBinSort8, ag_sort<8, 1>, 8);
  if (fits(4)) sort_bin(kBinSort16, ag_psort<16, 1>, 16); else sort_bin(kBinSort16, ag_sort<16, 1>, 16);
  if (fits(5)) sort_bin(kBinSort32, ag_psort<32, 1>, 32); else sort_bin(kBinSort32, ag_sort<32, 1>, 32);
  if (fits(6)) sort_bin(kBinSort64, ag_psort<32, 2>, 32); else sort_bin(kBinSort64, ag_sort<32, 2>, 32);
  if (fits(7)) sort_bin(kBinSort128, ag_psort<32, 4>, 32); else sort_bin(kBinSort128, ag_sort<32, 4>, 32);
  if (fits(8)) sort_bin(kBinSort256, ag_psort<32, 8>, 32); else sort_bin(kBinSort256, ag_sort<32, 8>, 32);
  if (b.count(kBinWarp)) {
    constexpr int T = 256;
    auto k = ag_group<32, kWarpCapLog, T>;
    const size_t smem = size_t(T / 32) * (1u << kWarpCapLog) * Tab::kSlotBytes;
    static const int occ = occupancy(k, T, smem);
    const u64 blocks = std::min<u64>((b.count(kBinWarp) + T / 32 - 1) / (T / 32), u64(sms) * occ);
    k<<<unsigned(blocks), T, smem, s>>>(a, b.of(kBinWarp), b.count(kBinWarp));
    LVN_LAUNCH();
  }
  const u64 nblk = b.count(kBinBlockT) + b.count(kBinBlockS) + b.count(kBinBlock);  // adjacent segments
  if (nblk) {
    const size_t smem = (size_t(1) << kBlockCapLog) * Tab::kSlotBytes + (kPrefixCap + 1) * sizeof(u32);
    static const int occ = occupancy(ag_block, kBlockThreads, smem);
    const u64 blocks = std::min<u64>(nblk, u64(sms) * occ);
    ag_block<<<unsigned(blocks), kBlockThreads, smem, s>>>(a, b.of(kBinBlockT), nblk);
    LVN_LAUNCH();
  }
  const u64 nbig = b.count(kBinGlobal);
  if (nbig) {
    DBuf<u32> redo(nbig), nredo(1);
    DBuf<u64> ext_c(a.count);
    LVN_CUDA(cudaMemsetAsync(nredo.p, 0, sizeof(u32), s));
    big_round(a, b.of(kBinGlobal), nbig, nullptr, redo.p, nredo.p, ext_c.p, s);
    u32 n2 = 0;
    LVN_CUDA(cudaMemcpyAsync(&n2, nredo.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
    if (const char* e = std::getenv("LVN_VERBOSE"); e && *e && *e != '0')
      std::fprintf(stderr, "[lvn] aggregate: %u of %llu giant communities outgrew their estimated regions\n", n2,
                   (unsigned long long)nbig);
    if (n2) big_round(a, redo.p, n2, ext_c.p, nullptr, nullptr, nullptr, s);
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

// lvn_params.probing for the tables of this file (reference probe_advance,
// compact_hashtable.hpp:60-82); stream-ordered
void set_probing_aggregate(int mode, cudaStream_t s) {
  static int value;  // pageable source: staged before the call returns
  value = mode;
  LVN_CUDA(cudaMemcpyToSymbolAsync(c_probing, &value, sizeof(int), 0, cudaMemcpyHostToDevice, s));
}

}  // namespace lvn
