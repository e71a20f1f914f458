// Packed-key register sort for the local-moving sort bins (lm_psort).
//
// The (community, weight) pairs of a row are grouped by community with a
// bitonic network over 32-bit keys (community << LB) | position, LB =
// log2(G*K): keys are distinct, the network moves one register per
// compare-exchange instead of a key and a value, and each weight is fetched
// once afterwards from its row position (one shuffle for K = 1, a per-group
// shared-memory stage otherwise). Equal communities end up adjacent in row
// order, so the runs are also stable. Requires n < 2^(32 - LB) (checked by the
// launcher, which otherwise uses the unpacked network of sortnet.cuh).
//
// Per compare-exchange: SHFL + one predicate extract + IMNMX. The direction
// of every stage depends only on the lane, so it is computed once per thread
// into a bit mask (psort_dirs).
#pragma once

#include "common.cuh"

namespace lvn {

template <int N>
constexpr int ilog2() {
  return N <= 1 ? 0 : 1 + ilog2<N / 2>();
}

constexpr u32 kNoKey = 0xFFFFFFFFu;  // padding / skipped arc; sorts last

// bit s = direction of stage s for this lane: cross-lane stages "this lane
// keeps the min", in-lane stages with size >= K "ascending"
template <int G, int K>
__device__ __forceinline__ ull psort_dirs(u32 lane) {
  constexpr int N = G * K;
  ull m = 0;
  int s = 0;
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1, ++s) {
      const bool asc = ((lane * K) & size) == 0;
      const bool bit = j < K ? asc : (((lane & (j / K)) == 0) == asc);
      m |= ull(bit) << s;
    }
  }
  return m;
}

// ascending sort of the G*K keys of a group (element e = lane*K + r)
template <int G, int K>
__device__ __forceinline__ void psort(u32 (&key)[K], ull dirs) {
  constexpr int N = G * K;
  constexpr u32 FULL = 0xffffffffu;
  int s = 0;
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1, ++s) {
      const bool bit = (dirs >> s) & 1ull;
      if (j < K) {
#pragma unroll
        for (int r = 0; r < K; ++r) {
          if (r & j) continue;
          const int r2 = r | j;
          const bool asc = size < K ? ((r & size) == 0) : bit;
          const u32 lo = min(key[r], key[r2]), hi = max(key[r], key[r2]);
          key[r] = asc ? lo : hi;
          key[r2] = asc ? hi : lo;
        }
      } else {
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const u32 pk = __shfl_xor_sync(FULL, key[r], j / K, G);
          key[r] = bit ? min(key[r], pk) : max(key[r], pk);
        }
      }
    }
  }
}

// Segmented inclusive sums over runs of equal ck (sorted order, element e =
// lane*K + r of a G-lane group whose lanes start at warp lane gshift): val[r]
// becomes the sum of its run up to the element; tail[r] marks run ends, where
// val is the run total. Run starts come from one ballot, so the lane-level
// scan moves only the partial sums.
template <int G, int K, class V>
__device__ __forceinline__ void prun_sums(const u32 (&ck)[K], V (&val)[K], bool (&tail)[K], u32 lane,
                                          u32 gshift) {
  constexpr u32 FULL = 0xffffffffu;
  constexpr u32 GMASK = G == 32 ? FULL : ((1u << G) - 1u);
  const u32 prev = __shfl_up_sync(FULL, ck[K - 1], 1, G);
  bool head[K];
  bool lh = false;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    head[r] = r == 0 ? (lane == 0 || ck[0] != prev) : ck[r] != ck[r - 1];
    if (r > 0 && !head[r]) val[r] += val[r - 1];
    lh = lh || head[r];
  }
  const u32 hb = (__ballot_sync(FULL, lh) >> gshift) & GMASK;
  const u32 start = 31u - __clz(hb & ((2u << lane) - 1u));  // lane 0 always holds a head
  V agg = val[K - 1];
#pragma unroll
  for (int d = 1; d < G; d <<= 1) {
    const V p = __shfl_up_sync(FULL, agg, d, G);
    if (lane >= start + d) agg += p;
  }
  if (K == 1) {
    val[0] = agg;
  } else {
    const V carry = __shfl_up_sync(FULL, agg, 1, G);
    bool open = lane != 0;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      open = open && !head[r];
      val[r] = open ? val[r] + carry : val[r];
    }
  }
  const u32 h0 = (__ballot_sync(FULL, head[0]) >> gshift) & GMASK;
  const bool last_lane_tail = lane == G - 1 || ((h0 >> (lane + 1)) & 1u);
#pragma unroll
  for (int r = 0; r < K; ++r) tail[r] = r + 1 < K ? head[r + 1] : last_lane_tail;
}

// The same run sums for elements already ordered in *row* order, element
// e = r*G + lane (the load layout), so an ascending row needs no network:
// each register row is scanned across the lanes, and the run open at the end
// of register r carries into register r+1.
template <int G, int K, class V>
__device__ __forceinline__ void prun_sums_rows(const u32 (&ck)[K], V (&val)[K], bool (&tail)[K], u32 lane,
                                               u32 gshift) {
  constexpr u32 FULL = 0xffffffffu;
  constexpr u32 GMASK = G == 32 ? FULL : ((1u << G) - 1u);
  bool head[K];
  u32 hb[K];
  V carry = V(0);  // total of the run open at the end of the previous register
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const u32 up = __shfl_up_sync(FULL, ck[r], 1, G);
    const u32 prev_last = r > 0 ? __shfl_sync(FULL, ck[r - 1], G - 1, G) : kEmpty;
    head[r] = lane == 0 ? (r == 0 || ck[r] != prev_last) : ck[r] != up;
    hb[r] = (__ballot_sync(FULL, head[r]) >> gshift) & GMASK;
    const u32 below = hb[r] & ((2u << lane) - 1u);  // heads at lanes <= this one
    const u32 start = below ? 31u - __clz(below) : 0u;
    V agg = val[r];
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
      const V p = __shfl_up_sync(FULL, agg, d, G);
      if (lane >= start + d) agg += p;
    }
    if (!below) agg += carry;  // the run entering this register continues here
    val[r] = agg;
    carry = __shfl_sync(FULL, agg, G - 1, G);
  }
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const bool next_head = lane + 1 < u32(G) ? ((hb[r] >> (lane + 1)) & 1u) : (r + 1 < K ? (hb[r + 1] & 1u) : 1u);
    tail[r] = next_head != 0;
  }
}

// order-preserving map of a double to u64 (greater double -> greater key)
__device__ __forceinline__ ull ordered_bits(double g) {
  const ull b = ull(__double_as_longlong(g + 0.0));  // -0 -> +0
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// Group argmax of (gain, community) with ties to the lowest community
// (compact_hashtable.hpp:152). Returns the group's best community (kEmpty if
// no lane has a candidate); every lane's own (bg, bc) are left untouched, so
// the lane whose bc equals the result holds the winning gain and weight.
template <int G>
__device__ __forceinline__ u32 group_best(double bg, u32 bc) {
  constexpr u32 FULL = 0xffffffffu;
  if (G == 32) {  // warp: three redux.sync instead of a shuffle tree
    const ull o = bc == kEmpty ? 0ull : ordered_bits(bg);
    const u32 hi = u32(o >> 32), lo = u32(o);
    const u32 mh = __reduce_max_sync(FULL, hi);
    const u32 ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
    return __reduce_min_sync(FULL, (hi == mh && lo == ml) ? bc : kEmpty);
  } else {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const double og = __shfl_xor_sync(FULL, bg, o, G);
      const u32 oc = __shfl_xor_sync(FULL, bc, o, G);
      if (oc != kEmpty && (bc == kEmpty || better(og, oc, bg, bc))) bg = og, bc = oc;
    }
    return bc;
  }
}

}  // namespace lvn
