// Register-resident bitonic sort and segmented reduction of (key, value)
// pairs across a group of G lanes holding K pairs each (N = G*K elements,
// element e in lane e / K, register e % K). Data-independent: every lane of a
// warp executes the same branch-free instruction stream, so groups of
// different vertices (G < 32) advance in lockstep with no divergence.
//
// Used by the local-moving sort kernels (K_{u->c} per neighbour community) and
// the aggregation sort kernels (super-edge weights per target community);
// keys kEmpty (padding, skipped arcs) sort last.
#pragma once

#include "common.cuh"

namespace lvn {

template <int G, int K, class V>
__device__ __forceinline__ void bitonic_sort(u32 (&key)[K], V (&val)[K], u32 lane) {
  constexpr int N = G * K;
  constexpr u32 FULL = 0xffffffffu;
#pragma unroll
  for (int size = 2; size <= N; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      if (j < K) {  // partner in the same lane
#pragma unroll
        for (int r = 0; r < K; ++r) {
          if (r & j) continue;
          const int r2 = r | j;
          const bool asc = ((lane * K + r) & size) == 0;
          const u32 lo_k = asc ? min(key[r], key[r2]) : max(key[r], key[r2]);
          const u32 hi_k = asc ? max(key[r], key[r2]) : min(key[r], key[r2]);
          const bool sw = lo_k != key[r];
          const V v1 = sw ? val[r2] : val[r], v2 = sw ? val[r] : val[r2];
          key[r] = lo_k, key[r2] = hi_k, val[r] = v1, val[r2] = v2;
        }
      } else {  // partner lane ^ (j / K), same register
        const int lj = j / K;
#pragma unroll
        for (int r = 0; r < K; ++r) {
          const u32 pk = __shfl_xor_sync(FULL, key[r], lj, G);
          const V pv = __shfl_xor_sync(FULL, val[r], lj, G);
          // keep the smaller key when (lower lane, ascending) or (upper, descending)
          const bool keep_min = (((lane & lj) == 0) == (((lane * K + r) & size) == 0));
          const u32 nk = keep_min ? min(key[r], pk) : max(key[r], pk);
          val[r] = nk != key[r] ? pv : val[r];
          key[r] = nk;
        }
      }
    }
  }
}

// After bitonic_sort: val[r] becomes the inclusive sum of its run of equal
// keys up to and including the element; tail[r] marks the last element of a
// run, where val holds the run total.
template <int G, int K, class V>
__device__ __forceinline__ void segmented_runs(const u32 (&key)[K], V (&val)[K], bool (&tail)[K], u32 lane) {
  constexpr u32 FULL = 0xffffffffu;
  const u32 prev_last = __shfl_up_sync(FULL, key[K - 1], 1, G);
  bool head[K];
  bool lane_head = false;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    head[r] = r == 0 ? (lane == 0 || key[0] != prev_last) : key[r] != key[r - 1];
    if (r > 0 && !head[r]) val[r] += val[r - 1];
    lane_head = lane_head || head[r];
  }
  // carry of the run entering each lane: segmented inclusive scan over lanes of
  // (lane total, lane has a head) with (a1,f1).(a2,f2) = (f2 ? a2 : a1 + a2, f1|f2)
  V agg = val[K - 1];
  int f = lane_head;
#pragma unroll
  for (int d = 1; d < G; d <<= 1) {
    const V pa = __shfl_up_sync(FULL, agg, d, G);
    const int pf = __shfl_up_sync(FULL, f, d, G);
    if (lane >= u32(d)) {
      agg = f ? agg : pa + agg;
      f = f | pf;
    }
  }
  const V carry_in = __shfl_up_sync(FULL, agg, 1, G);
  bool open = lane != 0;
#pragma unroll
  for (int r = 0; r < K; ++r) {
    open = open && !head[r];
    val[r] = open ? val[r] + carry_in : val[r];
  }
  const int next_head = __shfl_down_sync(FULL, int(head[0]), 1, G);
#pragma unroll
  for (int r = 0; r < K; ++r) tail[r] = r + 1 < K ? head[r + 1] : (lane == G - 1 || next_head);
}

// Warp-level pre-combine of one (key, value) per lane before a table insert,
// for lanes holding consecutive elements of a row. First, runs of equal
// adjacent keys are summed (segmented Hillis-Steele scan over the run heads;
// about 20 instructions): a row stored sorted by target whose neighbours share
// communities (hosts, blocks) keeps one value per run. If a key still repeats
// across the remaining run totals (more than 8 of them: unordered rows; one
// match.any tells; few hot communities), the 32 pairs are sorted by key and
// summed per run, so
// each distinct key is inserted once: same-key inserts serialise per lane in
// shared memory and per address in L2. Returns true on the lanes that hold a
// distinct key's total (never for kEmpty).
template <class V>
__device__ __forceinline__ bool warp_combine(u32& key, V& val, u32 lane) {
  constexpr u32 FULL = 0xffffffffu;
  const u32 up = __shfl_up_sync(FULL, key, 1);
  const u32 dn = __shfl_down_sync(FULL, key, 1);
  const u32 heads = __ballot_sync(FULL, lane == 0 || up != key);
  const u32 start = 31u - __clz(heads & (FULL >> (31u - lane)));  // this lane's run head
  V x = val;
#pragma unroll
  for (u32 d = 1; d < 32; d <<= 1) {
    const V y = __shfl_up_sync(FULL, x, d);
    if (lane >= start + d) x += y;
  }
  const bool tail = (lane == 31 || dn != key) && key != kEmpty;
  key = tail ? key : kEmpty;
  val = tail ? x : V(0);
  // few run totals left: inserting them directly beats the repeat check
  if (__popc(__ballot_sync(FULL, tail)) <= 8) return tail;
  const u32 peers = __match_any_sync(FULL, key);
  if (__any_sync(FULL, key != kEmpty && peers != (1u << lane))) {
    u32 kk[1] = {key};
    V vv[1] = {val};
    bitonic_sort<32, 1, V>(kk, vv, lane);
    bool tl[1];
    segmented_runs<32, 1, V>(kk, vv, tl, lane);
    key = kk[0], val = vv[0];
    return tl[0] && key != kEmpty;
  }
  return key != kEmpty;
}

// exclusive prefix count of `n` over the G lanes of a group, and the group total
template <int G>
__device__ __forceinline__ u32 group_exclusive(u32 n, u32 lane, u32& total) {
  constexpr u32 FULL = 0xffffffffu;
  u32 inc = n;
#pragma unroll
  for (int d = 1; d < G; d <<= 1) {
    const u32 p = __shfl_up_sync(FULL, inc, d, G);
    if (lane >= u32(d)) inc += p;
  }
  total = __shfl_sync(FULL, inc, G - 1, G);
  return inc - n;
}

}  // namespace lvn
