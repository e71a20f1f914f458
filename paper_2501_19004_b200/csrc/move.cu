// Local-moving phase: one sweep of compact_move (louvain_compact.cpp:116-212)
// over the active vertices, degree-binned:
//
//   bin 1  deg <= thread_max (<= 8)   thread per vertex, candidates in registers
//   bin 2  deg <= group_max  (<= 64)  8-lane group per vertex, 128-slot smem table
//   bin 3  deg <= warp_max   (<= 256) warp per vertex, 512-slot smem table
//   bin 4  deg <= block_max  (<= 4096) block per vertex, <= 8192-slot smem table
//   bin 5  larger                      block per vertex, table in global memory
//
// Per vertex u (scan_serial + decide_serial, louvain_compact.cpp:37-68):
// K_{u->c} is accumulated over the non-self arcs into an open-addressing table
// keyed by community (the weight to u's own community is kept privately per
// lane, which removes the one heavily contended key). Every slot a vertex
// claims is appended to a per-group live list, so ranking scans only live
// entries and the table is restored to empty by clearing just those slots.
// Each live entry c != C[u] is ranked by Eq. 2; ties go to the lowest id.
// The move is applied if its gain is positive and Pick-Less allows it
// (louvain_compact.cpp:151-152); applying it validates the gain against the
// Sigma values current at that instant (see decide()), updates Sigma with fp64
// L2 atomics and marks every arc target of u (louvain_compact.cpp:154-161).
//
// Ranking: the dry-run evaluation (lvn_evaluate_moves, the parity path) scores
// every candidate with the reference formula operation for operation
// (delta_q); the engine ranks with the same formula using precomputed 1/m and
// 1/(2m^2) (differences only at the last ulp) and decides with the exact
// formula.
//
// Table values: value_bits 32 -> fp32 accumulated in a packed 64-bit slot
// (key<<32 | float) updated by one CAS; value_bits 64 -> u32 key + fp64 value.
// (Shared-memory float/double atomicAdd are CAS loops on sm_100a anyway.)
//
// Algorithmic bytes: 12 B per scanned arc + 32 B per processed
// vertex; the kernels count both on the device.
#include <cooperative_groups.h>
#include <cooperative_groups/reduce.h>

#include <cmath>

#include <cub/device/device_radix_sort.cuh>

#include "kernels.cuh"
#include "psort.cuh"
#include "sortnet.cuh"
#include "tables.cuh"

namespace cg = cooperative_groups;

namespace lvn {
namespace {

constexpr int kThreadMaxD = 8;
constexpr int kWarpCapLog = 9;     // 512 slots (warp_max <= 256)
constexpr int kBlockCapLog = 13;   // 8192 slots (block_max <= 4096)
constexpr int kBlockThreads = 512;
constexpr int kBatch = 4;          // arcs (and ranked entries) in flight per lane
constexpr u64 kBlockSplit = kBlockSplitDeg;  // kBinBlockS rows: 4 sub-groups per block

// ---- per-thread accounting, flushed once per thread at kernel exit ----------
struct Tally {
  double gain = 0.0;
  ull verts = 0, arcs = 0, moves = 0, rand = 0;  // rand: random element accesses of this lane
  __device__ void flush(const MoveArgs& x) {
    const double g = warp_sum(gain);
    const ull v = warp_sum(verts), a = warp_sum(arcs), m = warp_sum(moves), r = warp_sum(rand);
    if ((threadIdx.x & 31) == 0) {
      if (g != 0.0) atomicAdd(x.gain_acc, g);
      if (v) atomicAdd(&x.counters[0], v);
      if (a) atomicAdd(&x.counters[1], a);
      if (m) atomicAdd(&x.counters[2], m);
      if (r) atomicAdd(&x.counters[3], r);
    }
  }
};

// community ids read back from a table must be vertex ids of this graph
__device__ __forceinline__ bool key_ok(const MoveArgs& x, u32 key) {
  if (key < x.g.n) return true;
  atomicOr(x.err, u32(kErrRange));
  return false;
}

// Eq. 2 for ranking: exact (reference operation order) or with reciprocals.
// With 32-bit scan values the reference stores each gain back into its f32
// table slot before taking the maximum (decide_serial, louvain_compact.cpp:
// 59-64), so gains that agree to f32 precision tie and the lowest community id
// wins; the ranking rounds the same way (V = float).
template <bool EXACT, class V = double>
__device__ __forceinline__ double score(const MoveArgs& x, double k_to_c, double own, double ku,
                                        double sigma_c, double sigma_d) {
  const double g = EXACT ? delta_q(k_to_c, own, ku, sigma_c, sigma_d, x.m)
                         : (k_to_c - own) * x.inv_m - ku * (ku + sigma_c - sigma_d) * x.inv_2m2;
  return sizeof(V) == 4 ? double(float(g)) : g;
}

// Sigma-free upper bound of Eq. 2: with Sigma_c >= 0 the gain of c is at most
// (K_{u->c} - K_{u->d})/m - K_u (K_u - Sigma_d)/(2m^2). A candidate whose bound
// is not positive can never be the move target (a move needs gain > 0,
// louvain_compact.cpp:151), so its Sigma gather is skipped. Once communities
// form, most candidates fall under the weight to the own community, and the
// random Sigma gathers (one L1TEX wavefront per lane) are what limits the sweep.
// The margin covers rounding (the bound and the score are evaluated alike).
__device__ __forceinline__ bool may_gain(const MoveArgs& x, double k_to_c, double own, double ku, double sf) {
  const double a = (k_to_c - own) * x.inv_m, b = ku * (ku - sf) * x.inv_2m2;
  return a - b >= -1e-12 * (fabs(a) + fabs(b));
}

// Move decision shared by every kernel; called by exactly one thread per vertex.
// bk = K_{u->bc}, own = K_{u->from}.
//
// Applying a move validates it against the true Sigma at the instant it
// lands: the join is one fp64 atomicAdd that returns Sigma_bc as it stood
// (all earlier joiners included), the gain is re-scored with that value (the
// reciprocal form of Eq. 2) and the current Sigma_from, and the join is undone if it is no
// longer positive. This is the reference's asynchronous semantics (every
// decision sees the moves applied before it, louvain_mc.hpp:80-86) kept under
// massive concurrency, where thousands of deciders would otherwise read the
// same stale Sigma and herd into one community.
template <bool DRY>
__device__ __forceinline__ bool decide(const MoveArgs& x, u32 u, u32 from, double ku, u32 bc,
                                       double bg, double bk, double own, Tally& t) {
  if (from >= x.g.n) {
    atomicOr(x.err, u32(kErrRange));
    return false;
  }
  bool mv = bc != kEmpty && bg > 0.0;  // bc != from by construction
  if (DRY) {
    x.out_to[u] = mv ? bc : from;
    x.out_gain[u] = mv ? bg : 0.0;
    return false;
  }
  if (x.probe) {  // report the live ranking's choice with the reference's exact gain
    const double ge = mv ? delta_q(bk, own, ku, x.sigma[bc], x.sigma[from], x.m) : 0.0;
    const double gr = x.value_f32 ? double(float(ge)) : ge;
    mv = mv && gr > 0.0;
    x.out_to[u] = mv ? bc : from;
    x.out_gain[u] = mv ? gr : 0.0;
    return false;
  }
  if (mv && (x.pickless_dev ? *x.pickless_dev : x.pickless) && bc > from) mv = false;
  // singleton pairs: two singletons that pick each other would swap labels
  // instead of merging when they decide concurrently; only the move toward
  // the lower id is taken, so the pair merges (Pick-Less, restricted to the
  // one configuration where it is always needed)
  if (mv && x.csize && bc > from && x.csize[from] == 1 && x.csize[bc] == 1) mv = false;
  if (mv) {
    const double sigma_c = atomicAdd(&x.sigma[bc], ku);
    const double sigma_d = *reinterpret_cast<volatile double*>(&x.sigma[from]);
    const double g = score<false>(x, bk, own, ku, sigma_c, sigma_d);
    if (g > 0.0) {
      atomicAdd(&x.sigma[from], -ku);
      x.C[u] = bc;
      if (x.moves_out) {  // sharded: record the move for the other ranks
        const auto grp = cg::coalesced_threads();
        u32 base = 0;
        if (grp.thread_rank() == 0) base = atomicAdd(x.moves_n, grp.size());
        const u32 i = grp.shfl(base, 0) + grp.thread_rank();
        x.moves_out[2 * u64(i)] = u;
        x.moves_out[2 * u64(i) + 1] = bc;
      }
      if (x.csize) {
        atomicSub(&x.csize[from], 1u);
        atomicAdd(&x.csize[bc], 1u);
      }
      t.gain += g;
      ++t.moves;
    } else {
      atomicAdd(&x.sigma[bc], -ku);
      mv = false;
    }
  }
  return mv;
}

// ---- bin 1: thread per vertex --------------------------------------------------
template <class V, bool DRY>
__global__ void __launch_bounds__(256) lm_thread(MoveArgs x, const u32* __restrict__ list,
                                                 u64 count) {
  Tally tl;
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < count;
       i += u64(gridDim.x) * blockDim.x) {
    const u32 u = list[i];
    if (!DRY) {
      if (x.prune && !x.flags[u]) continue;
      x.flags[u] = 0;
    }
    const u64 lo = x.g.off[u];
    const int d = int(x.g.off[u + 1] - lo);
    const u32 from = x.C[u];
    u32 t[kThreadMaxD], c[kThreadMaxD];
    V wv[kThreadMaxD];
#pragma unroll
    for (int k = 0; k < kThreadMaxD; ++k) {
      t[k] = kEmpty;
      c[k] = kEmpty;
      wv[k] = V(0);
      if (k < d) {
        t[k] = x.g.tgt[lo + k];
        wv[k] = V(x.g.w[lo + k]);
      }
    }
#pragma unroll
    for (int k = 0; k < kThreadMaxD; ++k)
      if (k < d && t[k] != u) c[k] = x.C[t[k]];
    V own = V(0);
#pragma unroll
    for (int k = 0; k < kThreadMaxD; ++k)
      if (c[k] == from) own += wv[k];
    const double ku = x.K[u], sf = x.sigma[from];
    double bg = -INFINITY, bk = 0.0;
    u32 bc = kEmpty;
#pragma unroll
    for (int k = 0; k < kThreadMaxD; ++k) {
      const u32 ck = c[k];
      bool first = ck != kEmpty && ck != from && key_ok(x, ck);
#pragma unroll
      for (int j = 0; j < k; ++j) first = first && c[j] != ck;
      V sum = V(0);  // row order, like the reference's serial scan
#pragma unroll
      for (int j = k; j < kThreadMaxD; ++j)
        if (c[j] == ck) sum += wv[j];
      if (first && (DRY || may_gain(x, double(sum), double(own), ku, sf))) {
        const double g = score<DRY, V>(x, double(sum), double(own), ku, x.sigma[ck], sf);
        ++tl.rand;
        if (better(g, ck, bg, bc)) bg = g, bc = ck, bk = double(sum);
      }
    }
    ++tl.verts;
    tl.arcs += d;
    tl.rand += d;
    if (decide<DRY>(x, u, from, ku, bc, bg, bk, double(own), tl) && x.prune) {
      tl.rand += d;
#pragma unroll
      for (int k = 0; k < kThreadMaxD; ++k)
        if (k < d) x.flags[t[k]] = 1;
    }
  }
  tl.flush(x);
}

// ---- shared scan / rank loops of the table kernels ----------------------------------
// Accumulate K_{u->c} over arcs [lo, hi) handled by `lane` of `stride` lanes, B
// arcs per lane per round: all B target/weight loads, then all B C[t] gathers,
// are issued before the first dependent use, so each lane keeps B independent
// memory requests in flight (the sweep is latency-bound otherwise).
//
// COMBINE (stride a multiple of 32, consecutive lanes on consecutive arcs):
// runs of equal adjacent communities among the 32 (community, weight) pairs a
// warp holds are summed first (warp_combine), so a run is merged into the
// table once. Late passes have few distinct neighbour communities per row;
// without this, all lanes of a block hammer the same few slots with CAS
// retries.
template <int B, bool COMBINE, class Tab, class V>
__device__ __forceinline__ void scan_arcs(const MoveArgs& x, const Tab& tab, u32 lg, u32 u, u32 from,
                                          u64 lo, u64 hi, u32 lane, u32 stride, V& own, u32* live,
                                          u32* nlive) {
  // the trip count is uniform across the lanes (COMBINE shuffles need every lane)
  for (u64 b0 = lo; b0 < hi; b0 += u64(stride) * B) {
    u32 t[B], c[B];
    V w[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const u64 a = b0 + lane + u64(k) * stride;
      t[k] = a < hi ? __ldcs(x.g.tgt + a) : u;  // out of range reads as a self-loop: skipped
      w[k] = a < hi ? V(arc_w(x.g, a)) : V(0);
    }
#pragma unroll
    for (int k = 0; k < B; ++k) c[k] = t[k] != u ? x.C[t[k]] : kEmpty;
#pragma unroll
    for (int k = 0; k < B; ++k) {
      bool tail = true;
      // sum runs of equal adjacent communities across the warp first
      if (COMBINE) tail = warp_combine(c[k], w[k], lane & 31);
      if (!tail || c[k] == kEmpty) continue;
      if (c[k] == from) {
        own += w[k];
      } else {
        const int slot = tab.insert(lg, c[k], w[k]);
        if (slot >= 0) live[atomicAdd(nlive, 1u)] = u32(slot);
      }
    }
  }
}

// Best live entry seen by this lane (B Sigma gathers in flight per round).
template <int B, bool DRY, class Tab>
__device__ __forceinline__ void rank_live(const MoveArgs& x, const Tab& tab, const u32* live, u32 n,
                                          u32 lane, u32 stride, double own, double ku, double sf,
                                          double& bg, u32& bc, double& bk) {
  for (u32 j0 = lane; j0 < n; j0 += stride * B) {
    u32 key[B];
    double val[B], sc[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const u32 j = j0 + k * stride;
      key[k] = kEmpty;
      val[k] = 0.0;
      if (j < n && !(tab.read(live[j], key[k], val[k]) && key_ok(x, key[k]) &&
                     (DRY || may_gain(x, val[k], own, ku, sf))))
        key[k] = kEmpty;
    }
#pragma unroll
    for (int k = 0; k < B; ++k) sc[k] = key[k] != kEmpty ? x.sigma[key[k]] : 0.0;
#pragma unroll
    for (int k = 0; k < B; ++k) {
      if (key[k] == kEmpty) continue;
      const double g = score<DRY, typename Tab::V>(x, val[k], own, ku, sc[k], sf);
      if (better(g, key[k], bg, bc)) bg = g, bc = key[k], bk = val[k];
    }
  }
}

// ---- bins 2 and 3: G lanes per vertex, smem table + live list per group ---------
template <class Tab, int G, int CAPLOG, int THREADS>
constexpr size_t group_smem() {
  return size_t(THREADS / G) * ((size_t(1) << CAPLOG) * Tab::kSlotBytes + (size_t(1) << (CAPLOG - 1)) * 4 + 16);
}

template <class Tab, int G, int CAPLOG, int THREADS, bool DRY>
__global__ void __launch_bounds__(THREADS, 4) lm_group(MoveArgs x, const u32* __restrict__ list,
                                                       u64 count) {
  using V = typename Tab::V;
  constexpr int GPB = THREADS / G;
  constexpr u32 CAP = 1u << CAPLOG;
  constexpr u32 LCAP = CAP / 2;
  constexpr u32 MINLOG = G == 8 ? 3 : 5;
  extern __shared__ __align__(16) unsigned char smem[];
  const auto tile = cg::tiled_partition<G>(cg::this_thread_block());
  const int gi = threadIdx.x / G;
  const u32 lane = tile.thread_rank();
  const Tab tab(smem + size_t(gi) * CAP * Tab::kSlotBytes, CAP);
  u32* live = reinterpret_cast<u32*>(smem + size_t(GPB) * CAP * Tab::kSlotBytes) + size_t(gi) * LCAP;
  u32* nlive = reinterpret_cast<u32*>(smem + size_t(GPB) * (CAP * Tab::kSlotBytes + LCAP * 4)) + gi;
  for (u32 s = lane; s < CAP; s += G) tab.clear(s);
  if (lane == 0) *nlive = 0;
  tile.sync();
  Tally tl;
  for (u64 i = blockIdx.x * u64(GPB) + gi; i < count; i += u64(gridDim.x) * GPB) {
    const u32 u = list[i];
    if (!DRY) {
      u32 act = 0;
      if (lane == 0) {
        act = !x.prune || x.flags[u];
        if (act) x.flags[u] = 0;
      }
      if (!tile.shfl(act, 0)) continue;
    }
    const u64 lo = x.g.off[u];
    const u64 d = x.g.off[u + 1] - lo;
    const u32 from = x.C[u];
    const u32 lg = table_log(d, MINLOG);
    if ((1u << lg) > CAP) {  // bin / table-capacity invariant
      if (lane == 0) atomicOr(x.err, u32(kErrTable));
      continue;
    }
    V own = V(0);
    scan_arcs<kBatch, G == 32>(x, tab, lg, u, from, lo, lo + d, lane, G, own, live, nlive);
    own = cg::reduce(tile, own, cg::plus<V>());
    tile.sync();
    const u32 n = *reinterpret_cast<volatile u32*>(nlive);
    const double ku = x.K[u], sf = x.sigma[from];
    double bg = -INFINITY, bk = 0.0;
    u32 bc = kEmpty;
    rank_live<kBatch, DRY>(x, tab, live, n, lane, G, double(own), ku, sf, bg, bc, bk);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const double og = tile.shfl_xor(bg, o);
      const u32 oc = tile.shfl_xor(bc, o);
      const double ok = tile.shfl_xor(bk, o);
      if (better(og, oc, bg, bc)) bg = og, bc = oc, bk = ok;
    }
    for (u32 j = lane; j < n; j += G) tab.clear(live[j]);
    u32 moved = 0;
    if (lane == 0) {
      *nlive = 0;
      ++tl.verts;
      tl.arcs += d;
      tl.rand += d + n;
      moved = decide<DRY>(x, u, from, ku, bc, bg, bk, double(own), tl);
    }
    if (!DRY && tile.shfl(moved, 0) && x.prune)
      for (u64 a = lo + lane; a < lo + d; a += G) x.flags[x.g.tgt[a]] = 1, ++tl.rand;
    tile.sync();
  }
  tl.flush(x);
}

// ---- sort bins: G lanes x K registers per vertex, register bitonic sort --------
// The (community, weight) pairs of a vertex's arcs are sorted by community
// across the G lanes of its group (element e lives in lane e / K, register
// e % K), so equal communities form adjacent runs, and a segmented scan leaves
// K_{u->c} on the last element of each run. The network is data-independent:
// every lane of a warp runs the same instruction stream (no atomics, no
// shared memory, no probe loops), which the hash kernels cannot achieve on
// short rows where each group's probing diverges. Row arcs are streamed with
// evict-first loads so the gathered C / Sigma lines keep their L2 residency.
//
// Software-pipelined one vertex deep: the loads of the group's next vertex
// (list entry, row bounds, own community, arcs, their communities, Sigma of
// the own community) are issued in stages between the compute steps of the
// current one (sort, Sigma gathers, scoring, decision), so each group keeps two
// vertices' dependent load chains in flight. The next vertex's gathers may
// miss the current vertex's move (one more source of the asynchrony the
// validated join already tolerates); the DRY path writes no state, so its
// results are unaffected.
template <int G, int K, class V, bool DRY>
__global__ void __launch_bounds__(256) lm_sort(MoveArgs x, const u32* __restrict__ list, u64 count) {
  constexpr int GPB = 256 / G;
  constexpr u32 FULL = 0xffffffffu;
  const u32 lane = threadIdx.x & (G - 1);
  const u32 gi = threadIdx.x / G;
  const u64 stride = u64(gridDim.x) * GPB;
  const ull keep = l2_keep_policy(x.l2_keep);
  Tally tl;
  // vertex in flight (the trip count is uniform across the block, so every
  // lane reaches every shuffle)
  u64 i0 = u64(blockIdx.x) * GPB;
  // full bin lists: a row whose prune flag is clear is a hole in the pipeline
  auto live = [&](u32 v) { return !x.full_lists || !x.prune || x.flags[v] != 0; };
  bool have = i0 + gi < count && live(list[i0 + gi]);
  u32 u = 0, from = kEmpty;
  u64 lo = 0, hi = 0;
  double ku = 0.0, sf = 0.0;
  u32 t[K], key[K];
  V val[K];
  if (have) {
    u = list[i0 + gi];
    lo = x.g.off[u];
    hi = x.g.off[u + 1];
    from = x.C[u];
    ku = x.K[u];
  }
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const u64 a = lo + u64(r) * G + lane;
    const bool ok = a < hi;
    t[r] = ok ? __ldcs(x.g.tgt + a) : kEmpty;
    val[r] = ok ? V(__ldcs(x.g.w + a)) : V(0);
  }
  if (have) sf = x.sigma[from];
#pragma unroll
  for (int r = 0; r < K; ++r) key[r] = (t[r] != kEmpty && t[r] != u) ? ld_keep(x.C + t[r], keep) : kEmpty;

  for (; i0 < count; i0 += stride) {
    // stage 1 (next): list entry
    const u64 in = i0 + stride + gi;
    const bool nhave = in < count;
    const u32 nu = nhave ? list[in] : 0u;

    // current: sort by community (padding and self-loops carry kEmpty and
    // sort last); K_{u->c} lands on the last element of each run
#pragma unroll
    for (int r = 0; r < K; ++r) tl.rand += key[r] != kEmpty ? 1 : 0;
    bitonic_sort<G, K, V>(key, val, lane);
    bool tail[K];
    segmented_runs<G, K, V>(key, val, tail, lane);
    const V (&run)[K] = val;

    // stage 2 (next): row bounds, own community, vertex weight
    u64 nlo = 0, nhi = 0;
    u32 nfrom = kEmpty;
    double nku = 0.0;
    if (nhave) {
      nlo = x.g.off[nu];
      nhi = x.g.off[nu + 1];
      nfrom = x.C[nu];
      nku = x.K[nu];
    }

    // current: own community weight, Sigma of the candidates
    V own_l = V(0);
    bool cand[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      if (tail[r] && key[r] == from) own_l = run[r];
      cand[r] = tail[r] && key[r] != kEmpty && key[r] != from;
    }
    V own = own_l;
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) own += __shfl_xor_sync(FULL, own, o, G);
    double sc[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      if (cand[r]) cand[r] = key_ok(x, key[r]) && (DRY || may_gain(x, double(run[r]), double(own), ku, sf));
      sc[r] = cand[r] ? ld_keep(x.sigma + key[r], keep) : 0.0;
      tl.rand += cand[r] ? 1 : 0;
    }

    // stage 3 (next): arcs
    u32 nt[K];
    V nval[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const u64 a = nlo + u64(r) * G + lane;
      const bool ok = a < nhi;
      nt[r] = ok ? __ldcs(x.g.tgt + a) : kEmpty;
      nval[r] = ok ? V(__ldcs(x.g.w + a)) : V(0);
    }

    // current: rank the candidates, group argmax
    double bg = -INFINITY, bk = 0.0;
    u32 bc = kEmpty;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      if (!cand[r]) continue;
      const double g = score<DRY, V>(x, double(run[r]), double(own), ku, sc[r], sf);
      if (better(g, key[r], bg, bc)) bg = g, bc = key[r], bk = double(run[r]);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      const double og = __shfl_xor_sync(FULL, bg, o, G);
      const u32 oc = __shfl_xor_sync(FULL, bc, o, G);
      const double ok = __shfl_xor_sync(FULL, bk, o, G);
      if (better(og, oc, bg, bc)) bg = og, bc = oc, bk = ok;
    }

    // stage 4 (next): communities of the arcs, Sigma of the own community
    u32 nkey[K];
#pragma unroll
    for (int r = 0; r < K; ++r) nkey[r] = (nt[r] != kEmpty && nt[r] != nu) ? ld_keep(x.C + nt[r], keep) : kEmpty;
    const double nsf = nhave ? x.sigma[nfrom] : 0.0;

    // current: decide and apply
    int moved = 0;
    if (have && lane == 0) {
      if (!DRY) x.flags[u] = 0;
      ++tl.verts;
      tl.arcs += hi - lo;
      moved = decide<DRY>(x, u, from, ku, bc, bg, bk, double(own), tl);
    }
    moved = __shfl_sync(FULL, moved, 0, G);
    if (!DRY && moved && x.prune) {
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (t[r] != kEmpty) x.flags[t[r]] = 1, ++tl.rand;
    }

    // rotate
    have = nhave, u = nu, lo = nlo, hi = nhi, from = nfrom, ku = nku, sf = nsf;
#pragma unroll
    for (int r = 0; r < K; ++r) t[r] = nt[r], key[r] = nkey[r], val[r] = nval[r];
  }
  tl.flush(x);
}

// ---- sort bins, packed keys (psort.cuh): the default when n < 2^(32 - LB) -------
// Same work split as lm_sort (G lanes x K registers per vertex) with fewer
// instructions per vertex: the network sorts 32-bit (community << LB | row
// position) keys and the weights are fetched once afterwards; run starts come
// from a ballot; the group argmax is three redux.sync for G = 32; the lane
// holding the winning candidate decides (no broadcast of gain and weight).
//
// Software pipeline, three vertices per group in flight. Iteration i:
//   targets + weights of i+1 | list entry of i+2 | sort i | C[t] of i+1 |
//   own weight + Sigma of i | row bounds of i+2 | rank, decide, mark i
// so every dependent load (list -> offsets -> targets -> communities) has a
// compute step of its own between issue and use. The targets of i and i+1 stay
// in registers for the neighbour marks. Gathers for i+1 may miss the move of
// i (asynchrony the validated join tolerates); DRY writes no state.
template <int G, int K, class V, bool DRY, bool U>
__global__ void __launch_bounds__(256, K == 1 ? 4 : (K <= 4 ? 3 : 2)) lm_psort(MoveArgs x, const u32* __restrict__ list, u64 count) {
  constexpr int GPB = 256 / G;
  constexpr int N = G * K;
  constexpr int LB = ilog2<N>();
  constexpr u32 FULL = 0xffffffffu;
  constexpr u32 GMASK = G == 32 ? FULL : ((1u << G) - 1u);
  __shared__ V vbuf[K > 1 ? 256 * K : 1];  // per group: weights in row order (K > 1)
  const u32 lane = threadIdx.x & (G - 1);
  const u32 gi = threadIdx.x / G;
  const u32 gshift = (threadIdx.x & 31u) & ~u32(G - 1);
  V* gbuf = vbuf + (K > 1 ? gi * N : 0);
  const ull dirs = psort_dirs<G, K>(lane);
  const u64 stride = u64(gridDim.x) * GPB;
  const ull keep = l2_keep_policy(x.l2_keep);
  Tally tl;

  auto load_row = [&](u32 v, u64 rlo, u64 rhi, u32 (&t)[K], V (&w)[K]) {
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const u64 a = rlo + u64(r) * G + lane;
      const bool ok = a < rhi;
      t[r] = ok ? __ldcs(x.g.tgt + a) : kEmpty;
      w[r] = ok ? V(__ldcs(x.g.w + a)) : V(0);
    }
  };
  // padding carries no key; a self-loop keeps its place in the row as a
  // zero-weight element of u's own community (K_{u->c} excludes self-loops,
  // louvain_compact.cpp:46), so rows stored sorted by target stay sorted
  // U (every arc weight equals x.uniform_w): the key is the community alone,
  // so any n fits, and self-loops are dropped
  auto gather = [&](u32 v, u32 vfrom, const u32 (&t)[K], u32 (&key)[K], V (&w)[K]) {
#pragma unroll
    for (int r = 0; r < K; ++r) {
      if (U) {
        key[r] = (t[r] != kEmpty && t[r] != v) ? ld_keep(x.C + t[r], keep) : kNoKey;
      } else {
        const u32 c = t[r] == v ? vfrom : (t[r] != kEmpty ? ld_keep(x.C + t[r], keep) : 0u);
        key[r] = t[r] != kEmpty ? (c << LB) | u32(r * G + lane) : kNoKey;
        if (t[r] == v) w[r] = V(0);
      }
    }
  };

  // prologue: vertex i fully loaded, vertex i+1's header
  u64 i0 = u64(blockIdx.x) * GPB;
  // full bin lists: a row whose prune flag is clear is a hole in the pipeline
  auto live = [&](u32 v) { return !x.full_lists || !x.prune || x.flags[v] != 0; };
  bool have = i0 + gi < count && live(list[i0 + gi]);
  u32 u = 0, from = kEmpty;
  u64 lo = 0, hi = 0;
  double ku = 0.0, sf = 0.0;
  u32 key[K], t[K];
  V val[K];
  if (have) {
    u = list[i0 + gi];
    lo = x.g.off[u];
    hi = x.g.off[u + 1];
    from = x.C[u];
    ku = x.K[u];
  }
  load_row(u, lo, hi, t, val);
  if (have) sf = x.sigma[from];
  gather(u, from, t, key, val);
  bool have1 = i0 + stride + gi < count && live(list[i0 + stride + gi]);
  u32 u1 = 0, from1 = kEmpty;
  u64 lo1 = 0, hi1 = 0;
  double ku1 = 0.0;
  if (have1) {
    u1 = list[i0 + stride + gi];
    lo1 = x.g.off[u1];
    hi1 = x.g.off[u1 + 1];
    from1 = x.C[u1];
    ku1 = x.K[u1];
  }

  for (; i0 < count; i0 += stride) {
    // (i+1) targets and weights; (i+2) list entry
    u32 t1[K], key1[K];
    V val1[K];
    load_row(u1, lo1, hi1, t1, val1);
    const u64 in2 = i0 + 2 * stride + gi;
    const u32 u2 = in2 < count ? list[in2] : 0u;
    const bool have2 = in2 < count && live(u2);

    // (i) group the arcs by community, fetch the weights in sorted order
    // rows whose communities already ascend in row order (every row in the
    // first sweep of a pass: rows are stored sorted by target and C is the
    // identity) skip the network and take the row-order run sums
    bool rows = true;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const u32 nxt = __shfl_down_sync(FULL, key[r], 1, G);
      const u32 wrap = r + 1 < K ? __shfl_sync(FULL, key[r + 1], 0, G) : kNoKey;
      rows = rows && key[r] <= (lane + 1 < u32(G) ? nxt : wrap);
    }
    rows = __all_sync(FULL, rows);
    if (!rows) {
      if (K > 1 && !U) {
        __syncwarp();
#pragma unroll
        for (int r = 0; r < K; ++r) gbuf[r * G + lane] = val[r];
        __syncwarp();
      }
      psort<G, K>(key, dirs);
    }
    u32 ck[K];
    V run[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const u32 pos = key[r] & u32(N - 1);
      V w;
      if (U) w = V(x.uniform_w);
      else if (rows) w = val[r];
      else if (K == 1) w = __shfl_sync(FULL, val[0], pos, G);
      else w = gbuf[pos];
      ck[r] = key[r] == kNoKey ? kEmpty : (U ? key[r] : key[r] >> LB);
      run[r] = key[r] == kNoKey ? V(0) : w;
    }
    bool tail[K];
    if (rows) prun_sums_rows<G, K, V>(ck, run, tail, lane, gshift);
    else prun_sums<G, K, V>(ck, run, tail, lane, gshift);

    // (i+1) communities of its arcs, Sigma of its community
    gather(u1, from1, t1, key1, val1);
    const double sf1 = have1 ? x.sigma[from1] : 0.0;

    // (i) weight to the own community (one run tail in the group holds it),
    // Sigma of the candidates
    V own_l = V(0);
    bool has_own = false, cand[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      if (tail[r] && ck[r] == from) own_l = run[r], has_own = true;
      cand[r] = tail[r] && ck[r] != kEmpty && ck[r] != from;
    }
    const u32 ob = (__ballot_sync(FULL, has_own) >> gshift) & GMASK;
    const V own_s = __shfl_sync(FULL, own_l, ob ? __ffs(ob) - 1 : 0, G);
    const V own = ob ? own_s : V(0);
    double sc[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      if (cand[r]) cand[r] = key_ok(x, ck[r]) && (DRY || may_gain(x, double(run[r]), double(own), ku, sf));
      sc[r] = cand[r] ? ld_keep(x.sigma + ck[r], keep) : 0.0;
      tl.rand += cand[r] ? 1 : 0;
    }

    // (i+2) row bounds, community, vertex weight
    u64 lo2 = 0, hi2 = 0;
    u32 from2 = kEmpty;
    double ku2 = 0.0;
    if (have2) {
      lo2 = x.g.off[u2];
      hi2 = x.g.off[u2 + 1];
      from2 = x.C[u2];
      ku2 = x.K[u2];
    }

    // (i) rank the candidates, group argmax; the lane holding the best
    // candidate (lane 0 if none) decides
    double bg = -INFINITY, bk = 0.0;
    u32 bc = kEmpty;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      if (!cand[r]) continue;
      const double g = score<DRY, V>(x, double(run[r]), double(own), ku, sc[r], sf);
      if (better(g, ck[r], bg, bc)) bg = g, bc = ck[r], bk = double(run[r]);
    }
    const u32 best = group_best<G>(bg, bc);
    const bool decider = have && (best == kEmpty ? lane == 0 : bc == best);
    bool moved = false;
    if (decider) {
      if (!DRY) x.flags[u] = 0;
      ++tl.verts;
      tl.arcs += hi - lo;
      tl.rand += hi - lo;  // C[t] gathers (one per arc)
      moved = decide<DRY>(x, u, from, ku, best, best == kEmpty ? -INFINITY : bg, bk, double(own), tl);
    }
    if (!DRY && x.prune && ((__ballot_sync(FULL, moved) >> gshift) & GMASK)) {
#pragma unroll
      for (int r = 0; r < K; ++r)  // every arc target, u itself on a self-loop (louvain_compact.cpp:160-161)
        if (t[r] != kEmpty) x.flags[t[r]] = 1, ++tl.rand;
    }

    // rotate: i <- i+1 <- i+2
    have = have1, u = u1, lo = lo1, hi = hi1, from = from1, ku = ku1, sf = sf1;
    have1 = have2, u1 = u2, lo1 = lo2, hi1 = hi2, from1 = from2, ku1 = ku2;
#pragma unroll
    for (int r = 0; r < K; ++r) key[r] = key1[r], val[r] = val1[r], t[r] = t1[r];
  }
  tl.flush(x);
}

// ---- sort bins, match variant: warp per vertex, K arcs per lane ----------------
// Equal communities among the 32 arcs of one register round are found with
// one match.any; the lowest lane of each peer set (the leader) sums the peers'
// weights in ascending lane (= row) order from a per-warp smem buffer. With
// K = 1 the leaders are the candidates. With K > 1 the leaders of every round
// merge their partial sums into a per-warp smem table: keys are distinct
// within a round, so a claim never races another lane of the warp for a key.
// Pipelined across vertices like lm_sort.
template <int K, class Tab>
constexpr size_t match_smem() {
  constexpr size_t cap = K > 1 ? size_t(64) * K : 0;
  return 8 * (32 * sizeof(typename Tab::V) + cap * Tab::kSlotBytes + cap / 2 * 4);
}

template <int K, class Tab, bool DRY>
__global__ void __launch_bounds__(256) lm_match(MoveArgs x, const u32* __restrict__ list, u64 count) {
  using V = typename Tab::V;
  constexpr u32 FULL = 0xffffffffu;
  constexpr u32 CAP = K > 1 ? 64u * K : 1u;
  constexpr int WPB = 8;
  extern __shared__ __align__(16) unsigned char smem[];
  const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const u32 lt = (1u << lane) - 1u;
  V* buf = reinterpret_cast<V*>(smem) + wid * 32;
  unsigned char* tb = smem + WPB * 32 * sizeof(V) + size_t(wid) * (CAP * Tab::kSlotBytes + CAP / 2 * 4);
  const Tab tab(tb, CAP);
  u32* live = reinterpret_cast<u32*>(tb + CAP * Tab::kSlotBytes);
  if (K > 1)
    for (u32 j = lane; j < CAP; j += 32) tab.clear(j);
  __syncwarp();
  const u64 stride = u64(gridDim.x) * WPB;
  Tally tl;
  u64 i0 = u64(blockIdx.x) * WPB;
  bool have = i0 + wid < count;
  u32 u = 0, from = kEmpty;
  u64 lo = 0, hi = 0;
  double ku = 0.0, sf = 0.0;
  u32 t[K], key[K];
  V val[K];
  if (have) {
    u = list[i0 + wid];
    lo = x.g.off[u];
    hi = x.g.off[u + 1];
    from = x.C[u];
    ku = x.K[u];
  }
#pragma unroll
  for (int r = 0; r < K; ++r) {
    const u64 a = lo + u64(r) * 32 + lane;
    const bool ok = a < hi;
    t[r] = ok ? __ldcs(x.g.tgt + a) : kEmpty;
    val[r] = ok ? V(__ldcs(x.g.w + a)) : V(0);
  }
  if (have) sf = x.sigma[from];
#pragma unroll
  for (int r = 0; r < K; ++r) key[r] = (t[r] != kEmpty && t[r] != u) ? x.C[t[r]] : kEmpty;

  for (; i0 < count; i0 += stride) {
    // stage 1 (next)
    const u64 in = i0 + stride + wid;
    const bool nhave = in < count;
    const u32 nu = nhave ? list[in] : 0u;

    // current: per-round peer sums
    V own_l = V(0);
    u32 ckey = kEmpty;  // K == 1: this lane's candidate
    V cval = V(0);
    u32 n = 0;          // K > 1: live entries
    const u32 lg = K > 1 ? table_log(hi - lo, 5) : 0;
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const u32 peers = __match_any_sync(FULL, key[r]);
      const bool lead = key[r] != kEmpty && (peers & lt) == 0;
      buf[lane] = val[r];
      __syncwarp();
      V sum = V(0);
      if (lead)
        for (u32 m = peers; m; m &= m - 1) sum += buf[__ffs(m) - 1];
      __syncwarp();
      bool fresh = false;
      int slot = -1;
      if (lead) {
        if (key[r] == from) {
          own_l += sum;
        } else if (K == 1) {
          ckey = key[r], cval = sum;
        } else {
          slot = tab.insert(lg, key[r], sum);
          fresh = slot >= 0;
        }
      }
      if (K > 1) {
        const u32 nb = __ballot_sync(FULL, fresh);
        if (fresh) live[n + __popc(nb & lt)] = u32(slot);
        n += __popc(nb);
      }
    }
    V own = own_l;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) own += __shfl_xor_sync(FULL, own, o);

    // stage 2 (next)
    u64 nlo = 0, nhi = 0;
    u32 nfrom = kEmpty;
    double nku = 0.0;
    if (nhave) {
      nlo = x.g.off[nu];
      nhi = x.g.off[nu + 1];
      nfrom = x.C[nu];
      nku = x.K[nu];
    }

    double bg = -INFINITY, bk = 0.0;
    u32 bc = kEmpty;
    if (K == 1) {
      const bool cand = ckey != kEmpty && key_ok(x, ckey);
      const double sc = cand ? x.sigma[ckey] : 0.0;
      if (cand) {
        bg = score<DRY, V>(x, double(cval), double(own), ku, sc, sf);
        bc = ckey, bk = double(cval);
      }
    } else {
      __syncwarp();
      rank_live<2, DRY>(x, tab, live, n, lane, 32, double(own), ku, sf, bg, bc, bk);
    }

    // stage 3 (next)
    u32 nt[K];
    V nval[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      const u64 a = nlo + u64(r) * 32 + lane;
      const bool ok = a < nhi;
      nt[r] = ok ? __ldcs(x.g.tgt + a) : kEmpty;
      nval[r] = ok ? V(__ldcs(x.g.w + a)) : V(0);
    }

#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double og = __shfl_xor_sync(FULL, bg, o);
      const u32 oc = __shfl_xor_sync(FULL, bc, o);
      const double ok = __shfl_xor_sync(FULL, bk, o);
      if (better(og, oc, bg, bc)) bg = og, bc = oc, bk = ok;
    }
    if (K > 1) {
      for (u32 j = lane; j < n; j += 32) tab.clear(live[j]);
      __syncwarp();
    }

    // stage 4 (next)
    u32 nkey[K];
#pragma unroll
    for (int r = 0; r < K; ++r) nkey[r] = (nt[r] != kEmpty && nt[r] != nu) ? x.C[nt[r]] : kEmpty;
    const double nsf = nhave ? x.sigma[nfrom] : 0.0;

    int moved = 0;
    if (have && lane == 0) {
      if (!DRY) x.flags[u] = 0;
      ++tl.verts;
      tl.arcs += hi - lo;
      tl.rand += hi - lo + n;
      moved = decide<DRY>(x, u, from, ku, bc, bg, bk, double(own), tl);
    }
    moved = __shfl_sync(FULL, moved, 0);
    if (!DRY && moved && x.prune) {
#pragma unroll
      for (int r = 0; r < K; ++r)
        if (t[r] != kEmpty) x.flags[t[r]] = 1, ++tl.rand;
    }

    have = nhave, u = nu, lo = nlo, hi = nhi, from = nfrom, ku = nku, sf = nsf;
#pragma unroll
    for (int r = 0; r < K; ++r) t[r] = nt[r], key[r] = nkey[r], val[r] = nval[r];
  }
  tl.flush(x);
}

// ---- bins 4 and 5: block per vertex, table in smem (4) or global memory (5) -----
template <class Tab>
constexpr size_t block_smem() {
  return (size_t(1) << kBlockCapLog) * Tab::kSlotBytes + (size_t(1) << (kBlockCapLog - 1)) * 4;
}
// lm_block also stages the row: 4096 (community, f32 weight) pairs
template <class Tab>
constexpr size_t block_stage_smem() {
  return block_smem<Tab>() + (size_t(1) << (kBlockCapLog - 1)) * 8;
}

// Sub-groups: the block runs SUB independent groups of kBlockThreads / SUB
// threads, each deciding its own vertex with its own slice of the smem table
// (8192 / SUB slots, rows up to 4096 / SUB arcs) and synchronising on its own
// named barrier, so a group never waits for another group's vertex. SUB = 4
// takes rows of 257..1024 arcs (four vertices in flight per block instead of
// one: per vertex the block is latency-bound on its dependent chain
// list -> row -> communities -> table -> Sigma -> join, and barrier-bound when
// a long row's 512 threads wait on a short one); SUB = 1 takes 1025..4096.
template <int SUB>
__device__ __forceinline__ void sub_sync(u32 g) {
  if (SUB == 1) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(kBlockThreads / SUB) : "memory");
  }
}

template <class Tab, bool DRY, int SUB>
__global__ void __launch_bounds__(kBlockThreads) lm_block(MoveArgs x, const u32* __restrict__ list,
                                                          u64 count, u64 dmin, u64 dmax) {
  using V = typename Tab::V;
  constexpr int ST = kBlockThreads / SUB;  // threads of a sub-group
  constexpr int W = ST / 32;               // warps of a sub-group
  constexpr int CAPLOG = kBlockCapLog - (SUB == 1 ? 0 : SUB == 2 ? 1 : SUB == 4 ? 2 : 3);
  constexpr u32 CAP = 1u << CAPLOG;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ V red_v[SUB][W];
  __shared__ double red_g[SUB][W], red_k[SUB][W];
  __shared__ u32 red_c[SUB][W];
  __shared__ u32 bcast[SUB], nlive[SUB], sorted_flag[SUB];
  const u32 g = threadIdx.x / ST, lt = threadIdx.x % ST;
  // sub-group slices: table, live list, stage (communities, weights)
  unsigned char* tbase = smem + size_t(g) * CAP * Tab::kSlotBytes;
  const Tab tab(tbase, CAP);
  u32* live = reinterpret_cast<u32*>(smem + size_t(SUB) * CAP * Tab::kSlotBytes) + size_t(g) * (CAP / 2);
  u32* st_c = reinterpret_cast<u32*>(smem + size_t(SUB) * CAP * Tab::kSlotBytes) + size_t(SUB) * (CAP / 2) +
              size_t(g) * (CAP / 2);
  float* st_w = reinterpret_cast<float*>(reinterpret_cast<u32*>(smem + size_t(SUB) * CAP * Tab::kSlotBytes) +
                                         size_t(2 * SUB) * (CAP / 2)) + size_t(g) * (CAP / 2);
  const int lane = threadIdx.x & 31, wid = lt >> 5;
  for (u32 sl = lt; sl < CAP; sl += ST) tab.clear(sl);
  if (lt == 0) nlive[g] = 0;
  sub_sync<SUB>(g);
  Tally tl;
  for (u64 i = u64(blockIdx.x) * SUB + g; i < count; i += u64(gridDim.x) * SUB) {
    const u32 u = list[i];
    const u64 lo = x.g.off[u];
    const u64 d = x.g.off[u + 1] - lo;
    if (d <= dmin || d > dmax) continue;  // the other sub-group width takes it
    if (!DRY) {
      if (lt == 0) {
        const u32 act = !x.prune || x.flags[u];
        if (act) x.flags[u] = 0;
        bcast[g] = act;
      }
      sub_sync<SUB>(g);
      const u32 act = bcast[g];
      sub_sync<SUB>(g);
      if (!act) continue;
    }
    const u32 from = x.C[u];
    const u32 lg = table_log(d, 5);
    if (lg > u32(CAPLOG)) {  // capacity invariant
      if (lt == 0) atomicOr(x.err, u32(kErrTable));
      continue;
    }
    // stage the row's (community, weight) pairs in smem (coalesced loads, B
    // gathers in flight per thread); a self-loop is staged as a zero-weight
    // entry of u's own community, so rows stored sorted by target under an
    // ascending C (every row of a pass's first sweep) stay strictly ascending
    V own = V(0);
    bool up = true;
    for (u64 b0 = 0; b0 < d; b0 += u64(ST) * kBatch) {
      u32 t[kBatch];
      float w[kBatch];
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        const u64 e = b0 + lt + u64(k) * ST;
        t[k] = e < d ? __ldcs(x.g.tgt + lo + e) : kEmpty;
        w[k] = e < d ? arc_w(x.g, lo + e) : 0.f;
      }
#pragma unroll
      for (int k = 0; k < kBatch; ++k) {
        const u64 e = b0 + lt + u64(k) * ST;
        if (t[k] == kEmpty) continue;
        const u32 c = t[k] == u ? from : x.C[t[k]];
        if (t[k] == u) w[k] = 0.f;
        if (c == from) own += V(w[k]);
        st_c[e] = c;
        st_w[e] = w[k];
      }
    }
    if (lt == 0) sorted_flag[g] = 1;
    sub_sync<SUB>(g);
    for (u64 e = lt; e + 1 < d; e += ST) up = up && st_c[e] < st_c[e + 1];
    if (!up) sorted_flag[g] = 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) own += __shfl_xor_sync(0xffffffffu, own, o);
    if (lane == 0) red_v[g][wid] = own;
    sub_sync<SUB>(g);
    const bool rows_sorted = sorted_flag[g] != 0;
    if (!rows_sorted) {
      // merge the staged pairs into the table, combining duplicates per warp round
      for (u64 e0 = 0; e0 < d; e0 += ST) {
        const u64 e = e0 + lt;
        u32 c = e < d ? st_c[e] : kEmpty;
        V w = e < d ? V(st_w[e]) : V(0);
        if (c == from) c = kEmpty;
        if (!warp_combine(c, w, u32(lane))) c = kEmpty;
        if (c != kEmpty) {
          const int slot = tab.insert(lg, c, w);
          if (slot >= 0) live[atomicAdd(&nlive[g], 1u)] = u32(slot);
        }
      }
    }
    sub_sync<SUB>(g);
    V own_all = V(0);
#pragma unroll
    for (int k = 0; k < W; ++k) own_all += red_v[g][k];
    const u32 n = rows_sorted ? u32(d) : nlive[g];
    const double ku = x.K[u], sf = x.sigma[from];
    double bg = -INFINITY, bk = 0.0;
    u32 bc = kEmpty;
    if (rows_sorted) {
      // every staged entry is its own community: rank them directly
      for (u32 j0 = lt; j0 < n; j0 += ST * kBatch) {
        u32 key[kBatch];
        double val[kBatch], sc[kBatch];
#pragma unroll
        for (int k = 0; k < kBatch; ++k) {
          const u32 j = j0 + k * ST;
          key[k] = j < n ? st_c[j] : kEmpty;
          val[k] = j < n ? double(V(st_w[j])) : 0.0;
          if (key[k] == from || (key[k] != kEmpty && !(key_ok(x, key[k]) &&
                                                      (DRY || may_gain(x, val[k], double(own_all), ku, sf)))))
            key[k] = kEmpty;
        }
#pragma unroll
        for (int k = 0; k < kBatch; ++k) sc[k] = key[k] != kEmpty ? x.sigma[key[k]] : 0.0;
#pragma unroll
        for (int k = 0; k < kBatch; ++k) {
          if (key[k] == kEmpty) continue;
          const double gk = score<DRY, V>(x, val[k], double(own_all), ku, sc[k], sf);
          if (better(gk, key[k], bg, bc)) bg = gk, bc = key[k], bk = val[k];
        }
      }
    } else {
      rank_live<kBatch, DRY>(x, tab, live, n, lt, ST, double(own_all), ku, sf, bg, bc, bk);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double og = __shfl_xor_sync(0xffffffffu, bg, o);
      const u32 oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
      if (better(og, oc, bg, bc)) bg = og, bc = oc, bk = ok;
    }
    if (lane == 0) red_g[g][wid] = bg, red_c[g][wid] = bc, red_k[g][wid] = bk;
    sub_sync<SUB>(g);
    if (!rows_sorted)
      for (u32 j = lt; j < n; j += ST) tab.clear(live[j]);
    if (lt == 0) {
      for (int k = 1; k < W; ++k)
        if (better(red_g[g][k], red_c[g][k], bg, bc)) bg = red_g[g][k], bc = red_c[g][k], bk = red_k[g][k];
      nlive[g] = 0;
      ++tl.verts;
      tl.arcs += d;
      tl.rand += d + n;
      bcast[g] = decide<DRY>(x, u, from, ku, bc, bg, bk, double(own_all), tl);
    }
    sub_sync<SUB>(g);
    if (!DRY && bcast[g] && x.prune)
      for (u64 a = lo + lt; a < lo + d; a += ST) x.flags[x.g.tgt[a]] = 1, ++tl.rand;
    sub_sync<SUB>(g);
  }
  tl.flush(x);
}

// ---- hubs (kBinGlobal): a hub's row is split into chunks of kHubChunk arcs --------
// so that many blocks share one hub instead of one block walking millions of
// arcs (the reference's team sweep processes hubs across the whole thread team
// for the same reason, louvain_compact.cpp:80-114, 165-205).
//   lm_hub_chunks  block per chunk: K_{u->c} of the chunk in an smem table (own
//                  community privatised), flushed into the hub's HBM table
//                  (claim by CAS, L2 reductions, live-slot list)
//   lm_hub_rank    block per chunk-sized slice of a hub's live entries: best
//                  candidate of the slice, slots restored to empty
//   lm_hub_decide  warp per hub: best of its slices, the validated move
//   lm_hub_mark    block per chunk: neighbour marks of the hubs that moved
// Every phase spreads a hub over as many blocks as it has chunks: the
// million-arc hubs of web graphs no longer leave one block ranking (or
// marking) millions of entries while the rest of the GPU idles.
#ifndef LVN_HUB_CHUNK_LOG
#define LVN_HUB_CHUNK_LOG 11
#endif
constexpr u32 kHubChunk = 1u << LVN_HUB_CHUNK_LOG;  // arcs of one chunk
constexpr int kHubCapLog = LVN_HUB_CHUNK_LOG + 1;   // its smem table: 2 slots per arc
template <class Tab>
constexpr size_t hub_smem() {
  return (size_t(1) << kHubCapLog) * Tab::kSlotBytes + (size_t(1) << (kHubCapLog - 1)) * 4;
}

__host__ __device__ __forceinline__ u64 hub_slots(u64 deg, u32 n) {
  const u64 distinct = deg < n ? deg : n;
  const u32 l = ceil_log2_u64(2 * (distinct ? distinct : 1));
  return u64(1) << (l > 5 ? l : 5);
}

template <class Tab>
__host__ __device__ __forceinline__ u64 hub_region_bytes(u64 slots) {
  return (slots * Tab::kSlotBytes + slots / 2 * 4 + 15) & ~u64(15);
}

template <class Tab>
__global__ void hub_plan_k(const u32* __restrict__ hubs, u64 count, DGraph g, u32* __restrict__ index,
                           u64* __restrict__ bytes) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < count; i += u64(gridDim.x) * blockDim.x) {
    const u32 u = hubs[i];
    index[u] = u32(i);
    bytes[i] = hub_region_bytes<Tab>(hub_slots(g.off[u + 1] - g.off[u], g.n));
  }
}

template <class Tab>
__global__ void hub_clear_k(const u32* __restrict__ hubs, u64 count, DGraph g, const u64* __restrict__ tab_off,
                            unsigned char* tables) {
  for (u64 i = blockIdx.x; i < count; i += gridDim.x) {
    const u32 u = hubs[i];
    const u64 slots = hub_slots(g.off[u + 1] - g.off[u], g.n);
    const Tab tab(tables + tab_off[i], slots);
    for (u64 s = threadIdx.x; s < slots; s += blockDim.x) tab.clear(u32(s));
  }
}

// (full bin lists: a hub whose prune flag is clear gets no chunk, and no decision)
__global__ void hub_chunk_counts_k(const u32* __restrict__ hubs, u64 count, const u64* __restrict__ off,
                                   u32* __restrict__ chunks, const u8* __restrict__ skip_clear) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < count; i += u64(gridDim.x) * blockDim.x) {
    const u32 u = hubs[i];
    chunks[i] = skip_clear && !skip_clear[u] ? 0u : u32((off[u + 1] - off[u] + kHubChunk - 1) / kHubChunk);
  }
}

// chunk_hub[v] = the hub of chunk v (chunks of hub i: [chunk_off[i], chunk_off[i+1]))
__global__ void hub_chunk_owner_k(const u64* __restrict__ chunk_off, u64 count, u32* __restrict__ chunk_hub) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < count; i += u64(gridDim.x) * blockDim.x)
    for (u64 v = chunk_off[i]; v < chunk_off[i + 1]; ++v) chunk_hub[v] = u32(i);
}

// Chunk schedule interleaving the hubs by position in their rows (opt-in,
// LVN_HUB_INTERLEAVE=1): key = the chunk's fractional position in its hub's
// row, so chunks in flight together cover the same target-id range of every
// hub (rows are sorted by target) and their C / Sigma gathers share L2 lines;
// entries past the last chunk sort last
__global__ void hub_order_keys_k(const u64* __restrict__ chunk_off, const u32* __restrict__ chunk_hub, u64 count,
                                 u64 cap, u32* __restrict__ key, u32* __restrict__ val) {
  const u64 total = chunk_off[count];
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < cap; i += u64(gridDim.x) * blockDim.x) {
    u32 k = 0xFFFFFFFFu;
    if (i < total) {
      const u64 h = chunk_hub[i];
      const u64 c0 = chunk_off[h], nc = chunk_off[h + 1] - c0;
      k = u32(((i - c0) << 24) / nc);
    }
    key[i] = k;
    val[i] = u32(i);
  }
}

template <class Tab>
__global__ void __launch_bounds__(kBlockThreads) lm_hub_chunks(MoveArgs x, const u32* __restrict__ hubs,
                                                               u64 count, const u64* __restrict__ chunk_off,
                                                               const u32* __restrict__ chunk_hub,
                                                               const u32* __restrict__ order) {
  using V = typename Tab::V;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ u32 nlive;
  __shared__ V red[kBlockThreads / 32];
  const Tab stab(smem, u64(1) << kHubCapLog);
  u32* slive = reinterpret_cast<u32*>(smem + (size_t(1) << kHubCapLog) * Tab::kSlotBytes);
  for (u32 s = threadIdx.x; s < (1u << kHubCapLog); s += kBlockThreads) stab.clear(s);
  if (threadIdx.x == 0) nlive = 0;
  __syncthreads();
  const u64 total = chunk_off[count];
  for (u64 i = blockIdx.x; i < total; i += gridDim.x) {
    const u64 v = order ? order[i] : i;
    const u64 lo = chunk_hub[v];  // hub of chunk v
    const u32 u = hubs[lo];
    const u32 pi = x.hub_index[u];
    const u64 row = x.g.off[u], row_end = x.g.off[u + 1];
    const u64 a0 = row + (v - chunk_off[lo]) * kHubChunk;
    const u64 a1 = min(a0 + kHubChunk, row_end);
    const u32 from = x.C[u];
    V own = V(0);
    scan_arcs<kBatch, true>(x, stab, u32(kHubCapLog), u, from, a0, a1, threadIdx.x, kBlockThreads, own, slive,
                      &nlive);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) own += __shfl_xor_sync(0xffffffffu, own, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = own;
    __syncthreads();
    if (threadIdx.x == 0) {
      V t = V(0);
      for (int w = 0; w < kBlockThreads / 32; ++w) t += red[w];
      if (t != V(0)) atomicAdd(static_cast<V*>(x.hub_own) + pi, t);
    }
    const u64 slots = hub_slots(row_end - row, x.g.n);
    unsigned char* base = x.hub_tables + x.hub_tab_off[pi];
    const Tab gtab(base, slots);
    u32* glive = reinterpret_cast<u32*>(base + slots * Tab::kSlotBytes);
    const u32 glg = ceil_log2_u64(slots);
    const u32 n = nlive;
    for (u32 j = threadIdx.x; j < n; j += kBlockThreads) {
      const u32 s = slive[j];
      u32 key;
      double val;
      stab.read(s, key, val);
      const int gs = gtab.insert(glg, key, V(val));
      if (gs >= 0) glive[atomicAdd(&x.hub_live[pi], 1u)] = u32(gs);
      stab.clear(s);
    }
    __syncthreads();
    if (threadIdx.x == 0) nlive = 0;
    __syncthreads();
  }
}

// Best candidate of one slice of a hub's live entries (the slice of chunk v:
// entries [(v - chunk_off[i]) kHubChunk, +kHubChunk) of hub i), so a hub with
// millions of distinct communities is ranked by hundreds of blocks instead of
// one; the slice's slots are restored to empty after the read.
struct HubBest {
  double g, k;
  u32 c, pad;
};

template <class Tab, bool DRY>
__global__ void __launch_bounds__(kBlockThreads) lm_hub_rank(MoveArgs x, const u32* __restrict__ hubs, u64 count,
                                                             const u64* __restrict__ chunk_off,
                                                             const u32* __restrict__ chunk_hub,
                                                             HubBest* __restrict__ best) {
  using V = typename Tab::V;
  constexpr int W = kBlockThreads / 32;
  __shared__ double red_g[W], red_k[W];
  __shared__ u32 red_c[W];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const u64 total = chunk_off[count];
  for (u64 v = blockIdx.x; v < total; v += gridDim.x) {
    const u64 lo = chunk_hub[v];  // hub of chunk v
    const u32 u = hubs[lo];
    const u32 pi = x.hub_index[u];
    const u64 d = x.g.off[u + 1] - x.g.off[u];
    const u32 n = x.hub_live[pi];
    const u64 j0 = (v - chunk_off[lo]) * kHubChunk;
    double bg = -INFINITY, bk = 0.0;
    u32 bc = kEmpty;
    const u64 slots = hub_slots(d, x.g.n);
    unsigned char* base = x.hub_tables + x.hub_tab_off[pi];
    const Tab gtab(base, slots);
    const u32* glive = reinterpret_cast<const u32*>(base + slots * Tab::kSlotBytes);
    const u32 m = j0 < n ? u32(n - j0 < kHubChunk ? n - j0 : u64(kHubChunk)) : 0u;
    if (m) {
      const u32 from = x.C[u];
      const double own = double(static_cast<const V*>(x.hub_own)[pi]);
      const double ku = x.K[u], sf = x.sigma[from];
      rank_live<kBatch, DRY>(x, gtab, glive + j0, m, threadIdx.x, kBlockThreads, own, ku, sf, bg, bc, bk);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double og = __shfl_xor_sync(0xffffffffu, bg, o);
      const u32 oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
      if (better(og, oc, bg, bc)) bg = og, bc = oc, bk = ok;
    }
    if (lane == 0) red_g[wid] = bg, red_c[wid] = bc, red_k[wid] = bk;
    __syncthreads();
    for (u32 j = threadIdx.x; j < m; j += kBlockThreads) gtab.clear(glive[j0 + j]);
    if (threadIdx.x == 0) {
      for (int k = 1; k < W; ++k)
        if (better(red_g[k], red_c[k], bg, bc)) bg = red_g[k], bc = red_c[k], bk = red_k[k];
      best[v] = HubBest{bg, bk, bc, m};
    }
    __syncthreads();
  }
}

// Per hub (a warp each): the best of its slices, the validated move; the
// hub's state (live count, own weight) is reset for the next sweep and
// moved[i] tells lm_hub_mark whether to flag the hub's neighbours.
template <class Tab, bool DRY>
__global__ void lm_hub_decide(MoveArgs x, const u32* __restrict__ hubs, u64 count,
                              const u64* __restrict__ chunk_off, const HubBest* __restrict__ best,
                              u8* __restrict__ moved) {
  using V = typename Tab::V;
  const int lane = threadIdx.x & 31;
  Tally tl;
  const u64 warps = u64(gridDim.x) * (blockDim.x >> 5);
  for (u64 i = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5; i < count; i += warps) {
    if (chunk_off[i] == chunk_off[i + 1]) continue;  // inactive (full lists); a hub has arcs
    double bg = -INFINITY, bk = 0.0;
    u32 bc = kEmpty, ranked = 0;
    for (u64 v = chunk_off[i] + lane; v < chunk_off[i + 1]; v += 32) {
      const HubBest h = best[v];
      ranked += h.pad;
      if (better(h.g, h.c, bg, bc)) bg = h.g, bc = h.c, bk = h.k;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double og = __shfl_xor_sync(0xffffffffu, bg, o);
      const u32 oc = __shfl_xor_sync(0xffffffffu, bc, o);
      const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
      ranked += __shfl_xor_sync(0xffffffffu, ranked, o);
      if (better(og, oc, bg, bc)) bg = og, bc = oc, bk = ok;
    }
    if (lane == 0) {
      const u32 u = hubs[i];
      const u32 pi = x.hub_index[u];
      const u64 d = x.g.off[u + 1] - x.g.off[u];
      const u32 from = x.C[u];
      const double own = double(static_cast<const V*>(x.hub_own)[pi]);
      x.hub_live[pi] = 0;
      static_cast<V*>(x.hub_own)[pi] = V(0);
      if (!DRY) x.flags[u] = 0;
      ++tl.verts;
      tl.arcs += d;
      tl.rand += d + ranked;
      moved[i] = decide<DRY>(x, u, from, x.K[u], bc, bg, bk, own, tl) ? 1 : 0;
    }
  }
  tl.flush(x);
}

// neighbour marks of the hubs that moved, chunk by chunk (louvain_compact.cpp:160-161)
__global__ void lm_hub_mark(MoveArgs x, const u32* __restrict__ hubs, u64 count, const u64* __restrict__ chunk_off,
                            const u32* __restrict__ chunk_hub, const u8* __restrict__ moved) {
  ull marks = 0;
  const u64 total = chunk_off[count];
  for (u64 v = blockIdx.x; v < total; v += gridDim.x) {
    const u64 lo = chunk_hub[v];  // hub of chunk v
    if (!moved[lo]) continue;
    const u32 u = hubs[lo];
    const u64 row = x.g.off[u], row_end = x.g.off[u + 1];
    const u64 a0 = row + (v - chunk_off[lo]) * kHubChunk;
    const u64 a1 = min(a0 + kHubChunk, row_end);
    for (u64 a = a0 + threadIdx.x; a < a1; a += blockDim.x) x.flags[x.g.tgt[a]] = 1, ++marks;
  }
  marks = warp_sum(marks);
  if ((threadIdx.x & 31) == 0 && marks) atomicAdd(&x.counters[3], marks);
}

// ---- launch plumbing ----------------------------------------------------------
template <class K>
int occupancy(K kernel, int threads, size_t smem) {
  int b = 0;
  LVN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, smem));
  return b > 0 ? b : 1;
}

template <class K>
void set_smem(K kernel, size_t smem) {
  if (smem > 48 * 1024)
    LVN_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
}

// Launch `kernel` over list[0, count) in chunks of at most a.chunk vertices;
// chunks run in vertex order on the stream, so a later chunk sees the moves
// of the earlier ones.
template <class K>
void launch_chunks(K kernel, const MoveArgs& a, const u32* list, u64 count, int threads, u64 per_block,
                   u64 max_blocks, size_t smem, cudaStream_t s) {
  const u64 chunk = a.chunk ? a.chunk : count;
  for (u64 off = 0; off < count; off += chunk) {
    const u64 c = std::min<u64>(chunk, count - off);
    const u64 blocks = std::max<u64>(1, std::min<u64>((c + per_block - 1) / per_block, max_blocks));
    kernel<<<unsigned(blocks), threads, smem, s>>>(a, list + off, c);
    LVN_LAUNCH();
  }
}

// LVN_MOVE_KERNEL=sort selects the unpacked register sort (lm_sort) for the
// sort bins, =match the match.any kernels (tuning aids; lm_psort is the default)
int move_kernel_choice() {
  static const int v = [] {
    const char* e = std::getenv("LVN_MOVE_KERNEL");
    if (!e) return 0;
    const std::string s(e);
    return s == "sort" ? 1 : s == "match" ? 2 : 0;
  }();
  return v;
}
bool use_match() { return move_kernel_choice() == 2; }

// Uniform-weight sort bins run on 16 lanes per vertex with twice the
// registers per lane (lm_psort<16, 2K>), so the per-vertex work (header
// loads, ranking reductions, the decision) is shared by half as many lanes and
// twice as many vertices are in flight per warp; unit sums are exact in any
// lane layout, so decisions do not depend on the layout. LVN_SORT16=mask
// picks the bins (bit 0: rows of 17-32 arcs, bit 1: 33-64, bit 2: 65-128,
// bit 3: 129-256);
// default 6 (C5 local moving 450 -> 412 ms; C2, C3 unchanged).
int sort16_mask() {
  static const int v = [] {
    const char* e = std::getenv("LVN_SORT16");
    return e ? std::atoi(e) : 6;
  }();
  return v;
}
int hub_interleave() {
  static const int v = [] {
    const char* e = std::getenv("LVN_HUB_INTERLEAVE");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

template <int G, int K, class V, bool DRY>
void launch_sort(const MoveArgs& a, const BinView& b, int bin, cudaStream_t s);

// the same bin on 16 lanes per vertex (uniform weights only, see sort16_mask)
template <int K, class V, bool DRY>
bool launch_sort16(const MoveArgs& a, const BinView& b, int bin, cudaStream_t s) {
  const int bit = K == 1 ? 1 : K == 2 ? 2 : K == 4 ? 4 : 8;
  if (DRY || !a.uniform || move_kernel_choice() != 0 || !(sort16_mask() & bit)) return false;
  constexpr int T = 256;
  auto k = lm_psort<16, K * 2, V, DRY, true>;
  static const int occ = occupancy(k, T, 0);
  launch_chunks(k, a, b.of(bin), b.count(bin), T, T / 16, u64(sm_count()) * occ, 0, s);
  return true;
}

template <int G, int K, class V, bool DRY>
void launch_sort(const MoveArgs& a, const BinView& b, int bin, cudaStream_t s) {
  if (!b.count(bin)) return;
  if constexpr (G == 32 && K <= 8 && !DRY) {
    if (launch_sort16<K, V, DRY>(a, b, bin, s)) return;
  }
  constexpr int T = 256;
  constexpr int LB = ilog2<G * K>();
  // community-only keys for uniform weights; packed keys need (n - 1) << LB | (N - 1) < 0xFFFFFFFF
  if (move_kernel_choice() == 0 && a.uniform && !DRY) {
    auto k = lm_psort<G, K, V, DRY, true>;
    static const int occ = occupancy(k, T, 0);
    launch_chunks(k, a, b.of(bin), b.count(bin), T, T / G, u64(sm_count()) * occ, 0, s);
    return;
  }
  if (move_kernel_choice() == 0 && u64(a.g.n) < (u64(1) << (32 - LB))) {
    auto k = lm_psort<G, K, V, DRY, false>;
    static const int occ = occupancy(k, T, 0);
    launch_chunks(k, a, b.of(bin), b.count(bin), T, T / G, u64(sm_count()) * occ, 0, s);
    return;
  }
  auto k = lm_sort<G, K, V, DRY>;
  static const int occ = occupancy(k, T, 0);
  launch_chunks(k, a, b.of(bin), b.count(bin), T, T / G, u64(sm_count()) * occ, 0, s);
}

template <int K, class Tab, bool DRY>
void launch_match(const MoveArgs& a, const BinView& b, int bin, cudaStream_t s) {
  if (!b.count(bin)) return;
  constexpr int T = 256;
  auto k = lm_match<K, Tab, DRY>;
  constexpr size_t smem = match_smem<K, Tab>();
  static const int occ = (set_smem(k, smem), occupancy(k, T, smem));
  launch_chunks(k, a, b.of(bin), b.count(bin), T, T / 32, u64(sm_count()) * occ, smem, s);
}

template <class Tab, bool DRY>
void sweep(const MoveArgs& a, const BinView& b, cudaStream_t s) {
  using V = typename Tab::V;
  const int sms = sm_count();
  auto launch_bin = [&](int bin, cudaStream_t s) {
    if (!b.count(bin)) return;
    switch (bin) {
      case kBinThread: {
        auto k = lm_thread<V, DRY>;
        static const int occ = occupancy(k, 256, 0);
        launch_chunks(k, a, b.of(bin), b.count(bin), 256, 256, u64(sms) * occ, 0, s);
        break;
      }
      case kBinSort8: launch_sort<8, 1, V, DRY>(a, b, bin, s); break;
      case kBinSort16: launch_sort<16, 1, V, DRY>(a, b, bin, s); break;
      case kBinSort32:
        if (use_match()) launch_match<1, Tab, DRY>(a, b, bin, s); else launch_sort<32, 1, V, DRY>(a, b, bin, s);
        break;
      case kBinSort64:
        if (use_match()) launch_match<2, Tab, DRY>(a, b, bin, s); else launch_sort<32, 2, V, DRY>(a, b, bin, s);
        break;
      case kBinSort128:
        if (use_match()) launch_match<4, Tab, DRY>(a, b, bin, s); else launch_sort<32, 4, V, DRY>(a, b, bin, s);
        break;
      case kBinSort256:
        if (use_match()) launch_match<8, Tab, DRY>(a, b, bin, s); else launch_sort<32, 8, V, DRY>(a, b, bin, s);
        break;
      case kBinWarp: {
        constexpr int T = 256;
        auto k = lm_group<Tab, 32, kWarpCapLog, T, DRY>;
        constexpr size_t smem = group_smem<Tab, 32, kWarpCapLog, T>();
        static const int occ = (set_smem(k, smem), occupancy(k, T, smem));
        launch_chunks(k, a, b.of(bin), b.count(bin), T, T / 32, u64(sms) * occ, smem, s);
        break;
      }
      case kBinBlockT:
      case kBinBlockS:
      case kBinBlock: {
        // rows of <= 512 arcs: eight sub-groups of 64 threads per block, <= 1024:
        // four of 128 (vertices in flight per SM: 16 / 8 instead of 2); longer
        // rows: the whole block
        constexpr size_t smem = block_stage_smem<Tab>();
        auto k8 = lm_block<Tab, DRY, 8>;
        auto k4 = lm_block<Tab, DRY, 4>;
        auto k1 = lm_block<Tab, DRY, 1>;
        static const int occ8 = (set_smem(k8, smem), occupancy(k8, kBlockThreads, smem));
        static const int occ4 = (set_smem(k4, smem), occupancy(k4, kBlockThreads, smem));
        static const int occ1 = (set_smem(k1, smem), occupancy(k1, kBlockThreads, smem));
        const int per = bin == kBinBlockT ? 8 : bin == kBinBlockS ? 4 : 1;
        const int occ = per == 8 ? occ8 : per == 4 ? occ4 : occ1;
        const u64 chunk = std::min(a.chunk, a.hub_chunk);
        const u32* list = b.of(bin);
        const u64 cnt = b.count(bin);
        for (u64 off = 0; off < cnt; off += chunk) {
          const u64 c = std::min<u64>(chunk, cnt - off);
          const u64 nb = std::max<u64>(1, std::min<u64>((c + per - 1) / per, u64(sms) * occ));
          if (per == 8) k8<<<unsigned(nb), kBlockThreads, smem, s>>>(a, list + off, c, 0, kBlockSplit / 2);
          else if (per == 4) k4<<<unsigned(nb), kBlockThreads, smem, s>>>(a, list + off, c, 0, kBlockSplit);
          else k1<<<unsigned(nb), kBlockThreads, smem, s>>>(a, list + off, c, 0, ~u64(0));
          LVN_LAUNCH();
        }
        break;
      }
      case kBinGlobal: {
        // hubs in groups of hub_chunk: a later group sees the moves of the earlier ones
        if (!a.hub_tables) fail(kInternal, "hub plan not provisioned");
        const u64 all = b.count(bin);
        const u64 step = std::max<u64>(1, std::min(a.hub_chunk, all));
        DBuf<u32> chunks(std::min(step, all));
        DBuf<u64> coff(std::min(step, all) + 1);
        // slices of every hub of a group: at most arcs / kHubChunk + hubs
        DBuf<HubBest> hbest(a.g.arcs / kHubChunk + std::min(step, all) + 1);
        DBuf<u32> owner(a.g.arcs / kHubChunk + std::min(step, all) + 1);
        DBuf<u8> hmoved(std::min(step, all));
        DBuf<u32> hkey, hval, hkey2, hval2;  // interleaved chunk schedule (hub_interleave)
        auto kc = lm_hub_chunks<Tab>;
        constexpr size_t smem = hub_smem<Tab>();
        static const int occ = (set_smem(kc, smem), occupancy(kc, kBlockThreads, smem));
        for (u64 h0 = 0; h0 < all; h0 += step) {
          const u64 cnt = std::min(step, all - h0);
          const u32* hubs = b.of(bin) + h0;
          hub_chunk_counts_k<<<unsigned(std::min<u64>((cnt + 255) / 256, u64(sms) * 4)), 256, 0, s>>>(
              hubs, cnt, a.g.off, chunks.p, a.full_lists && a.prune && !DRY ? a.flags : nullptr);
          LVN_LAUNCH();
          exclusive_scan_u32_to_u64(chunks.p, coff.p, cnt, s);
          hub_chunk_owner_k<<<unsigned(std::min<u64>((cnt + 255) / 256, u64(sms) * 4)), 256, 0, s>>>(coff.p, cnt,
                                                                                                    owner.p);
          LVN_LAUNCH();
          const u32* order = nullptr;
          if (hub_interleave()) {
            const u64 cap = a.g.arcs / kHubChunk + cnt + 1;
            hkey.ensure(cap), hval.ensure(cap), hkey2.ensure(cap), hval2.ensure(cap);
            hub_order_keys_k<<<unsigned(std::min<u64>((cap + 255) / 256, u64(sms) * 8)), 256, 0, s>>>(
                coff.p, owner.p, cnt, cap, hkey.p, hval.p);
            LVN_LAUNCH();
            size_t bytes = 0;
            LVN_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, hkey.p, hkey2.p, hval.p, hval2.p, cap, 0, 32, s));
            DBuf<unsigned char> tmp(bytes);
            LVN_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, hkey.p, hkey2.p, hval.p, hval2.p, cap, 0, 32, s));
            order = hval2.p;
          }
          kc<<<unsigned(sms * occ), kBlockThreads, smem, s>>>(a, hubs, cnt, coff.p, owner.p, order);
          LVN_LAUNCH();
          lm_hub_rank<Tab, DRY><<<unsigned(sms * 4), kBlockThreads, 0, s>>>(a, hubs, cnt, coff.p, owner.p, hbest.p);
          LVN_LAUNCH();
          lm_hub_decide<Tab, DRY><<<unsigned(std::min<u64>((cnt + 7) / 8, u64(sms) * 8)), 256, 0, s>>>(
              a, hubs, cnt, coff.p, hbest.p, hmoved.p);
          LVN_LAUNCH();
          if (!DRY && a.prune) {
            lm_hub_mark<<<unsigned(sms * 8), 256, 0, s>>>(a, hubs, cnt, coff.p, owner.p, hmoved.p);
            LVN_LAUNCH();
          }
        }
        break;
      }
      default: break;
    }
  };
  // hubs first: the highest-degree vertices settle before the rows that follow
  // them (on power-law graphs this is what a sequential id-order sweep does,
  // since hubs carry low ids); the reference compact engine sweeps low degree first
  int order[kBins], nb = 0;
  if (a.hubs_first) {
    for (int bin = kBinGlobal; bin >= kBinThread; --bin)
      if (b.count(bin)) order[nb++] = bin;
  } else {
    for (int bin = kBinThread; bin <= kBinGlobal; ++bin)
      if (b.count(bin)) order[nb++] = bin;
  }
  // concurrent bins: every class but the hubs forks onto an aux stream behind
  // one event of s and joins back into s; the hub chain stays on s, where its
  // scratch buffers are allocated and stream-ordered freed (inside a capture:
  // parallel graph branches)
  int others = 0;
  for (int j = 0; j < nb; ++j) others += order[j] != kBinGlobal;
  if (a.nfork <= 0 || others <= 1) {
    for (int j = 0; j < nb; ++j) launch_bin(order[j], s);
    return;
  }
  Context& c = ctx();
  const int nf = std::min(a.nfork, others);
  if (int(c.aux.size()) < nf || int(c.aux_ev.size()) < nf + 1) fail(kInternal, "forked sweep streams not provisioned");
  LVN_CUDA(cudaEventRecord(c.aux_ev[0], s));
  for (int k = 0; k < nf; ++k) LVN_CUDA(cudaStreamWaitEvent(c.aux[k], c.aux_ev[0]));
  for (int j = 0, k = 0; j < nb; ++j) launch_bin(order[j], order[j] == kBinGlobal ? s : c.aux[k++ % nf]);
  for (int k = 0; k < nf; ++k) {
    LVN_CUDA(cudaEventRecord(c.aux_ev[1 + k], c.aux[k]));
    LVN_CUDA(cudaStreamWaitEvent(s, c.aux_ev[1 + k]));
  }
}

template <class Tab>
void hub_plan_impl(const DGraph& g, const u32* hubs, u64 count, HubPlan& p, cudaStream_t s) {
  p.count = count;
  if (!count) return;
  const int sms = sm_count();
  p.index.ensure(g.n ? g.n : 1);
  p.tab_off.ensure(count + 1);
  DBuf<u64> bytes(count);
  hub_plan_k<Tab><<<unsigned(std::min<u64>((count + 255) / 256, u64(sms) * 4)), 256, 0, s>>>(
      hubs, count, g, p.index.p, bytes.p);
  LVN_LAUNCH();
  exclusive_scan_u64(bytes.p, p.tab_off.p, count, s);
  u64* h = ctx().pinned;
  LVN_CUDA(cudaMemcpyAsync(h, p.tab_off.p + count, sizeof(u64), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  p.tables.ensure(h[0] ? h[0] : 16);
  hub_clear_k<Tab><<<unsigned(std::min<u64>(count, u64(sms) * 4)), 256, 0, s>>>(hubs, count, g, p.tab_off.p,
                                                                                p.tables.p);
  LVN_LAUNCH();
  p.live.ensure(count);
  p.own.ensure(count);
  LVN_CUDA(cudaMemsetAsync(p.live.p, 0, count * sizeof(u32), s));
  LVN_CUDA(cudaMemsetAsync(p.own.p, 0, count * sizeof(double), s));
}

__global__ void apply_moves_k(const u32* __restrict__ rec, u64 total, u64 skip_lo, u64 skip_hi, DGraph g,
                              u32* __restrict__ C, const double* __restrict__ K, double* __restrict__ sigma,
                              u8* __restrict__ flags, int prune) {
  const u32 lane = threadIdx.x & 31;
  const u64 warps = u64(gridDim.x) * (blockDim.x >> 5);
  for (u64 i = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5; i < total; i += warps) {
    if (i >= skip_lo && i < skip_hi) continue;
    const u32 u = rec[2 * i], to = rec[2 * i + 1];
    if (lane == 0) {
      const u32 from = C[u];
      const double ku = K[u];
      C[u] = to;
      atomicAdd(&sigma[to], ku);
      atomicAdd(&sigma[from], -ku);
    }
    if (prune)
      for (u64 a = g.off[u] + lane; a < g.off[u + 1]; a += 32) flags[g.tgt[a]] = 1;
  }
}

// records in per-rank blocks of fixed capacity (segoff), only the first
// counts[j] of block j valid; the own block (me) is skipped
__global__ void apply_segments_k(const u32* __restrict__ rec, const u64* __restrict__ segoff,
                                 const u32* __restrict__ counts, int P, int me, u64 total, u32* __restrict__ C,
                                 const double* __restrict__ K, double* __restrict__ sigma) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < total; i += u64(gridDim.x) * blockDim.x) {
    int lo = 0, hi = P;  // block of record i: last j with segoff[j] <= i
    while (hi - lo > 1) {
      const int mid = (lo + hi) / 2;
      if (segoff[mid] <= i) lo = mid; else hi = mid;
    }
    if (lo == me || i - segoff[lo] >= counts[lo]) continue;
    const u32 u = rec[2 * i], to = rec[2 * i + 1];
    const u32 from = C[u];
    const double ku = K[u];
    C[u] = to;
    atomicAdd(&sigma[to], ku);
    atomicAdd(&sigma[from], -ku);
  }
}

}  // namespace

int move_kernel_variant() { return move_kernel_choice(); }

void apply_moves_segments(const u32* rec, const u64* segoff, const u32* counts, int P, int me, u64 total, u32* C,
                          const double* K, double* sigma, cudaStream_t s) {
  if (!total) return;
  const u64 blocks = std::min<u64>((total + 255) / 256, u64(sm_count()) * 8);
  apply_segments_k<<<unsigned(blocks), 256, 0, s>>>(rec, segoff, counts, P, me, total, C, K, sigma);
  LVN_LAUNCH();
}

void apply_moves(const u32* rec, u64 total, u64 skip_lo, u64 skip_hi, const DGraph& g, u32* C, const double* K,
                 double* sigma, u8* flags, int prune, cudaStream_t s) {
  if (total <= skip_hi - skip_lo) return;
  const u64 blocks = std::min<u64>((total + 7) / 8, u64(sm_count()) * 16);
  apply_moves_k<<<unsigned(blocks), 256, 0, s>>>(rec, total, skip_lo, skip_hi, g, C, K, sigma, flags, prune);
  LVN_LAUNCH();
}

void hub_plan_build(const DGraph& g, const u32* hubs, u64 count, int value_bits, HubPlan& p,
                    cudaStream_t s) {
  if (value_bits == 64)
    hub_plan_impl<SplitF64>(g, hubs, count, p, s);
  else
    hub_plan_impl<PackedF32>(g, hubs, count, p, s);
}

void move_sweep(const MoveArgs& a0, const BinView& b, int value_bits, cudaStream_t s) {
  if (b.edges.thread_max > kThreadMaxD || b.edges.group_max > 256 ||
      b.edges.warp_max > (1u << (kWarpCapLog - 1)) ||
      b.edges.block_max > (1u << (kBlockCapLog - 1)))
    fail(kInvalid, "degree bin edges exceed the device table capacities");
  MoveArgs a = a0;
  a.inv_m = 1.0 / a.m;
  a.inv_2m2 = 1.0 / (2.0 * a.m * a.m);
  if (value_bits == 64) {
    a.dry ? sweep<SplitF64, true>(a, b, s) : sweep<SplitF64, false>(a, b, s);
  } else {
    a.dry ? sweep<PackedF32, true>(a, b, s) : sweep<PackedF32, false>(a, b, s);
  }
}

// lvn_params.probing for the tables of this file (reference probe_advance,
// compact_hashtable.hpp:60-82); stream-ordered
void set_probing_move(int mode, cudaStream_t s) {
  static int value;  // pageable source: staged before the call returns
  value = mode;
  LVN_CUDA(cudaMemcpyToSymbolAsync(c_probing, &value, sizeof(int), 0, cudaMemcpyHostToDevice, s));
}

}  // namespace lvn
