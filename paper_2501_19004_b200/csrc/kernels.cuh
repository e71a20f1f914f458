// Host-side launchers of the device kernels (one .cu per family). All run on
// the context stream; none synchronises unless it says so.
#pragma once

#include "common.cuh"

namespace lvn {

// ---- scan.cu: exclusive prefix sums, out has n+1 entries (prefix_sum.hpp:12-23)
void exclusive_scan_u32(const u32* in, u32* out, u64 n, cudaStream_t s);
void exclusive_scan_u64(const u64* in, u64* out, u64 n, cudaStream_t s);
void exclusive_scan_u32_to_u64(const u32* in, u64* out, u64 n, cudaStream_t s);
// max-reduction of a u32 array into *out (device)
void reduce_max_u32(const u32* in, u64 n, u32* out, cudaStream_t s);

// ---- bins.cu: degree bins + pass reset ------------------------------------
// Degree classes (the kernel that handles a row / community):
enum : int {
  kBinIso = 0,      // no arcs
  kBinThread = 1,   // deg <= thread_max: thread per vertex, registers
  kBinSort8 = 2,    // deg <= 8 (and <= group_max): 8 lanes, register bitonic sort
  kBinSort16 = 3,   // deg <= 16: 16 lanes
  kBinSort32 = 4,   // deg <= 32: 32 lanes
  kBinSort64 = 5,   // deg <= 64: 32 lanes x 2 registers
  kBinSort128 = 6,  // deg <= 128: 32 lanes x 4 registers
  kBinSort256 = 7,  // deg <= 256: 32 lanes x 8 registers
  kBinWarp = 8,     // deg <= warp_max: warp, smem hash table
  kBinBlockT = 9,   // deg <= min(block_max, kBlockSplitDeg / 2): eight sub-groups per block
  kBinBlockS = 10,  // deg <= min(block_max, kBlockSplitDeg): four sub-groups per block
  kBinBlock = 11,   // deg <= block_max: block, smem hash table
  kBinGlobal = 12,  // larger: block, global-memory hash table
  kBins = 13
};
// rows of the block class up to this degree share a block with three others,
// up to half of it with seven others (own bins, so no kernel walks rows it
// does not take)
constexpr unsigned long long kBlockSplitDeg = 1024;
struct BinEdges {
  u32 thread_max = 4, group_max = 256, warp_max = 256, block_max = 4096;
};
// A set of per-bin vertex lists (the full bins, or the active subset of an iteration)
struct BinView {
  const u32* list = nullptr;
  u64 off[kBins] = {};
  u64 cnt[kBins] = {};
  u64 max_degree = 0;
  BinEdges edges;
  u64 count(int b) const { return cnt[b]; }
  const u32* of(int b) const { return list + off[b]; }
};
struct Bins {
  DBuf<u32> list;       // vertex ids grouped by bin, ascending within a bin
  u64 start[kBins + 1]; // host copy of the bin boundaries in `list`
  u64 max_degree = 0;
  BinEdges edges;
  u64 count(int b) const { return start[b + 1] - start[b]; }
  const u32* of(int b) const { return list.p + start[b]; }
  BinView view() const {
    BinView v;
    v.list = list.p;
    for (int b = 0; b < kBins; ++b) v.off[b] = start[b], v.cnt[b] = count(b);
    v.max_degree = max_degree;
    v.edges = edges;
    return v;
  }
};
// active subset of b: out_list gets, inside each bin's segment, the vertices
// whose flag is set (order within a bin not preserved); counts[b] (device,
// zeroed here) receives the per-bin sizes
void compact_active(const Bins& b, const u8* flags, u32* out_list, ull* counts, cudaStream_t s);
// bin of row v by min(off[v+1]-off[v], cap): rows of a CSR, or community
// budgets during aggregation. Synchronises (reads the bin sizes).
// id_base is added to the row index written into the lists (bins of a
// vertex range: off points at the range's first offset).
void compute_bins(const u64* off, u32 n, const BinEdges& e, Bins& out, cudaStream_t s,
                  u64 cap = ~u64(0), u32 id_base = 0);
// K_u = row sums (fp64), Sigma = K, C = identity, flags = deg > 0; *uniform
// (when given) ends non-zero iff every arc weight equals the first one
void pass_reset(const DGraph& g, const Bins& b, double* K, double* sigma, u32* C, u8* flags,
                cudaStream_t s, u32* uniform = nullptr);
void vertex_weights(const DGraph& g, const Bins& b, double* K, cudaStream_t s);

// ---- move.cu: local-moving sweep ------------------------------------------
struct MoveArgs {
  DGraph g;
  u32* C = nullptr;
  const double* K = nullptr;
  double* sigma = nullptr;
  u8* flags = nullptr;
  double m = 1.0;
  int pickless = 0;
  const int* pickless_dev = nullptr;  // graph-mode passes: Pick-Less of the running iteration (device word)
  int prune = 1;
  int dry = 0;              // evaluate only: write out_to / out_gain, apply nothing
  // probe (lvn_probe_moves): the live kernels (the engine's ranking: reciprocal
  // Eq. 2, may_gain pruning, community-only keys on uniform weights) with the
  // decision written to out_to / out_gain instead of applied
  int probe = 0;
  int value_f32 = 1;        // probe: round the reported gain to f32 like the V = float table
  u32* out_to = nullptr;
  double* out_gain = nullptr;
  double* gain_acc = nullptr;  // summed gain of applied moves
  ull* counters = nullptr;     // [0] vertices processed, [1] arcs scanned, [2] moves, [3] random accesses
  u32* err = nullptr;
  u64 chunk = ~u64(0);         // max vertices of one bin decided per launch
  u64 hub_chunk = ~u64(0);     // max vertices of the block / hub bins decided per launch
  int uniform = 0;             // every arc weight equals uniform_w: sort bins key on the community alone
  float uniform_w = 0.f;
  double inv_m = 0.0, inv_2m2 = 0.0;  // set by move_sweep
  int hubs_first = 0;          // bin order of a sweep: highest degree class first
  // L2 priority of the sort kernels' C / Sigma gathers: 1 evict_last (default),
  // 0 evict_normal, 2 evict_first (LVN_L2_KEEP, tuning aid)
  int l2_keep = 1;
  // full bin lists (graph-mode passes): every kernel skips the rows whose
  // prune flag is clear instead of relying on a compacted active list
  int full_lists = 0;
  // > 0: the degree bins of one sweep run on this many forked streams
  // (captured sweeps of small passes): the launch tails of the classes overlap
  int nfork = 0;
  u32* csize = nullptr;        // community member counts (singleton-pair rule), or null
  // sharded runs: every applied move appends (u, to) here (count in *moves_n)
  u32* moves_out = nullptr;
  u32* moves_n = nullptr;
  // hub plan of the pass (kBinGlobal vertices): see HubPlan
  const u32* hub_index = nullptr;
  const u64* hub_tab_off = nullptr;
  u32* hub_live = nullptr;
  void* hub_own = nullptr;
  unsigned char* hub_tables = nullptr;
};

// Per-pass storage for the chunked hub kernels: every kBinGlobal vertex owns an
// HBM table of next_pow2(2 min(deg, n)) slots plus a live list, kept empty
// between sweeps by the kernels themselves.
struct HubPlan {
  DBuf<u32> index;            // vertex -> position in the pass hub list
  DBuf<u64> tab_off;          // position -> byte offset of its region
  DBuf<u32> live;             // position -> live entries
  DBuf<double> own;           // position -> weight to the own community (f32 or f64 view)
  DBuf<unsigned char> tables;
  u64 count = 0;
  void attach(MoveArgs& a) const {
    a.hub_index = index.p, a.hub_tab_off = tab_off.p, a.hub_live = live.p;
    a.hub_own = own.p, a.hub_tables = tables.p;
  }
};
void hub_plan_build(const DGraph& g, const u32* hubs, u64 count, int value_bits, HubPlan& p,
                    cudaStream_t s);
// remote moves of a sharded round: records (u, to) pairs [0, total) except
// [skip_lo, skip_hi) (this rank's own, already applied): C[u] = to, Sigma moves
// K[u] from C[u] to `to`, and u's neighbours are flagged when prune is set
void apply_moves(const u32* rec, u64 total, u64 skip_lo, u64 skip_hi, const DGraph& g, u32* C, const double* K,
                 double* sigma, u8* flags, int prune, cudaStream_t s);
// table probing mode of the local-moving / aggregation kernels (lvn_probing)
int move_kernel_variant();  // LVN_MOVE_KERNEL: 0 = default (lm_psort), 1 = sort, 2 = match
void set_probing_move(int mode, cudaStream_t s);
void set_probing_aggregate(int mode, cudaStream_t s);
// the same from per-rank record blocks of fixed capacity: block j holds
// counts[j] (device) valid records from segoff[j] (device, P+1 entries); block
// me is this rank's own (already applied)
void apply_moves_segments(const u32* rec, const u64* segoff, const u32* counts, int P, int me, u64 total, u32* C,
                          const double* K, double* sigma, cudaStream_t s);
// one sweep over the bins of `bins` (see the kBin* classes)
void move_sweep(const MoveArgs& a, const BinView& bins, int value_bits, cudaStream_t s);

// ---- community.cu -----------------------------------------------------------
// used[c] = 1 for every c in C (used zeroed here), sized n
void mark_used(const u32* C, u64 n, u32* used, u64 width, cudaStream_t s);
// C[v] = rank[C[v]]
void remap(u32* C, u64 n, const u32* rank, cudaStream_t s);
// global[i] = level[global[i]], range-checked into *err
void lookup(u32* global, u64 n, const u32* level, u64 nl, u32* err, cudaStream_t s);
// per-community member counts (u32) and arc budgets (u64), zeroed here
void community_counts(const DGraph& g, const u32* C, u32 count, u32* members, u64* budget,
                      cudaStream_t s);
// members[coff[c] + cursor[c]++] = v (cursor zeroed here)
void community_scatter(const u32* C, u32 n, const u64* coff, u32 count, u32* cursor, u32* members,
                       cudaStream_t s);
// sort every segment [off[i], off[i+1]) of keys ascending (vals permuted alongside)
void segmented_sort_u32(u32* keys, float* vals, const u64* off, u32 nseg, u64 max_seg,
                        cudaStream_t s);
void iota_u32(u32* p, u64 n, cudaStream_t s);
// out[c] = sum of v[u] over C[u] == c (fp64; out zeroed here, count entries)
void sum_by_community(const u32* C, const double* v, u64 n, double* out, u32 count, cudaStream_t s);
void fill_u32(u32* p, u64 n, u32 v, cudaStream_t s);

// ---- aggregate.cu -----------------------------------------------------------
struct AggArgs {
  DGraph g;
  const u32* C = nullptr;        // contiguous ids < count
  u32 count = 0;
  const u64* coff = nullptr;     // community -> member offsets
  const u32* members = nullptr;
  const u64* boff = nullptr;     // scanned total member degrees (work per community)
  const u64* hoff = nullptr;     // holey row offsets (scanned min(budget, count))
  u32* htgt = nullptr;           // holey targets / weights
  float* hw = nullptr;
  double* hw64 = nullptr;        // sharded partial rows: fp64 weights instead of hw
  u32* fill = nullptr;           // entries written per row
  u32* err = nullptr;
  u32* inexact = nullptr;        // set when narrowing a non-self entry to f32 loses bits (may be null)
  double* self64 = nullptr;      // fp64 self-loop (internal weight) of every super-vertex (may be null)
  int big_mode = 0;              // giant-community regions: 0 by size, 1 hash, 2 dense (LVN_BIG_MODE)
};
// Synchronises once when the kBinGlobal bin is non-empty (sizes its HBM tables).
void aggregate_rows(const AggArgs& a, const Bins& bins, cudaStream_t s);
// capped[c] = min(x[c] + plus_one, count): holey row capacity from the budget
// (plus_one false) or from the external arcs (ext + 1 with the self-loop)
void cap_budgets(const u64* x, u64* capped, u32 count, cudaStream_t s, bool plus_one);
// out rows = holey rows compacted (noff = scan of fill), total weight (fp64) into *tw
void compact_rows(const u64* hoff, const u32* htgt, const float* hw, const u32* fill,
                  const u64* noff, u32 count, u32* otgt, float* ow, double* tw,
                  cudaStream_t s);

// ---- modularity.cu ----------------------------------------------------------
// sums: [0] internal arc weight, [1] sum_c Sigma_c^2 ; tot (width entries) zeroed here
void modularity_terms(const DGraph& g, const Bins& b, const u32* C, double* tot, u64 width,
                      double* sums, cudaStream_t s, double two_m);
// the two halves of modularity_terms (a sharded run allreduces tot and sums[0]
// between them): the row pass (tot, sums zeroed here) and sums[1] += sum_c (tot_c / 2m)^2
void modularity_rows(const DGraph& g, const Bins& b, const u32* C, double* tot, u64 width, double* sums,
                     cudaStream_t s);
void modularity_squares(const double* tot, u64 width, double two_m, double* sums, cudaStream_t s);
// modularity_terms on a super-graph whose per-vertex total degree (kx) and
// self-loop (self64) are given exactly in fp64 (the f32 arcs of self-loops are ignored)
void modularity_exact(const DGraph& g, const u32* C, const double* kx, const double* self64, double* tot, u64 width,
                      double* sums, cudaStream_t s, double two_m);
// ext[c] = arcs from members of c to other communities (width entries, zeroed
// here): bounds the distinct targets of super-row c (aggregation capacities)
void external_arcs(const DGraph& g, const Bins& b, const u32* C, u64* ext, u64 width, cudaStream_t s);

// ---- generate.cu: device-built synthetic inputs --------------------------------
struct OwnedCsr {
  u32 n = 0;
  u64 arcs = 0;
  DBuf<u64> off;
  DBuf<u32> tgt;
  DBuf<float> w;
  double total_weight = 0.0;
  DGraph view() const { return DGraph{n, arcs, off.p, tgt.p, w.p}; }
};
struct GenSpec {
  int kind = 0;
  u64 n = 0, edges = 0;
  u32 scale = 0, blocks = 0;
  double a = 0.57, b = 0.19, c = 0.19, mu = 0.1, p = 0.6, avg_degree = 16.0;
  u64 seed = 1;
};
void generate(const GenSpec& g, OwnedCsr& out, cudaStream_t s);
// build.cu: build_csr (graph.cpp:15-87) on the device from device triples;
// throws kInvalid on bad endpoints / weights
void build_csr_device(u32 n, u64 T, const u32* src, const u32* dst, const double* w, int symmetrize,
                      OwnedCsr& out, cudaStream_t s);
// sorted arc keys (source<<32 | target, ~0 = dropped) -> deduplicated unit-weight CSR
void keys_to_csr(DBuf<ull>& keys, u64 nkeys, u64 n, OwnedCsr& out, cudaStream_t s);

// ---- aggsort.cu: aggregation of a uniform integer-weight pass by external arcs
// true when a sample of the arcs finds at most max_frac of them between communities
bool external_arcs_few(const DGraph& g, const u32* C, double max_frac, cudaStream_t s, double* sampled = nullptr);
// the super-graph of g under C (count communities, budget = member arcs per
// community) from the external arcs (ext receives their count per community;
// cap = key buffer entries); false when more than cap arcs are external (out
// untouched, ext complete). Rows come out sorted by target.
bool aggregate_by_external_arcs(const DGraph& g, const Bins& b, const u32* C, u32 count, const u64* budget,
                                u64* ext, u64 cap, OwnedCsr& out, u32* inexact, double* self64, cudaStream_t s);

}  // namespace lvn
