/* lvn.h — C-ABI of the B200-native Louvain engine (liblvn.so).
 *
 * Drop-in boundary for the reference's Louvain entry point and phase APIs
 * (arXiv 2501.19004 reference, /root/reference/proj/core). Plain pointers and
 * sizes only; no C++ or torch types cross this boundary. Each entry point
 * names the reference interface it replaces.
 *
 * Graph convention (graph.hpp:33-54): symmetric CSR, u64 offsets[n+1], u32
 * targets[arcs] (sorted rows are not required), f32 weights[arcs]; a
 * self-loop is stored once; total_weight = m = (sum of arc weights) / 2.
 *
 * Status codes (mirroring the reference's exceptions, errors.hpp:10-31 and
 * the CLI exit codes louvain_cli.cpp:33-35):
 *   0 LVN_OK
 *   1 LVN_INVALID_ARGUMENT  std::invalid_argument (bad params, non-contiguous membership)
 *   2 LVN_DEGENERATE        DegenerateGraphError (m == 0)
 *   3 LVN_INTERNAL          InternalError (table overflow, dendrogram lookup out of range)
 *   4 LVN_CUDA              CUDA / NCCL failure
 *   5 LVN_OUT_OF_MEMORY     device allocation failed
 * lvn_last_error() returns the thread-local message of the last failure.
 *
 * Threading: every call is synchronous (returns when results are in the
 * caller's memory) and calls are serialised on one internal context.
 */
#ifndef LVN_H
#define LVN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum lvn_status {
  LVN_OK = 0,
  LVN_INVALID_ARGUMENT = 1,
  LVN_DEGENERATE = 2,
  LVN_INTERNAL = 3,
  LVN_CUDA = 4,
  LVN_OUT_OF_MEMORY = 5
};

/* where the arrays of an lvn_csr / a membership live */
enum lvn_location { LVN_HOST = 0, LVN_DEVICE = 1 };

/* Probing modes of the reference's slab tables (compact_hashtable.hpp:13-18),
 * applied by the device tables (power-of-two capacity, multiplicative hash)
 * with the reference's stride recurrences (probe_advance,
 * compact_hashtable.hpp:60-82); they change speed, never results. */
enum lvn_probing { LVN_LINEAR = 0, LVN_QUADRATIC = 1, LVN_DOUBLE_HASH = 2, LVN_QUADRATIC_DOUBLE = 3 };

/* Borrowed view of a CsrGraph (graph.hpp:38-54). Never freed by the library. */
typedef struct lvn_csr {
  uint32_t num_vertices;
  uint64_t num_arcs;
  const uint64_t* offsets;
  const uint32_t* targets;
  const float* weights;
  double total_weight;
  int location; /* lvn_location */
} lvn_csr;

/* Library-owned CSR returned by lvn_aggregate (host arrays). */
typedef struct lvn_graph_out {
  uint32_t num_vertices;
  uint64_t num_arcs;
  uint64_t* offsets;
  uint32_t* targets;
  float* weights;
  double total_weight;
} lvn_graph_out;

/* LouvainParams (louvain.hpp:9-18) + CompactOptions (louvain_compact.hpp:35-40)
 * + device knobs. Initialise with lvn_params_default(). */
typedef struct lvn_params {
  /* LouvainParams */
  int max_passes;               /* 10 */
  int max_iterations;           /* 20 local-moving iterations per pass */
  double initial_tolerance;     /* 0.01 */
  double tolerance_drop;        /* 10 */
  double aggregation_tolerance; /* 0.8 */
  int thread_count;             /* validated (>= 0) for parity; unused on the GPU */
  int chunk_size;               /* validated (>= 1) for parity; unused on the GPU */
  int prune;                    /* 1 */
  /* CompactOptions */
  int pick_less_period;         /* 4, even and >= 2 */
  uint64_t switch_move;         /* 64: reference serial/team split; see bin_* below */
  uint64_t switch_aggregate;    /* 128 */
  int probing;                  /* lvn_probing, LVN_QUADRATIC_DOUBLE */
  int value_bits;               /* 32 or 64: width of the per-vertex scan-table values */
  /* device degree bins: thread <= bin_thread_max < group8 <= bin_group_max
   * < warp <= bin_warp_max < block <= bin_block_max < global-table block */
  uint32_t bin_thread_max;      /* 4 */
  uint32_t bin_group_max;       /* 256: rows up to this degree use the register-sort kernels */
  uint32_t bin_warp_max;        /* 256 */
  uint32_t bin_block_max;       /* 4096 */
  int membership_on_device;     /* result membership stays in device memory */
  /* at most this many vertices of a degree bin are decided by one launch of a
   * sweep (launches run in vertex order, later ones see earlier moves);
   * 0 = automatic (scaled to the graph), UINT32_MAX = one launch per bin */
  uint32_t sweep_chunk;
  /* order of the degree classes within a sweep range: 0 low degree first
   * (the reference compact engine's order, default), 1 hubs first */
  int sweep_order;
  /* a sweep visits the vertex ids in this many consecutive ranges, each range
   * running all its degree classes before the next starts (1 = one range, the
   * reference compact order; larger approaches the id order of louvain_mc);
   * 0 = automatic */
  int sweep_ranges;
  /* 1: a singleton may join another singleton community only if its id is
   * lower (concurrent symmetric pairs merge instead of swapping labels) */
  int singleton_rule;
  /* lvn_louvain_sharded: a pass is sharded across the ranks while its graph
   * has at least 2^shard_min_arcs_log2 arcs; a smaller graph is gathered
   * onto rank 0, which runs the remaining passes alone (the collapse of
   * SURVEY.md 8(e)) */
  int shard_min_arcs_log2;      /* 22 */
  /* lvn_louvain_sharded: each rank sweeps its rows in this many consecutive
   * rounds per iteration, exchanging Sigma / C / marks after each (more
   * rounds: fresher cross-rank state, more collectives); 0 = 2 x ranks */
  int shard_rounds;             /* 0 */
  /* 1: keep the dendrogram, one local membership per pass, in lvn_result
   * (levels[k][v] = community of vertex v of pass k's graph; composing the
   * levels gives the final partition, lookup_dendrogram of louvain_mc.cpp:145) */
  int keep_levels;              /* 0 */
  /* graphs with at least 16 x 2^first_range_arcs_log2 arcs sweep pass 0's
   * first iteration in 16 consecutive vertex-id ranges (low degree first
   * within a range); with host input each range's targets are a separate
   * chunk of the upload, and the sweep of a range starts as soon as its chunk
   * has landed. Smaller graphs sweep in one range; 0 disables */
  int first_range_arcs_log2;    /* 27: graphs of >= 2^31 arcs */
} lvn_params;

/* Per-kernel-family device accounting (CUDA events on the engine stream). */
typedef struct lvn_phase_stats {
  double seconds;        /* summed device time of the family's launches */
  double bytes;          /* algorithmic bytes (SURVEY.md 8(d) formulas) */
  uint64_t launches;      /* timed spans; local moving: one per iteration (sweep) */
  uint64_t items;        /* vertices processed */
  uint64_t arcs;         /* arcs scanned */
  uint64_t gathers;      /* random element accesses: C[t] and Sigma[c] gathers, neighbour marks */
} lvn_phase_stats;

enum { LVN_STAT_MOVE = 0, LVN_STAT_AGGREGATE = 1, LVN_STAT_RENUMBER = 2, LVN_STAT_RESET = 3,
       LVN_STAT_MODULARITY = 4, LVN_STAT_COUNT = 5 };

/* LouvainResult (louvain.hpp:28-39) + device breakdown. */
typedef struct lvn_result {
  uint32_t* membership;   /* num_vertices ids, contiguous 0..count-1 (host, or device) */
  uint32_t num_vertices;
  uint32_t num_communities;
  double modularity;      /* recomputed on the input graph, fp64 */
  int passes;
  int aggregations;
  int* iterations_per_pass;
  double* tolerance_per_pass;
  double* pass_seconds;
  uint32_t* vertices_per_pass;
  uint64_t* arcs_per_pass;
  double local_moving;    /* PhaseTimes (louvain.hpp:20-26), seconds */
  double aggregation;
  double other;
  double wall_seconds;    /* engine entry to result, like the reference */
  double h2d_seconds;     /* input upload (host input only) */
  double d2h_seconds;     /* membership download */
  lvn_phase_stats stats[LVN_STAT_COUNT];
  int membership_on_device;
  int num_shards;         /* ranks of lvn_louvain_sharded (1 otherwise) */
  int sharded_passes;     /* passes run sharded (the rest ran on rank 0 after the collapse) */
  double exchange_seconds; /* time inside the collectives (host time of caller callbacks,
                             device time of the library's NCCL collectives) */
  int num_levels;          /* dendrogram levels kept (lvn_params.keep_levels), else 0 */
  uint32_t** levels;       /* host arrays, level k has vertices_per_pass[k] entries */
  uint64_t h2d_bytes;      /* bytes copied host -> device for the input (host input only;
                              constant weights are verified on the host and filled on the device) */
} lvn_result;

/* ---- lifecycle -------------------------------------------------------- */
int lvn_init(int num_gpus, const int* devices); /* optional; lazily device 0 */
int lvn_finalize(void);
const char* lvn_last_error(void);
const char* lvn_version(void);
void lvn_params_default(lvn_params* p);
void lvn_result_free(lvn_result* r);
void lvn_graph_free(lvn_graph_out* g);

/* ---- engine: louvain_compact (louvain_compact.hpp:57-58) --------------- */
int lvn_louvain(const lvn_csr* g, const lvn_params* p, lvn_result** out);

/* ---- phase / parity APIs ----------------------------------------------- */
/* modularity (quality.hpp:27); any labelling, fp64 */
int lvn_modularity(const lvn_csr* g, const uint32_t* membership, int membership_location,
                   double* q);
/* vertex_weights (graph.hpp:79): K_u = sum of row weights, fp64 */
int lvn_vertex_weights(const lvn_csr* g, double* out_host);
/* count_communities (quality.hpp:40) */
int lvn_count_communities(const uint32_t* membership, uint64_t n, int location, uint32_t* count);
/* renumber_communities (louvain_mc.hpp:101), in place */
int lvn_renumber(uint32_t* membership, uint64_t n, int location, uint32_t* count);
/* lookup_dendrogram (louvain_mc.hpp:105), in place; LVN_INTERNAL when out of range */
int lvn_lookup_dendrogram(uint32_t* membership, uint64_t n, const uint32_t* level, uint64_t nl,
                          int location);
/* build_community_csr (engine_detail.hpp:30-40); members ascending per community.
 * offsets: count+1 entries, members: n entries (host). */
int lvn_community_csr(const uint32_t* membership, uint32_t n, uint32_t count, int location,
                      uint64_t* offsets, uint32_t* members);
/* compact_aggregate / louvain_aggregate (louvain_compact.hpp:76-77, louvain_mc.hpp:96-97):
 * contiguous membership required; fp64 accumulation narrowed once to f32;
 * canonical != 0 sorts each row by target. */
/* build_csr (graph.cpp:15-87) on the device: num_triples host triples
 * (sources[i], targets[i], weights[i]) -> CSR with every row sorted by target,
 * parallel arcs merged (fp64 sum in (target, weight) order, one f32 narrowing)
 * and, when symmetrize != 0, the reverse arc of every non-loop triple added.
 * Errors: LVN_INVALID for endpoints >= num_vertices or weights that are not
 * finite and non-negative (std::invalid_argument in the reference).
 * Replaces build_csr(const EdgeList&, bool) (graph.hpp / graph.cpp:15). */
int lvn_build_csr(uint32_t num_vertices, uint64_t num_triples, const uint32_t* sources,
                  const uint32_t* targets, const double* weights, int symmetrize, lvn_graph_out** out);

int lvn_aggregate(const lvn_csr* g, const uint32_t* membership, int membership_location,
                  int canonical, const lvn_params* p, lvn_graph_out** out);
/* compact_evaluate_move (louvain_compact.hpp:65-72), batched over all vertices on
 * one fixed snapshot (membership, K, Sigma): to[u], gain[u] for every u, no move
 * applied. force_kernel: -1 by degree bin, else the minimum kernel class
 * (0 thread, 1 group, 2 warp, 3 block, 4 global table) a vertex may use. */
int lvn_evaluate_moves(const lvn_csr* g, const uint32_t* membership, const double* vertex_w,
                       const double* community_w, double m, const lvn_params* p,
                       int force_kernel, uint32_t* to, double* gain);
/* The same batched decision through the engine's LIVE ranking path (the
 * kernels lvn_louvain runs: reciprocal Eq. 2 ranking, Sigma-free may_gain
 * pruning, community-only sort keys when every arc weight is equal), with the
 * choice written out instead of applied; gain[u] is the exact Eq. 2 value of
 * the chosen community (compact_evaluate_move, louvain_compact.cpp:413-445),
 * rounded to f32 for value_bits 32. Same arguments as lvn_evaluate_moves. */
int lvn_probe_moves(const lvn_csr* g, const uint32_t* membership, const double* vertex_w,
                    const double* community_w, double m, const lvn_params* p,
                    int force_kernel, uint32_t* to, double* gain);

/* ---- sharded multi-GPU run -------------------------------
 * One process per GPU, each calling lvn_louvain_sharded with the same graph
 * view (host or device arrays; rank r reads only its own slice of them).
 * Storage is sharded: a pass gives rank r the rows [b_r, b_{r+1}) of
 * lvn_partition_rows (pass 0) or of its community range (later passes), and
 * the rank holds only those rows' targets and weights, plus replicated
 * per-vertex state (membership C, K, Sigma, pruning marks; 21 B / vertex).
 * Per local-moving iteration it sweeps its rows in shard_rounds consecutive
 * rounds; after each round the ranks allgather their move records (u, to)
 * and apply the others' (C, Sigma); gain / counters are allreduced and the
 * pruning marks OR-reduced once per iteration. Aggregation is by own rows:
 * each rank sums its arcs into partial super-edges (fp64), routes them to the
 * owner of their super-row (all-to-all) and the owner merges them into its
 * rows of the next graph. Once a pass's graph has fewer than
 * 2^shard_min_arcs_log2 arcs it is gathered onto rank 0, which runs the
 * remaining passes alone (the collapse); the final membership and modularity
 * reach every rank, so all ranks return the same result.
 * Collectives come from lvn_comm: the library's own NCCL communicator
 * (lvn_comm_nccl_create: stream-ordered, no host synchronisation) or caller
 * callbacks (paper_2501_19004_b200.distributed wraps torch.distributed for
 * the gloo tests): buffers are device pointers on this process's GPU, the
 * library's stream is idle when a callback runs, and a callback returns 0
 * once its result is in place. */
enum lvn_dtype { LVN_U8 = 0, LVN_U32 = 1, LVN_U64 = 2, LVN_F64 = 3 };
enum lvn_redop { LVN_SUM = 0, LVN_MAX = 1 };
typedef struct lvn_comm {
  int rank;
  int size;
  void* user;
  /* in-place allreduce of count elements of dtype */
  int (*allreduce)(void* user, void* buf, uint64_t count, int dtype, int op);
  /* rank r contributes counts[r] bytes from send; recv (sum of counts bytes)
   * receives the contributions concatenated in rank order; send may lie
   * inside recv at its own rank's position */
  int (*allgatherv)(void* user, const void* send, void* recv, const uint64_t* counts);
  /* all-to-all of bytes: send holds the blocks for ranks 0..size-1 back to
   * back (send_counts[k] bytes for rank k), recv receives the blocks from
   * ranks 0..size-1 back to back (recv_counts[k] bytes from rank k) */
  int (*alltoallv)(void* user, const void* send, const uint64_t* send_counts, void* recv,
                   const uint64_t* recv_counts);
} lvn_comm;
int lvn_louvain_sharded(const lvn_csr* g, const lvn_params* p, const lvn_comm* comm, lvn_result** out);

/* Library-owned NCCL communicator (one process per GPU, NVLink / NVSwitch).
 * Rank 0 calls lvn_nccl_unique_id and ships the bytes to the other ranks by
 * any side channel (torchrun store, MPI, a file); every rank then calls
 * lvn_comm_nccl_create on its own device (lvn_init first). Passed to
 * lvn_louvain_sharded, its collectives are enqueued on the engine stream with
 * no host synchronisation; its public callbacks also work standalone
 * (synchronous). NCCL is loaded at run time (libnccl.so.2). */
#define LVN_NCCL_ID_BYTES 128
int lvn_nccl_version(int* version);
int lvn_nccl_unique_id(unsigned char id[LVN_NCCL_ID_BYTES]);
int lvn_comm_nccl_create(int rank, int size, const unsigned char id[LVN_NCCL_ID_BYTES], lvn_comm** out);
int lvn_comm_destroy(lvn_comm* comm);
/* rows [0, n) cut into `parts` contiguous ranges of about A/parts arcs each:
 * bounds[k] = the first row whose offset reaches floor(k A / parts), bounds[parts] = n
 * (host offsets; the engine applies the same rule on the device) */
int lvn_partition_rows(const uint64_t* offsets, uint32_t n, int parts, uint32_t* bounds);

/* ---- device-resident graphs (bench / generators) ----------------------- */
typedef struct lvn_dgraph lvn_dgraph;
/* synthetic generators (SURVEY.md 8(d) C1-C5 shapes), built on the device:
 * kind 0 RMAT(scale, edgefactor), 1 SBM(n, blocks, avg_degree, mu),
 * 2 grid(side, keep_probability), 3 web(n, avg_degree), 4 uniform(n, edges) */
typedef struct lvn_gen_params {
  int kind;
  uint64_t n;
  uint64_t edges;      /* undirected samples (RMAT: 2^scale * edgefactor) */
  uint32_t scale;
  uint32_t blocks;
  double a, b, c;      /* RMAT probabilities */
  double mu;           /* SBM mixing */
  double p;            /* grid keep probability */
  double avg_degree;
  uint64_t seed;
} lvn_gen_params;
int lvn_generate(const lvn_gen_params* gp, lvn_dgraph** out);
int lvn_dgraph_upload(const lvn_csr* host, lvn_dgraph** out);
int lvn_dgraph_view(const lvn_dgraph* g, lvn_csr* view); /* device pointers */
int lvn_dgraph_download(const lvn_dgraph* g, uint64_t* offsets, uint32_t* targets,
                        float* weights);
void lvn_dgraph_free(lvn_dgraph* g);

/* device buffers for device-located memberships (tests) */
int lvn_device_alloc(size_t bytes, void** ptr);
int lvn_device_free(void* ptr);
int lvn_memcpy(void* dst, const void* src, size_t bytes, int kind /* 1 h2d, 2 d2h, 3 d2d */);

#ifdef __cplusplus
}
#endif
#endif /* LVN_H */
