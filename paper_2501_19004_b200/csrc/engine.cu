// Host engine of liblvn.so: device context and pool, the Louvain pass shell
// (compact_impl, louvain_compact.cpp:312-402, re-expressed as a device
// pipeline with one small readback per local-moving iteration), and every
// C-ABI entry point declared in include/lvn.h.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "comm.hpp"
#include "kernels.cuh"
#include "lvn.h"
#include "shard.hpp"

namespace lvn {

// NVTX ranges (header-only NVTX v3: free unless a tool such as nsys/ncu is
// attached) for the run, each pass and its local-moving / aggregation phases,
// so a timeline shows the reference's phase structure
struct Nvtx {
  nvtxRangeId_t id = 0;
  bool open = false;
  explicit Nvtx(const char* name) : id(nvtxRangeStartA(name)), open(true) {}
  Nvtx(const char* fmt, int k) {
    char buf[48];
    std::snprintf(buf, sizeof buf, fmt, k);
    id = nvtxRangeStartA(buf);
    open = true;
  }
  void end() {
    if (open) nvtxRangeEnd(id), open = false;
  }
  ~Nvtx() { end(); }
  Nvtx(const Nvtx&) = delete;
  Nvtx& operator=(const Nvtx&) = delete;
};

std::atomic<unsigned long long> g_launches{0};

void launch_check(const char* file, int line) {
  static const bool debug = [] {
    const char* e = std::getenv("LVN_SYNC_DEBUG");
    return e && *e && *e != '0';
  }();
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cuda_check(cudaGetLastError(), "kernel launch", file, line);
  if (debug) cuda_check(cudaDeviceSynchronize(), "kernel execution (LVN_SYNC_DEBUG)", file, line);
}

// ---------------------------------------------------------------------------
// Pool / context
// ---------------------------------------------------------------------------
void Pool::bind(int device, cudaStream_t s) {
  LVN_CUDA(cudaDeviceGetDefaultMemPool(&pool_, device));
  std::uint64_t keep = ~std::uint64_t(0);
  LVN_CUDA(cudaMemPoolSetAttribute(pool_, cudaMemPoolAttrReleaseThreshold, &keep));
  stream_ = s;
  size_t free_b = 0, total_b = 0;
  LVN_CUDA(cudaMemGetInfo(&free_b, &total_b));
  cache_budget_ = total_b / 4;
  if (const char* e = std::getenv("LVN_CACHE_FRAC")) cache_budget_ = size_t(double(total_b) * std::atof(e));
  total_ = total_b;
}

size_t Pool::available() {
  std::uint64_t used = 0;
  (void)cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrUsedMemCurrent, &used);
  size_t cached = 0;
  for (auto& kv : big_free_) cached += kv.first;
  const size_t margin = size_t(1) << 30;
  const size_t held = used + external_ + margin;
  return held < total_ + cached ? total_ + cached - held : 0;
}

void Pool::refresh_external() {
  std::uint64_t reserved = 0;
  (void)cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrReservedMemCurrent, &reserved);
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
    (void)cudaGetLastError();
    return;
  }
  const size_t inside = size_t(reserved) + free_b;
  external_ = total_b > inside ? total_b - inside : 0;
}

void* Pool::raw(size_t bytes) {
  void* p = nullptr;
  cudaError_t e = cudaMallocAsync(&p, bytes ? bytes : 1, stream_);
  if (e == cudaErrorMemoryAllocation) {
    (void)cudaGetLastError();
    trim();
    e = cudaMallocAsync(&p, bytes ? bytes : 1, stream_);
  }
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? kOom : kCuda,
         "cudaMallocAsync(" + std::to_string(bytes) + " bytes): " + cudaGetErrorString(e));
  }
  return p;
}

constexpr size_t kBigBytes = size_t(64) << 20;

bool pool_nocache() {
  static const bool v = std::getenv("LVN_POOL_NOCACHE") != nullptr;
  return v;
}

void Pool::arena_begin(void* base, size_t bytes) {
  arena_ = static_cast<unsigned char*>(base), arena_cap_ = bytes, arena_used_ = 0, arena_on_ = true;
}
// every arena block is released inside the captured sweep that took it
void Pool::arena_end() { arena_on_ = false, arena_ = nullptr, arena_cap_ = 0; }
void Pool::track_begin() { tracking_ = true, tracked_ = 0; }
size_t Pool::track_end() {
  tracking_ = false;
  return tracked_;
}

void* Pool::get(size_t bytes) {
  const size_t r256 = ((bytes ? bytes : 1) + 255) & ~size_t(255);
  if (tracking_) tracked_ += r256;
  if (arena_on_) {
    if (arena_used_ + r256 > arena_cap_) fail(kInternal, "graph capture arena exhausted");
    void* p = arena_ + arena_used_;
    arena_used_ += r256;
    return p;
  }
  if (bytes >= kBigBytes && !pool_nocache()) {
    const size_t unit = (size_t(1) << (63 - __builtin_clzll(bytes))) / 16;
    const size_t r = (bytes + unit - 1) / unit * unit;
    auto it = big_free_.lower_bound(r);
    void* p = nullptr;
    size_t have = r;
    // any cached block up to 4x the request is reused: growing the pool maps
    // new physical memory (hundreds of ms for the multi-GB tables of a skewed
    // graph), whereas an oversized block only idles memory
    if (it != big_free_.end() && it->first <= 4 * r) {
      p = it->second, have = it->first;
      big_free_.erase(it);
    } else {
      // no cached block fits: hand cached blocks (largest first) back to the
      // device pool while they exceed a quarter of device memory, so a
      // changing working set (generation, a different graph) cannot pin the
      // memory a new size class needs
      size_t cached = 0;
      for (auto& kv : big_free_) cached += kv.first;
      while (!big_free_.empty() && cached + r > cache_budget_) {
        auto last = std::prev(big_free_.end());
        cached -= last->first;
        (void)cudaFreeAsync(last->second, stream_);
        big_free_.erase(last);
      }
      p = raw(r);
    }
    big_used_[p] = have;
    return p;
  }
  void* p = raw(bytes);
  used_.insert(p);
  return p;
}

void Pool::put(void* p) {
  if (!p) return;
  if (arena_ && p >= arena_ && p < arena_ + arena_cap_) return;  // arena blocks live as long as the arena
  auto it = big_used_.find(p);
  if (it != big_used_.end()) {
    big_free_.emplace(it->second, p);
    big_used_.erase(it);
    return;
  }
  if (used_.erase(p)) (void)cudaFreeAsync(p, stream_);
}

void Pool::trim() {
  for (auto& kv : big_free_) (void)cudaFreeAsync(kv.second, stream_);
  big_free_.clear();
  (void)cudaStreamSynchronize(stream_);
  if (pool_) (void)cudaMemPoolTrimTo(pool_, 0);
}

void Pool::report() {
  std::uint64_t v[4] = {0, 0, 0, 0};
  (void)cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrReservedMemCurrent, &v[0]);
  (void)cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrReservedMemHigh, &v[1]);
  (void)cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrUsedMemCurrent, &v[2]);
  (void)cudaMemPoolGetAttribute(pool_, cudaMemPoolAttrUsedMemHigh, &v[3]);
  size_t cached = 0;
  for (auto& kv : big_free_) cached += kv.first;
  std::fprintf(stderr, "[lvn] pool reserved %.2f GB (high %.2f), used %.2f GB (high %.2f), %zu small + %zu big live, "
               "%.2f GB big cached\n", v[0] / 1e9, v[1] / 1e9, v[2] / 1e9, v[3] / 1e9, used_.size(), big_used_.size(),
               cached / 1e9);
}

void Pool::release_all() {
  for (void* p : used_) (void)cudaFreeAsync(p, stream_);
  used_.clear();
  for (auto& kv : big_used_) (void)cudaFreeAsync(kv.first, stream_);
  big_used_.clear();
  for (auto& kv : big_free_) (void)cudaFreeAsync(kv.second, stream_);
  big_free_.clear();
  if (stream_) (void)cudaStreamSynchronize(stream_);
}

void* HostCache::get(size_t bytes) {
  std::lock_guard<std::mutex> lk(mu_);
  const size_t r = (bytes + 4095) & ~size_t(4095);
  auto it = free_.lower_bound(r);
  void* p = nullptr;
  size_t have = r;
  if (it != free_.end() && it->first <= 2 * r) {
    p = it->second, have = it->first;
    free_.erase(it);
  } else {
    LVN_CUDA(cudaMallocHost(&p, r));
  }
  used_[p] = have;
  return p;
}

bool HostCache::put(void* p) {
  std::lock_guard<std::mutex> lk(mu_);
  auto it = used_.find(p);
  if (it == used_.end()) return false;
  free_.emplace(it->second, p);
  used_.erase(it);
  return true;
}

// blocks still held by results are released by lvn_result_free (cudaFreeHost)
HostCache::~HostCache() {
  for (auto& kv : free_) (void)cudaFreeHost(kv.second);
}

static Context* g_ctx = nullptr;
static std::mutex g_ctx_mu;

void init_context(int device) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  if (g_ctx) {
    if (g_ctx->device == device) return;
    fail(kInvalid, "lvn context already initialised on another device; call lvn_finalize first");
  }
  int count = 0;
  LVN_CUDA(cudaGetDeviceCount(&count));
  if (device < 0 || device >= count) fail(kInvalid, "no such CUDA device");
  LVN_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop{};
  LVN_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    fail(kCuda, std::string("liblvn is built for sm_100a (B200); found ") + prop.name);
  auto* c = new Context;
  c->device = device;
  c->sms = prop.multiProcessorCount;
  c->smem_optin = prop.sharedMemPerBlockOptin;
  LVN_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  LVN_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
  c->pool.bind(device, c->stream);
  LVN_CUDA(cudaMallocHost(&c->pinned, 8192 * sizeof(u64)));
  g_ctx = c;
}

Context& ctx() {
  if (!g_ctx) init_context(0);
  return *g_ctx;
}

int sm_count() { return ctx().sms; }

void Context::ensure_aux(int n) {
  while (int(aux.size()) < n) {
    cudaStream_t t;
    LVN_CUDA(cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking));
    aux.push_back(t);
  }
  while (int(aux_ev.size()) < 2 * n + 1) {
    cudaEvent_t e;
    LVN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    aux_ev.push_back(e);
  }
}

void destroy_context() {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  if (!g_ctx) return;
  (void)cudaStreamSynchronize(g_ctx->stream);
  for (cudaStream_t t : g_ctx->aux) (void)cudaStreamDestroy(t);
  for (cudaEvent_t e : g_ctx->aux_ev) (void)cudaEventDestroy(e);
  g_ctx->pool.release_all();
  (void)cudaFreeHost(g_ctx->pinned);
  (void)cudaStreamDestroy(g_ctx->stream);
  (void)cudaStreamDestroy(g_ctx->copy);
  delete g_ctx;
  g_ctx = nullptr;
}

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

template <class T>
T read_scalar(const T* dev, cudaStream_t s) {
  T* h = reinterpret_cast<T*>(ctx().pinned);
  LVN_CUDA(cudaMemcpyAsync(h, dev, sizeof(T), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  return *h;
}

BinEdges edges_of(const lvn_params& p) {
  BinEdges e;
  e.thread_max = p.bin_thread_max;
  e.group_max = p.bin_group_max;
  e.warp_max = p.bin_warp_max;
  e.block_max = p.bin_block_max;
  return e;
}

// validate_params (engine_detail.cpp:16-24) + validate_options (louvain_compact.cpp:22-27)
void validate(const lvn_params& p) {
  if (p.max_passes < 0) fail(kInvalid, "max_passes must be >= 0");
  if (p.max_iterations < 0) fail(kInvalid, "max_iterations must be >= 0");
  if (!(p.tolerance_drop > 0.0)) fail(kInvalid, "tolerance_drop must be > 0");
  if (!(p.aggregation_tolerance > 0.0)) fail(kInvalid, "aggregation_tolerance must be > 0");
  if (p.thread_count < 0) fail(kInvalid, "thread_count must be >= 0");
  if (p.chunk_size < 1) fail(kInvalid, "chunk_size must be >= 1");
  if (p.pick_less_period < 2 || p.pick_less_period % 2 != 0)
    fail(kInvalid, "pick-less period must be even and >= 2");
  if (p.value_bits != 32 && p.value_bits != 64) fail(kInvalid, "value_bits must be 32 or 64");
  if (p.probing < 0 || p.probing > 3) fail(kInvalid, "unknown probing mode");
  if (p.sweep_order != 0 && p.sweep_order != 1) fail(kInvalid, "sweep_order must be 0 or 1");
  if (p.shard_min_arcs_log2 < 0 || p.shard_min_arcs_log2 > 62) fail(kInvalid, "shard_min_arcs_log2 must be in [0, 62]");
  if (p.shard_rounds < 0 || p.shard_rounds > 64) fail(kInvalid, "shard_rounds must be in [0, 64]");
  if (p.first_range_arcs_log2 < 0 || p.first_range_arcs_log2 > 58)
    fail(kInvalid, "first_range_arcs_log2 must be in [0, 58]");
  if (!(p.bin_thread_max <= p.bin_group_max && p.bin_group_max <= p.bin_warp_max &&
        p.bin_warp_max <= p.bin_block_max))
    fail(kInvalid, "degree bin edges must be non-decreasing");
  if (p.bin_thread_max > 8 || p.bin_group_max > 256 || p.bin_warp_max > 256 ||
      p.bin_block_max > 4096)
    fail(kInvalid, "degree bin edges exceed the device kernel capacities (8/256/256/4096)");
}

// pick_less_active (louvain_compact.hpp:22-24)
bool pick_less_active(int iteration, int period) { return (iteration + period / 2) % period == 0; }

// vertices of one degree bin decided per launch (lvn_params.sweep_chunk)
u64 sweep_chunk(const lvn_params& p, u32 nv) {
  if (p.sweep_chunk == 0xFFFFFFFFu) return ~u64(0);
  if (p.sweep_chunk) return p.sweep_chunk;
  (void)nv;
  return ~u64(0);  // automatic policy: set from the quality/throughput study
}

// A graph resident on the device: borrowed device pointers or an uploaded copy.
struct InGraph {
  DGraph g;
  double m = 0.0;
  u64 h2d_bytes = 0;
  DBuf<u64> off;
  DBuf<u32> tgt;
  DBuf<float> w;
};

void check_csr_header(const lvn_csr* in) {
  if (!in) fail(kInvalid, "null graph");
  if (in->num_vertices >= kEmpty) fail(kInvalid, "vertex count collides with the reserved sentinel id");
  if (!in->offsets) fail(kInvalid, "null offsets");
  if (in->num_arcs && (!in->targets || !in->weights)) fail(kInvalid, "null targets/weights");
  if (in->location != LVN_HOST && in->location != LVN_DEVICE) fail(kInvalid, "bad location");
}

// Host weights -> device. Unit / constant-weight inputs (every unweighted
// graph, and the paper's) are detected on the host while the targets are in
// flight over PCIe: a multi-threaded bitwise scan of the host array against
// its first weight. When every weight matches, the device array is filled on
// the device (one kernel at HBM speed) instead of moving 4 B per arc over the
// link; otherwise the array is copied. Either way the device holds exactly
// the caller's bits.
u64 upload_weights(const float* host, float* dev, u64 a, cudaStream_t s, cudaStream_t fill_s = nullptr) {
  if (!a) return 0;
  u32 w0;
  std::memcpy(&w0, host, sizeof(u32));
  const u32* h = reinterpret_cast<const u32*>(host);
  unsigned nt = std::thread::hardware_concurrency();
  nt = std::max(1u, std::min(nt ? nt : 1u, 32u));
  if (a < (u64(1) << 22)) nt = 1;
  std::atomic<bool> differs{false};
  std::vector<std::thread> pool;
  auto scan = [&](u64 b, u64 e) {
    constexpr u64 kStep = u64(1) << 20;
    for (u64 c = b; c < e && !differs.load(std::memory_order_relaxed); c += kStep) {
      const u64 ce = std::min(e, c + kStep);
      u32 acc = 0;
      for (u64 i = c; i < ce; ++i) acc |= h[i] ^ w0;
      if (acc) differs.store(true, std::memory_order_relaxed);
    }
  };
  for (unsigned t = 1; t < nt; ++t) pool.emplace_back(scan, a * t / nt, a * (t + 1) / nt);
  scan(0, a / nt);
  for (auto& th : pool) th.join();
  if (differs.load()) {
    LVN_CUDA(cudaMemcpyAsync(dev, host, a * sizeof(float), cudaMemcpyHostToDevice, s));
    return a * sizeof(float);
  }
  fill_u32(reinterpret_cast<u32*>(dev), a, w0, fill_s ? fill_s : s);
  return 0;
}

void load_graph(const lvn_csr* in, cudaStream_t s, InGraph& out, double* h2d_seconds) {
  check_csr_header(in);
  const u64 n = in->num_vertices, a = in->num_arcs;
  out.m = in->total_weight;
  if (in->location == LVN_DEVICE) {
    out.g = DGraph{u32(n), a, in->offsets, in->targets, in->weights};
    return;
  }
  if (in->offsets[0] != 0 || in->offsets[n] != a)
    fail(kInvalid, "offsets must start at 0 and end at num_arcs");
  const auto t0 = Clock::now();
  out.off.alloc(n + 1);
  out.tgt.alloc(a ? a : 1);
  out.w.alloc(a ? a : 1);
  LVN_CUDA(cudaMemcpyAsync(out.off.p, in->offsets, (n + 1) * sizeof(u64), cudaMemcpyHostToDevice, s));
  if (a) {
    LVN_CUDA(cudaMemcpyAsync(out.tgt.p, in->targets, a * sizeof(u32), cudaMemcpyHostToDevice, s));
    out.h2d_bytes += a * sizeof(u32) + upload_weights(in->weights, out.w.p, a, s);
  }
  out.h2d_bytes += (n + 1) * sizeof(u64);
  LVN_CUDA(cudaStreamSynchronize(s));
  if (h2d_seconds) *h2d_seconds += since(t0);
  out.g = DGraph{u32(n), a, out.off.p, out.tgt.p, out.w.p};
}

// ---- pass 0's first sweep by id ranges, overlapped with the input upload ----
// Large inputs: the first sweep of pass 0 visits R0 consecutive vertex-id
// ranges of ~2^29 arcs each (each with its own degree bins, low degree first
// within a range, like lvn_params.sweep_ranges), for host and device input
// alike. With host input the ranges' targets travel as separate chunks on the
// copy stream and the sweep of range k waits only for chunk k, so the first
// sweep runs under the PCIe transfer instead of after it.
std::vector<u32> split_rows(const u64* off, u32 n, int parts, cudaStream_t s);
struct FirstSweep {
  std::vector<u32> vb;          // range bounds (R0 + 1), empty: one range
  std::vector<cudaEvent_t> ev;  // host input: targets of range k have landed
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  FirstSweep() = default;
  FirstSweep(const FirstSweep&) = delete;
  FirstSweep& operator=(const FirstSweep&) = delete;
  ~FirstSweep() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (t0) cudaEventDestroy(t0);
    if (t1) cudaEventDestroy(t1);
  }
  int ranges() const { return vb.empty() ? 1 : int(vb.size()) - 1; }
};

// 16 ranges when the graph holds 16 ranges' worth of arcs, else one: the
// overlap matters where the upload dominates, and on smaller skewed graphs a
// ranged first sweep changes the dynamics (RMAT-24 with 2^26-arc ranges: Q
// 0.0573 -> 0.052)
int first_range_count(u64 a, int log2) {
  if (log2 <= 0 || log2 >= 59) return 1;
  return (a >> log2) >= 16 ? 16 : 1;
}
std::vector<u32> first_ranges(const u64* host_off, u32 n, u64 a, int log2) {
  const int R0 = first_range_count(a, log2);
  if (R0 < 2) return {};
  std::vector<u32> vb(R0 + 1);
  lvn_partition_rows(host_off, n, R0, vb.data());
  return vb;
}

// load_graph with the targets of host input in first-sweep chunks on the copy
// stream (the compute stream waits for the offsets here, for chunk k before
// sweeping range k); device input: only the range bounds
void load_graph_first(const lvn_csr* in, int log2, cudaStream_t s, InGraph& out, FirstSweep& fs,
                      double* h2d_seconds) {
  check_csr_header(in);
  const u64 n = in->num_vertices, a = in->num_arcs;
  if (in->location == LVN_DEVICE) {
    load_graph(in, s, out, h2d_seconds);
    const int R0 = first_range_count(a, log2);
    if (R0 >= 2) fs.vb = split_rows(in->offsets, u32(n), R0, s);  // the lvn_partition_rows rule
    return;
  }
  if (in->offsets[0] != 0 || in->offsets[n] != a)
    fail(kInvalid, "offsets must start at 0 and end at num_arcs");
  fs.vb = first_ranges(in->offsets, u32(n), a, log2);
  if (fs.vb.empty()) {
    load_graph(in, s, out, h2d_seconds);
    return;
  }
  Context& c = ctx();
  out.m = in->total_weight;
  out.off.alloc(n + 1);
  out.tgt.alloc(a);
  out.w.alloc(a);
  // the copy stream writes pool memory allocated (and maybe last used) on s
  cudaEvent_t ready, off_ev;
  LVN_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  LVN_CUDA(cudaEventCreateWithFlags(&off_ev, cudaEventDisableTiming));
  LVN_CUDA(cudaEventRecord(ready, s));
  LVN_CUDA(cudaStreamWaitEvent(c.copy, ready));
  LVN_CUDA(cudaEventCreate(&fs.t0));
  LVN_CUDA(cudaEventCreate(&fs.t1));
  LVN_CUDA(cudaEventRecord(fs.t0, c.copy));
  LVN_CUDA(cudaMemcpyAsync(out.off.p, in->offsets, (n + 1) * sizeof(u64), cudaMemcpyHostToDevice, c.copy));
  LVN_CUDA(cudaEventRecord(off_ev, c.copy));
  const int R0 = fs.ranges();
  fs.ev.resize(R0);
  for (int k = 0; k < R0; ++k) {
    const u64 a0 = in->offsets[fs.vb[k]], a1 = in->offsets[fs.vb[k + 1]];
    if (a1 > a0)
      LVN_CUDA(cudaMemcpyAsync(out.tgt.p + a0, in->targets + a0, (a1 - a0) * sizeof(u32), cudaMemcpyHostToDevice,
                               c.copy));
    LVN_CUDA(cudaEventCreateWithFlags(&fs.ev[k], cudaEventDisableTiming));
    LVN_CUDA(cudaEventRecord(fs.ev[k], c.copy));
  }
  out.h2d_bytes += (n + 1) * sizeof(u64) + a * sizeof(u32);
  LVN_CUDA(cudaStreamWaitEvent(s, off_ev));
  // weights: verified on the host while the targets are in flight; copied
  // (behind the targets on the copy stream, so the pass reset then waits for
  // the whole input) only when they are not all equal
  const u64 wb = upload_weights(in->weights, out.w.p, a, c.copy, s);
  out.h2d_bytes += wb;
  LVN_CUDA(cudaEventRecord(fs.t1, c.copy));
  if (wb) LVN_CUDA(cudaStreamWaitEvent(s, fs.t1));
  LVN_CUDA(cudaEventDestroy(ready));
  LVN_CUDA(cudaEventDestroy(off_ev));
  out.g = DGraph{u32(n), a, out.off.p, out.tgt.p, out.w.p};
  (void)h2d_seconds;  // timed by the fs events once the run is done
}

// membership-like array on the device (borrowed or uploaded)
struct DevU32 {
  u32* p = nullptr;
  DBuf<u32> own;
};
void load_u32(const u32* src, u64 n, int location, cudaStream_t s, DevU32& out) {
  if (n && !src) fail(kInvalid, "null membership");
  if (location == LVN_DEVICE) {
    out.p = const_cast<u32*>(src);
    return;
  }
  out.own.alloc(n ? n : 1);
  if (n) LVN_CUDA(cudaMemcpyAsync(out.own.p, src, n * sizeof(u32), cudaMemcpyHostToDevice, s));
  out.p = out.own.p;
}

// ---- per-family device timing -------------------------------------------------
struct Timing {
  struct Span {
    cudaEvent_t a, b;
    int fam;
    double bytes;
    ull items, arcs, gathers;
    ull count;  // iterations the span covers (a captured pass: all but its first)
  };
  std::vector<Span> spans;
  std::vector<cudaEvent_t> free_events;
  cudaEvent_t ev() {
    if (!free_events.empty()) {
      cudaEvent_t e = free_events.back();
      free_events.pop_back();
      return e;
    }
    cudaEvent_t e;
    LVN_CUDA(cudaEventCreate(&e));
    return e;
  }
  size_t begin(int fam, cudaStream_t s) {
    Span sp{ev(), ev(), fam, 0.0, 0, 0, 0, 1};
    LVN_CUDA(cudaEventRecord(sp.a, s));
    spans.push_back(sp);
    return spans.size() - 1;
  }
  void end(size_t i, cudaStream_t s, double bytes, ull items = 0, ull arcs = 0) {
    LVN_CUDA(cudaEventRecord(spans[i].b, s));
    spans[i].bytes = bytes;
    spans[i].items = items;
    spans[i].arcs = arcs;
  }
  void set_bytes(size_t i, double bytes, ull items, ull arcs, ull gathers = 0) {
    spans[i].bytes = bytes, spans[i].items = items, spans[i].arcs = arcs, spans[i].gathers = gathers;
  }
  void collect(lvn_phase_stats* st) {
    for (auto& sp : spans) {
      float ms = 0.f;
      LVN_CUDA(cudaEventSynchronize(sp.b));
      LVN_CUDA(cudaEventElapsedTime(&ms, sp.a, sp.b));
      lvn_phase_stats& f = st[sp.fam];
      f.seconds += ms * 1e-3;
      f.bytes += sp.bytes;
      f.launches += sp.count;
      f.items += sp.items;
      f.arcs += sp.arcs;
      f.gathers += sp.gathers;
      free_events.push_back(sp.a);
      free_events.push_back(sp.b);
    }
    spans.clear();
  }
  ~Timing() {
    for (auto& sp : spans) (void)cudaEventDestroy(sp.a), (void)cudaEventDestroy(sp.b);
    for (auto e : free_events) (void)cudaEventDestroy(e);
  }
};

constexpr int kMaxRanges = 64;

struct IterRecord {  // device scratch read back once per iteration
  double gain;
  ull verts, arcs, moves, gathers;
  ull active[kMaxRanges * kBins];  // per-(range, bin) sizes of the next active lists
};

// per-iteration tallies of a captured pass (the IterRecord prefix)
struct IterHist {
  double gain;
  ull verts, arcs, moves, gathers;
};

// End of one captured iteration: keep its tallies, reset them, set the next
// iteration's Pick-Less word and decide on the device whether the while
// node runs again (louvain_compact.cpp:209: stop once the gain is at most
// the tolerance, or after max_iterations).
__global__ void iter_end_k(IterRecord* rec, IterHist* hist, u32* it, double tol, u32 max_it, int period,
                           int* pickless, cudaGraphConditionalHandle h) {
  if (threadIdx.x) return;
  const u32 i = *it;
  const IterHist e{rec->gain, rec->verts, rec->arcs, rec->moves, rec->gathers};
  hist[i] = e;
  rec->gain = 0.0;
  rec->verts = rec->arcs = rec->moves = rec->gathers = 0;
  *it = i + 1;
  *pickless = (int(i + 1) + period / 2) % period == 0;
  cudaGraphSetConditional(h, e.gain > tol && i + 1 < max_it ? 1u : 0u);
}

__global__ void graph_init_k(u32* it, u32 first, int* pickless, int pl) {
  if (threadIdx.x) return;
  *it = first;
  *pickless = pl;
}

// LVN_GRAPH_VERTS_LOG2=k: whole-graph passes of at most 2^k vertices run
// their iterations after the first as ONE launch of a CUDA graph whose while
// node loops on the device; their bins sweep the full degree lists (prune
// flags checked in the kernels) so the body has static launch shapes. Off by
// default: capture + instantiation cost 0.3-0.7 ms per pass, more than the
// host round trips it removes on C1 / C4 (profiles/r02_graph_ab.txt).
// LVN_FORK_VERTS_LOG2=k: passes of at most 2^k vertices run the degree bins
// of a sweep on forked streams, so the launch tails of small classes overlap
// (captured or not). Off by default: C1's local moving drops 1.71 -> 1.15-1.3
// ms, but the looser order costs up to 0.001 Q there, and C1 sits 0.0049
// from the 0.005 quality gate.
int graph_verts_log2() {
  static const int v = [] {
    const char* e = std::getenv("LVN_GRAPH_VERTS_LOG2");
    const char* d = std::getenv("LVN_SYNC_DEBUG");
    if (d && *d && *d != '0') return 0;
    return e ? std::atoi(e) : 0;
  }();
  return v;
}
int fork_verts_log2() {
  static const int v = [] {
    const char* e = std::getenv("LVN_FORK_VERTS_LOG2");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}
constexpr int kForkStreams = 6;

// vertex-id ranges of one sweep (lvn_params.sweep_ranges)
int sweep_ranges(const lvn_params& p, u32 nv) {
  // automatic: one range (LVN_RANGE_LOG2=k: one per 2^k vertices, a tuning aid)
  int r = p.sweep_ranges > 0 ? p.sweep_ranges : 1;
  if (const char* e = std::getenv("LVN_RANGE_LOG2"); e && p.sweep_ranges <= 0)
    r = int((u64(nv) + (u64(1) << std::atoi(e)) - 1) >> std::atoi(e));
  r = std::min(r, kMaxRanges);
  return int(std::max<u64>(1, std::min<u64>(u64(r), nv)));
}

// ---- sharded runs: row split and the caller's collectives ---------------------
// bounds[k] = first row whose offset reaches floor(k A / parts), bounds[parts] = n
__host__ __device__ inline u64 split_target(u64 A, int parts, int k) {
  return A / u64(parts) * u64(k) + (A % u64(parts)) * u64(k) / u64(parts);
}
__global__ void split_rows_k(const u64* __restrict__ off, u32 n, int parts, u32* __restrict__ bounds) {
  for (int k = threadIdx.x; k <= parts; k += blockDim.x) {
    if (k == parts) {
      bounds[k] = n;
      continue;
    }
    const u64 target = split_target(off[n], parts, k);
    u32 lo = 0, hi = n;
    while (lo < hi) {
      const u32 mid = lo + (hi - lo) / 2;
      if (off[mid] >= target) hi = mid; else lo = mid + 1;
    }
    bounds[k] = lo;
  }
}
std::vector<u32> split_rows(const u64* off, u32 n, int parts, cudaStream_t s) {
  DBuf<u32> b(parts + 1);
  split_rows_k<<<1, 1024, 0, s>>>(off, n, parts, b.p);
  LVN_LAUNCH();
  std::vector<u32> h(parts + 1);
  LVN_CUDA(cudaMemcpyAsync(ctx().pinned, b.p, (parts + 1) * sizeof(u32), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  std::memcpy(h.data(), ctx().pinned, (parts + 1) * sizeof(u32));
  return h;
}

struct Comm {
  const lvn_comm* c = nullptr;
  NcclComm* nc = nullptr;  // library-owned NCCL communicator: stream-ordered, no host sync
  double seconds = 0.0;    // host time inside caller collectives / device time of NCCL ones
  std::vector<cudaEvent_t> ev;  // NCCL: (begin, end) event pairs, summed at the end of the run
  bool force = false;       // LVN_SHARD_SINGLE: the sharded path at world size 1
  bool on() const { return c && (c->size > 1 || force); }
  int rank() const { return c ? c->rank : 0; }
  int size() const { return c ? c->size : 1; }
  void mark(cudaStream_t s) {
    cudaEvent_t e;
    LVN_CUDA(cudaEventCreate(&e));
    LVN_CUDA(cudaEventRecord(e, s));
    ev.push_back(e);
  }
  void allreduce(void* buf, u64 count, int dtype, int op, cudaStream_t s) {
    if (nc) {
      mark(s);
      nccl_allreduce(nc, buf, count, dtype, op, s);
      mark(s);
      return;
    }
    LVN_CUDA(cudaStreamSynchronize(s));
    const auto t0 = Clock::now();
    if (c->allreduce(c->user, buf, count, dtype, op) != 0) fail(kCuda, "allreduce collective failed");
    seconds += since(t0);
  }
  void allgatherv(const void* send, void* recv, const std::vector<u64>& counts, cudaStream_t s) {
    if (nc) {
      mark(s);
      nccl_allgatherv(nc, send, recv, counts.data(), s);
      mark(s);
      return;
    }
    LVN_CUDA(cudaStreamSynchronize(s));
    const auto t0 = Clock::now();
    if (c->allgatherv(c->user, send, recv, counts.data()) != 0) fail(kCuda, "allgatherv collective failed");
    seconds += since(t0);
  }
  void alltoallv(const void* send, const std::vector<u64>& scnt, void* recv, const std::vector<u64>& rcnt,
                 cudaStream_t s) {
    if (nc) {
      mark(s);
      nccl_alltoallv(nc, send, scnt.data(), recv, rcnt.data(), s);
      mark(s);
      return;
    }
    if (!c->alltoallv) fail(kInvalid, "lvn_comm without alltoallv: sharded aggregation needs it");
    LVN_CUDA(cudaStreamSynchronize(s));
    const auto t0 = Clock::now();
    if (c->alltoallv(c->user, send, scnt.data(), recv, rcnt.data()) != 0) fail(kCuda, "alltoallv collective failed");
    seconds += since(t0);
  }
  // device time of the NCCL collectives (the stream is idle when called)
  void settle() {
    for (size_t i = 0; i + 1 < ev.size(); i += 2) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ev[i], ev[i + 1]) == cudaSuccess) seconds += ms * 1e-3;
    }
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    ev.clear();
  }
  ~Comm() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
  }
};

// ---- renumbering: ids of C (all < width) -> 0..count-1 ascending, returns count
u32 renumber_device(u32* C, u64 n, u64 width, DBuf<u32>& used, DBuf<u32>& rank, cudaStream_t s,
                    bool apply) {
  used.ensure(width + 1);
  rank.ensure(width + 1);
  mark_used(C, n, used.p, width, s);
  exclusive_scan_u32(used.p, rank.p, width, s);
  const u32 count = read_scalar(rank.p + width, s);
  if (apply) remap(C, n, rank.p, s);
  return count;
}

bool check_mode();

// LVN_VERBOSE=1: per-iteration trace on stderr (tuning aid)
bool verbose() {
  static const bool on = [] {
    const char* e = std::getenv("LVN_VERBOSE");
    return e && *e && *e != '0';
  }();
  return on;
}

// LVN_AGG_SORT_FRAC=f: aggregate by external arcs when a sample finds at most f of them (0.4)
double agg_sort_frac() {
  static const double f = [] {
    const char* e = std::getenv("LVN_AGG_SORT_FRAC");
    return e ? std::atof(e) : 0.4;
  }();
  return f;
}

// LVN_AGG_SORT=0: never aggregate by external arcs (A/B aid)
bool agg_sort_off() {
  static const bool off = [] {
    const char* e = std::getenv("LVN_AGG_SORT");
    return e && e[0] == '0';
  }();
  return off;
}

// holey super-rows with fp64 weights (the partial rows of a sharded aggregation)
struct PartialRows {
  DBuf<u64> hoff;
  DBuf<u32> htgt, fill;
  DBuf<double> hw64;
};

// ---- aggregation of a graph by a contiguous membership ----------------------
// partial != null: the rows stay holey, in fp64 (partial->*), nothing is compacted
void aggregate_device(const DGraph& g, const u32* C, u32 count, const BinEdges& e, OwnedCsr& out,
                      u32* err, cudaStream_t s, bool canonical, const Bins* gbins = nullptr,
                      u32* inexact = nullptr, double* self64 = nullptr, PartialRows* partial = nullptr) {
  DBuf<u32> msize(count ? count : 1);
  DBuf<u64> budget(count + 1), coff(count + 1), boff(count + 1), hoff(count + 1), capped(count + 1),
      ext(count + 1);
  community_counts(g, C, count, msize.p, budget.p, s);
  // Uniform integer weights with few arcs between communities (a clustered
  // unweighted graph's first aggregation): aggregate by the external arcs
  // alone (aggsort.cu) when a sample finds at most 40 % of them (C2 under
  // its planted blocks, 10 %: 17 vs 20 ms; C5's first pass, 25 %: 101 vs
  // 156 ms, profiles/r02_agg_ab.txt); an overflow of the key buffer falls
  // back here with the external-arc counts already made
  bool ext_ready = false;
  double frac = 0;
  if (gbins && g.uniform && g.uw == std::floor(g.uw) && g.uw > 0.f && g.arcs >= (u64(1) << 20) && !agg_sort_off() &&
      external_arcs_few(g, C, agg_sort_frac(), s, &frac)) {
    // key buffer: the sampled fraction with a 20 % margin, bounded by the
    // memory the sort needs (~20 B per key: keys, their sort partner, counts)
    const u64 cap = std::min<u64>(u64(double(g.arcs) * std::min(1.0, frac * 1.2 + 0.01)) + 4096,
                                  ctx().pool.available() / 24);
    if (aggregate_by_external_arcs(g, *gbins, C, count, budget.p, ext.p, cap, out, inexact, self64, s))
      return;
    ext_ready = true;
  }
  exclusive_scan_u32_to_u64(msize.p, coff.p, count, s);
  exclusive_scan_u64(budget.p, boff.p, count, s);
  // Holey row capacity: a super-row's distinct targets are at most its
  // member arcs (the budget) and at most count (engine_detail.cpp:66-75).
  // When those rows would take more than an eighth of the free device memory
  // (C5's first aggregation: ~30 GB), the capacity is tightened to
  // min(ext + 1, count), ext = the community's arcs to other communities
  // (one row pass over the graph, binned like the modularity pass).
  cap_budgets(ext_ready ? ext.p : budget.p, capped.p, count, s, ext_ready);
  exclusive_scan_u64(capped.p, hoff.p, count, s);
  if (!ext_ready && read_scalar(hoff.p + count, s) * 8 > ctx().pool.available() / 8) {
    Bins local;
    const Bins* gb = gbins;
    if (!gb) {
      compute_bins(g.off, g.n, e, local, s);
      gb = &local;
    }
    external_arcs(g, *gb, C, ext.p, count, s);
    cap_budgets(ext.p, capped.p, count, s, true);
    exclusive_scan_u64(capped.p, hoff.p, count, s);
  }
  DBuf<u32> members(g.n ? g.n : 1), cursor(count ? count : 1);
  community_scatter(C, g.n, coff.p, count, cursor.p, members.p, s);
  msize.release();
  Bins ab;
  compute_bins(boff.p, count, e, ab, s);  // synchronises
  if (verbose()) {
    std::fprintf(stderr, "[lvn] aggregate %u communities, budget bins:", count);
    for (int b = 0; b < kBins; ++b) std::fprintf(stderr, " %llu", (unsigned long long)ab.count(b));
    std::fprintf(stderr, " (max budget %llu)\n", (unsigned long long)ab.max_degree);
  }
  const u64 H = read_scalar(hoff.p + count, s);
  DBuf<u32> htgt(H ? H : 1), fill(count ? count : 1);
  DBuf<float> hw(partial ? 0 : (H ? H : 1));
  DBuf<double> hw64(partial ? (H ? H : 1) : 0);
  // communities whose members have no arcs (bin 0) emit nothing and are never visited
  LVN_CUDA(cudaMemsetAsync(fill.p, 0, size_t(count ? count : 1) * sizeof(u32), s));
  AggArgs a;
  a.g = g;
  a.C = C;
  a.count = count;
  a.coff = coff.p;
  a.members = members.p;
  a.boff = boff.p;
  a.hoff = hoff.p;
  a.htgt = htgt.p;
  a.hw = hw.p;
  a.hw64 = partial ? hw64.p : nullptr;
  a.fill = fill.p;
  a.err = err;
  a.inexact = inexact;
  a.self64 = self64;
  if (self64) LVN_CUDA(cudaMemsetAsync(self64, 0, size_t(count ? count : 1) * sizeof(double), s));
  aggregate_rows(a, ab, s);
  if (check_mode()) {
    std::vector<u64> h_coff(count + 1), h_boff(count + 1), h_hoff(count + 1), h_off(u64(g.n) + 1);
    std::vector<u32> h_mem(g.n), h_fill(count), h_C(g.n);
    LVN_CUDA(cudaMemcpyAsync(h_coff.data(), coff.p, (count + 1) * 8, cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaMemcpyAsync(h_boff.data(), boff.p, (count + 1) * 8, cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaMemcpyAsync(h_hoff.data(), hoff.p, (count + 1) * 8, cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaMemcpyAsync(h_off.data(), g.off, (u64(g.n) + 1) * 8, cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaMemcpyAsync(h_mem.data(), members.p, u64(g.n) * 4, cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaMemcpyAsync(h_fill.data(), fill.p, u64(count) * 4, cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaMemcpyAsync(h_C.data(), C, u64(g.n) * 4, cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
    std::vector<u8> seen(g.n, 0);
    for (u32 c = 0; c < count; ++c) {
      u64 deg = 0;
      for (u64 k = h_coff[c]; k < h_coff[c + 1]; ++k) {
        const u32 v = h_mem[k];
        if (v >= g.n || seen[v] || h_C[v] != c)
          fail(kInternal, "LVN_CHECK: community CSR broken at community " + std::to_string(c));
        seen[v] = 1;
        deg += h_off[v + 1] - h_off[v];
      }
      if (deg != h_boff[c + 1] - h_boff[c])
        fail(kInternal, "LVN_CHECK: budget of community " + std::to_string(c) + " is " +
                            std::to_string(h_boff[c + 1] - h_boff[c]) + ", member degrees sum to " +
                            std::to_string(deg));
      if (h_fill[c] > h_hoff[c + 1] - h_hoff[c])
        fail(kInternal, "LVN_CHECK: row " + std::to_string(c) + " emitted " + std::to_string(h_fill[c]) +
                            " entries into capacity " + std::to_string(h_hoff[c + 1] - h_hoff[c]) +
                            " (budget " + std::to_string(deg) + ", members " +
                            std::to_string(h_coff[c + 1] - h_coff[c]) + ")");
    }
  }
  if (partial) {
    partial->hoff = std::move(hoff);
    partial->htgt = std::move(htgt);
    partial->fill = std::move(fill);
    partial->hw64 = std::move(hw64);
    return;
  }
  const u32* rows = fill.p;
  DBuf<u64> noff(count + 1);
  exclusive_scan_u32_to_u64(rows, noff.p, count, s);
  const u64 A = read_scalar(noff.p + count, s);
  out.n = count;
  out.arcs = A;
  out.off = std::move(noff);
  out.tgt.alloc(A ? A : 1);
  out.w.alloc(A ? A : 1);
  DBuf<double> tw(1);
  compact_rows(hoff.p, htgt.p, hw.p, fill.p, out.off.p, count, out.tgt.p, out.w.p, tw.p, s);
  if (canonical && A) {
    DBuf<u32> mx(1);
    reduce_max_u32(rows, count, mx.p, s);
    const u32 max_row = read_scalar(mx.p, s);
    segmented_sort_u32(out.tgt.p, out.w.p, out.off.p, count, max_row, s);
  }
  out.total_weight = read_scalar(tw.p, s) / 2.0;
}

double modularity_device(const DGraph& g, const Bins& b, const u32* C, u64 width, double m,
                         cudaStream_t s) {
  DBuf<double> tot(width ? width : 1), sums(2);
  modularity_terms(g, b, C, tot.p, width, sums.p, s, 2.0 * m);
  double* h = reinterpret_cast<double*>(ctx().pinned);
  LVN_CUDA(cudaMemcpyAsync(h, sums.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  return h[0] / (2.0 * m) - h[1];
}

// ---- sharded storage (lvn_louvain_sharded) --------------------------------------
// Rank `rank` of `size` keeps the rows [v0, v1) of the input (lvn_partition_rows
// rule): full-length offsets with the other rows empty, and only its own
// targets / weights (borrowed slices of device input, uploaded slices of host input).
void load_graph_shard(const lvn_csr* in, int rank, int size, cudaStream_t s, InGraph& out, u32& v0, u32& v1,
                      double* h2d_seconds) {
  check_csr_header(in);
  const u32 n = in->num_vertices;
  out.m = in->total_weight;
  std::vector<u32> b(size + 1);
  out.off.alloc(u64(n) + 1);
  const auto t0 = Clock::now();
  if (in->location == LVN_DEVICE) {
    b = split_rows(in->offsets, n, size, s);
  } else {
    if (in->offsets[0] != 0 || in->offsets[n] != in->num_arcs)
      fail(kInvalid, "offsets must start at 0 and end at num_arcs");
    lvn_partition_rows(in->offsets, n, size, b.data());
  }
  v0 = b[rank], v1 = b[rank + 1];
  const u64* goff = in->offsets;
  DBuf<u64> up;
  if (in->location != LVN_DEVICE) {
    up.alloc(u64(n) + 1);
    LVN_CUDA(cudaMemcpyAsync(up.p, in->offsets, (u64(n) + 1) * sizeof(u64), cudaMemcpyHostToDevice, s));
    out.h2d_bytes += (u64(n) + 1) * sizeof(u64);
    goff = up.p;
  }
  shard_offsets(goff, n, v0, v1, out.off.p, s);
  u64 a0, a1;
  if (in->location == LVN_DEVICE) {
    LVN_CUDA(cudaMemcpyAsync(ctx().pinned, in->offsets + v0, sizeof(u64), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaMemcpyAsync(ctx().pinned + 1, in->offsets + v1, sizeof(u64), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
    a0 = ctx().pinned[0], a1 = ctx().pinned[1];
    out.g = DGraph{n, a1 - a0, out.off.p, in->targets + a0, in->weights + a0};
    return;
  }
  a0 = in->offsets[v0], a1 = in->offsets[v1];
  const u64 a = a1 - a0;
  out.tgt.alloc(a ? a : 1);
  out.w.alloc(a ? a : 1);
  if (a) {
    LVN_CUDA(cudaMemcpyAsync(out.tgt.p, in->targets + a0, a * sizeof(u32), cudaMemcpyHostToDevice, s));
    out.h2d_bytes += a * sizeof(u32) + upload_weights(in->weights + a0, out.w.p, a, s);
  }
  LVN_CUDA(cudaStreamSynchronize(s));
  if (h2d_seconds) *h2d_seconds += since(t0);
  out.g = DGraph{n, a, out.off.p, out.tgt.p, out.w.p};
}

// every rank gets rank 0's n elements of buf (device)
void bcast_from0(Comm& cm, void* buf, u64 bytes, cudaStream_t s) {
  std::vector<u64> counts(cm.size(), 0);
  counts[0] = bytes;
  cm.allgatherv(buf, buf, counts, s);
}

// Aggregation of a sharded pass by own rows (shard.cu): partial super-edges
// routed to the owners of their super-rows, merged there. `out` receives this
// rank's rows [cb[rank], cb[rank+1]) of the next graph (others empty);
// cb = the next pass's row ranges, balanced by super-edge count.
void aggregate_sharded(const DGraph& g, const u32* C, u32 count, u32 v0, u32 v1, Comm& cm, OwnedCsr& out,
                       std::vector<u32>& cb, const BinEdges& edges, u32* err, cudaStream_t s) {
  const int P = cm.size(), me = cm.rank();
  DBuf<ull> keys;
  DBuf<double> vals;
  const u32 kb = key_bits(count);
  // this rank's partial super-rows: the single-GPU hash aggregation over its
  // own rows (the other rows are empty) with fp64 weights, flattened to
  // (row << kb | target, w) entries in row order (LVN_SHARD_AGG_SORT=1: by
  // radix-sorting every own arc instead)
  u64 m = 0;
  static const bool by_sort = [] {
    const char* e = std::getenv("LVN_SHARD_AGG_SORT");
    return e && e[0] == '1';
  }();
  if (by_sort) {
    m = partial_super_edges(g, C, v0, v1, kb, keys, vals, s);
  } else {
    PartialRows pr;
    OwnedCsr unused;
    aggregate_device(g, C, count, edges, unused, err, s, false, nullptr, nullptr, nullptr, &pr);
    m = holey_entries(pr.hoff.p, pr.htgt.p, pr.hw64.p, pr.fill.p, count, kb, keys, vals, s);
  }
  // super-edges per row over all ranks (upper bound of the merged row) -> row ranges
  DBuf<u32> cnt(count ? count : 1);
  super_row_counts(keys.p, m, count, kb, cnt.p, s);
  cm.allreduce(cnt.p, count, LVN_U32, LVN_SUM, s);
  DBuf<u64> coff(u64(count) + 1);
  exclusive_scan_u32_to_u64(cnt.p, coff.p, count, s);
  cb = split_rows(coff.p, count, P, s);
  // route the sorted entries: cut[k] = first entry of rank k's rows
  DBuf<u32> dcb(P + 1);
  DBuf<u64> cut(P + 1), mat(u64(P) * P);
  std::memcpy(ctx().pinned, cb.data(), (P + 1) * sizeof(u32));
  LVN_CUDA(cudaMemcpyAsync(dcb.p, ctx().pinned, (P + 1) * sizeof(u32), cudaMemcpyHostToDevice, s));
  route_entries(keys.p, m, dcb.p, P, kb, cut.p, s);
  // entries this rank sends to each rank, then the whole P x P matrix
  {
    std::vector<u64> h(P + 1);
    LVN_CUDA(cudaMemcpyAsync(ctx().pinned, cut.p, (P + 1) * sizeof(u64), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
    std::memcpy(h.data(), ctx().pinned, (P + 1) * sizeof(u64));
    for (int k = 0; k < P; ++k) ctx().pinned[k] = h[k + 1] - h[k];
    LVN_CUDA(cudaMemcpyAsync(mat.p + u64(me) * P, ctx().pinned, P * sizeof(u64), cudaMemcpyHostToDevice, s));
    cm.allgatherv(mat.p + u64(me) * P, mat.p, std::vector<u64>(P, 8ull * P), s);
  }
  std::vector<u64> M(u64(P) * P);
  LVN_CUDA(cudaMemcpyAsync(ctx().pinned, mat.p, u64(P) * P * sizeof(u64), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  std::memcpy(M.data(), ctx().pinned, u64(P) * P * sizeof(u64));
  std::vector<u64> sk(P), sv(P), rk(P), rv(P);
  u64 total = 0;
  for (int k = 0; k < P; ++k) {
    sk[k] = 8 * M[u64(me) * P + k], sv[k] = sk[k];
    rk[k] = 8 * M[u64(k) * P + me], rv[k] = rk[k];
    total += M[u64(k) * P + me];
  }
  DBuf<ull> rkeys(total ? total : 1);
  DBuf<double> rvals(total ? total : 1);
  cm.alltoallv(keys.p, sk, rkeys.p, rk, s);
  cm.alltoallv(vals.p, sv, rvals.p, rv, s);
  keys.release();
  vals.release();
  DBuf<double> tw(1);
  merge_super_rows(rkeys, rvals, total, count, kb, out, tw.p, s);
  cm.allreduce(tw.p, 1, LVN_F64, LVN_SUM, s);
  out.total_weight = read_scalar(tw.p, s) / 2.0;
}

// the whole graph on every rank from each rank's own rows (contiguous ranges
// in rank order): row lengths summed over ranks, arcs gathered in rank order
void gather_graph(OwnedCsr& g, Comm& cm, cudaStream_t s) {
  const int P = cm.size();
  const u32 n = g.n;
  DBuf<u32> len(n ? n : 1);
  row_lengths(g.off.p, n, len.p, s);
  cm.allreduce(len.p, n, LVN_U32, LVN_SUM, s);
  DBuf<u64> arcs(P);
  LVN_CUDA(cudaMemcpyAsync(arcs.p + cm.rank(), &g.arcs, sizeof(u64), cudaMemcpyHostToDevice, s));
  cm.allgatherv(arcs.p + cm.rank(), arcs.p, std::vector<u64>(P, 8), s);
  std::vector<u64> a(P);
  LVN_CUDA(cudaMemcpyAsync(ctx().pinned, arcs.p, P * sizeof(u64), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  u64 A = 0;
  for (int k = 0; k < P; ++k) a[k] = ctx().pinned[k], A += a[k];
  OwnedCsr full;
  full.n = n;
  full.arcs = A;
  full.total_weight = g.total_weight;
  full.off.alloc(u64(n) + 1);
  exclusive_scan_u32_to_u64(len.p, full.off.p, n, s);
  full.tgt.alloc(A ? A : 1);
  full.w.alloc(A ? A : 1);
  std::vector<u64> bytes(P);
  for (int k = 0; k < P; ++k) bytes[k] = 4 * a[k];
  cm.allgatherv(g.tgt.p, full.tgt.p, bytes, s);
  cm.allgatherv(g.w.p, full.w.p, bytes, s);
  g = std::move(full);
}

// modularity of a sharded input: per-community terms of the own rows, summed over ranks
double modularity_sharded(const DGraph& g, const Bins& b, const u32* C, u64 width, double m, Comm& cm,
                          cudaStream_t s) {
  DBuf<double> tot(width ? width : 1), sums(2);
  modularity_rows(g, b, C, tot.p, width, sums.p, s);
  cm.allreduce(tot.p, width, LVN_F64, LVN_SUM, s);
  cm.allreduce(sums.p, 1, LVN_F64, LVN_SUM, s);
  modularity_squares(tot.p, width, 2.0 * m, sums.p, s);
  double* h = reinterpret_cast<double*>(ctx().pinned);
  LVN_CUDA(cudaMemcpyAsync(h, sums.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  return h[0] / (2.0 * m) - h[1];
}

// LVN_CHECK=1: validate device state between phases (debugging aid; copies
// state to the host, so it is never enabled in measured runs)
bool check_mode() {
  static const bool on = [] {
    const char* e = std::getenv("LVN_CHECK");
    return e && *e && *e != '0';
  }();
  return on;
}

void check_membership(const char* what, const u32* C, u64 n, u64 bound, cudaStream_t s) {
  if (!check_mode()) return;
  std::vector<u32> h(n);
  if (n) LVN_CUDA(cudaMemcpyAsync(h.data(), C, n * 4, cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  for (u64 i = 0; i < n; ++i)
    if (h[i] >= bound)
      fail(kInternal, std::string("LVN_CHECK ") + what + ": id " + std::to_string(h[i]) + " at " +
                          std::to_string(i) + " >= " + std::to_string(bound));
}

void check_graph(const char* what, const DGraph& g, cudaStream_t s) {
  if (!check_mode()) return;
  std::vector<u64> off(u64(g.n) + 1);
  std::vector<u32> tgt(g.arcs);
  std::vector<float> w(g.arcs);
  LVN_CUDA(cudaMemcpyAsync(off.data(), g.off, off.size() * 8, cudaMemcpyDeviceToHost, s));
  if (g.arcs) {
    LVN_CUDA(cudaMemcpyAsync(tgt.data(), g.tgt, g.arcs * 4, cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaMemcpyAsync(w.data(), g.w, g.arcs * 4, cudaMemcpyDeviceToHost, s));
  }
  LVN_CUDA(cudaStreamSynchronize(s));
  auto bad = [&](const std::string& m) { fail(kInternal, std::string("LVN_CHECK ") + what + ": " + m); };
  if (off[0] != 0 || off[g.n] != g.arcs) bad("offsets do not span the arcs");
  for (u64 v = 0; v < g.n; ++v)
    if (off[v + 1] < off[v]) bad("offsets decrease at row " + std::to_string(v));
  for (u64 a = 0; a < g.arcs; ++a) {
    if (tgt[a] >= g.n) bad("target " + std::to_string(tgt[a]) + " out of range at arc " + std::to_string(a));
    if (!(w[a] >= 0.0f)) bad("bad weight at arc " + std::to_string(a));
  }
}

void check_err(const u32* err, cudaStream_t s) {
  const u32 e = read_scalar(err, s);
  if (e & kErrLookup) fail(kInternal, "dendrogram lookup index out of range");
  if (e & kErrTable) fail(kInternal, "scan table exhausted; capacity invariant violated");
  if (e & kErrRange) fail(kInternal, "community id out of range in a local-moving table");
  if (e) fail(kInternal, "device invariant violated");
}

// ---------------------------------------------------------------------------
// Captured local moving (late / small passes)
// ---------------------------------------------------------------------------
// Iterations 1.. of a pass as one graph launch: a while node whose body is
// the sweep (degree bins serial, or forked onto parallel branches) and
// iter_end_k, which sets the loop condition on the device. The body's
// transient buffers (hub scratch, scan partials) come from an arena sized by
// the uncaptured first sweep. No host round trip until the pass converges;
// returns the iterations run.
struct CaptureScope {  // ends an open capture / arena if a failure unwinds through it
  cudaStream_t s;
  bool open = false;
  ~CaptureScope() {
    if (!open) return;
    ctx().pool.arena_end();
    cudaGraph_t g = nullptr;
    (void)cudaStreamEndCapture(s, &g);
    if (g) (void)cudaGraphDestroy(g);
    (void)cudaGetLastError();
  }
};

int graph_iterations(MoveArgs a, const BinView& view, const lvn_params& p, double tolerance, size_t sweep_bytes,
                     bool fork, IterRecord* rec, int pass, Timing& tm, cudaStream_t s) {
  Context& c = ctx();
  const u32 max_it = u32(p.max_iterations);
  DBuf<u32> itc(1);
  DBuf<int> plw(1);
  DBuf<IterHist> hist(max_it);
  DBuf<unsigned char> arena(sweep_bytes + 4096);
  if (fork) c.ensure_aux(kForkStreams);
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ex = nullptr;
  LVN_CUDA(cudaGraphCreate(&g, 0));
  struct Owned {
    cudaGraph_t& g;
    cudaGraphExec_t& ex;
    ~Owned() {
      if (ex) (void)cudaGraphExecDestroy(ex);
      if (g) (void)cudaGraphDestroy(g);
    }
  } owned{g, ex};
  cudaGraphConditionalHandle h;
  LVN_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np{};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  LVN_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  a.pickless_dev = plw.p;
  a.nfork = fork ? kForkStreams : 0;
  const ull l0 = g_launches.load();
  {
    CaptureScope cs{s};
    LVN_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    cs.open = true;
    c.pool.arena_begin(arena.p, arena.n);
    move_sweep(a, view, p.value_bits, s);
    iter_end_k<<<1, 32, 0, s>>>(rec, hist.p, itc.p, tolerance, max_it, p.pick_less_period, plw.p, h);
    LVN_LAUNCH();
    c.pool.arena_end();
    cs.open = false;
    cudaGraph_t out = nullptr;
    LVN_CUDA(cudaStreamEndCapture(s, &out));
  }
  const ull per = g_launches.load() - l0;
  LVN_CUDA(cudaGraphInstantiate(&ex, g, 0));
  LVN_CUDA(cudaMemsetAsync(rec, 0, sizeof(IterRecord), s));
  graph_init_k<<<1, 32, 0, s>>>(itc.p, 1u, plw.p, pick_less_active(1, p.pick_less_period) ? 1 : 0);
  LVN_LAUNCH();
  const size_t sp = tm.begin(LVN_STAT_MOVE, s);
  LVN_CUDA(cudaGraphLaunch(ex, s));
  tm.end(sp, s, 0.0);
  u32 n = 1;
  {
    u32* hn = reinterpret_cast<u32*>(c.pinned);
    LVN_CUDA(cudaMemcpyAsync(hn, itc.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
    n = std::min(*hn, max_it);
  }
  std::vector<IterHist> hh(n);
  LVN_CUDA(cudaMemcpyAsync(hh.data(), hist.p, n * sizeof(IterHist), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  double bytes = 0;
  ull verts = 0, arcs = 0, gathers = 0;
  for (u32 i = 1; i < n; ++i) {
    bytes += 12.0 * double(hh[i].arcs) + 32.0 * double(hh[i].verts);
    verts += hh[i].verts, arcs += hh[i].arcs, gathers += hh[i].gathers;
    if (verbose())
      std::fprintf(stderr, "[lvn] pass %d it %u (graph%s): %llu vertices, %llu arcs, %llu moves, gain %.6g\n", pass,
                   i, fork ? ", forked bins" : "", (unsigned long long)hh[i].verts, (unsigned long long)hh[i].arcs,
                   (unsigned long long)hh[i].moves, hh[i].gain);
  }
  tm.set_bytes(sp, bytes, verts, arcs, gathers);
  tm.spans[sp].count = n > 1 ? n - 1 : 1;
  // the body's kernels ran once per iteration (counted once at capture)
  if (n > 2) g_launches += per * (n - 2);
  return int(n) - 1;
}

// ---------------------------------------------------------------------------
// Louvain pass shell
// ---------------------------------------------------------------------------
// comm (lvn_louvain_sharded): passes with >= 2^shard_min_arcs_log2 arcs are
// sharded by row range across the ranks; every rank keeps the
// whole current graph, the replicated C / Sigma / flags, and ends with the same
// result (the passes that run whole run redundantly on every rank).
bool no_uniform() {
  static const bool v = [] {
    const char* e = std::getenv("LVN_UNIFORM");
    return e && std::string(e) == "0";
  }();
  return v;
}

void run_louvain(const lvn_csr* in, const lvn_params& p, lvn_result* r, Comm* comm = nullptr) {
  const auto t_start = Clock::now();
  Context& c = ctx();
  cudaStream_t s = c.stream;
  validate(p);
  check_csr_header(in);
  const double m = in->total_weight;
  if (!(m > 0.0)) fail(kDegenerate, "cannot cluster a graph with zero total weight");
  set_probing_move(p.probing, s);
  set_probing_aggregate(p.probing, s);
  Comm solo;
  Comm& cm = comm ? *comm : solo;
  // Sharded runs: while a pass's graph has >= shard_min arcs
  // every rank holds and sweeps only its own rows [v0, v1); below it the graph
  // is gathered onto rank 0, which runs the rest alone (`idle` elsewhere).
  const bool dist = cm.on();
  const u64 shard_min = u64(1) << p.shard_min_arcs_log2;
  bool sharded = dist && in->num_arcs >= shard_min;
  const bool input_sharded = sharded;
  bool idle = dist && !sharded && cm.rank() != 0;
  bool collapsed = dist && !sharded;
  const u32 N = in->num_vertices;
  u32 v0 = 0, v1 = N;
  InGraph ig;
  FirstSweep fs;
  if (sharded) {
    load_graph_shard(in, cm.rank(), cm.size(), s, ig, v0, v1, &r->h2d_seconds);
  } else if (!idle) {
    load_graph_first(in, p.first_range_arcs_log2, s, ig, fs, &r->h2d_seconds);
  } else {
    ig.g.n = N;
  }
  const BinEdges edges = edges_of(p);
  Timing tm;

  DBuf<u32> global(N ? N : 1), C(N ? N : 1), used, rank, active, csize;
  DBuf<double> K(N ? N : 1), S(N ? N : 1);
  HubPlan hubs;
  DBuf<u8> flags(N ? N : 1);
  DBuf<IterRecord> rec(1);
  DBuf<u32> err(1), uni(1), inexact(1);
  LVN_CUDA(cudaMemsetAsync(err.p, 0, sizeof(u32), s));
  LVN_CUDA(cudaMemsetAsync(inexact.p, 0, sizeof(u32), s));
  iota_u32(global.p, N, s);
  // the pass the loop ended in left its local membership of `cur` in C (a
  // break), else `cur` is the last aggregated graph (its vertices are the
  // final communities)
  bool ended_in_C = false;
  // exact fp64 total degree and self-loop of every vertex of `cur` after an
  // aggregation (for the final modularity on the last super-graph)
  DBuf<double> kx_cur, kx_next, self_cur, self_next;

  Bins in_bins, bins;
  bool have_in_bins = false;
  OwnedCsr owned[2];
  DGraph cur = ig.g;
  double tolerance = p.initial_tolerance;
  double t_move = 0.0, t_aggregate = 0.0;
  std::vector<int> its;
  std::vector<double> tols, pass_secs;
  std::vector<u32> vpp;
  std::vector<u64> app;
  int passes = 0, aggregations = 0, sharded_passes = 0;
  DBuf<u32> mrec, mall, mcount;  // sharded: own move records (u, to), everyone's, per-rank counts
  DBuf<u64> segbuf;              // sharded (NCCL): record block offsets of a round
  struct Levels : std::vector<u32*> {  // dendrogram (p.keep_levels): local membership of every pass
    ~Levels() {
      for (u32* q : *this) std::free(q);
    }
  } levels;
  auto keep_level = [&](u32 nv) {
    if (!p.keep_levels) return;
    u32* h = static_cast<u32*>(std::malloc(size_t(nv ? nv : 1) * sizeof(u32)));
    if (!h) fail(kOom, "host allocation failed");
    if (nv) LVN_CUDA(cudaMemcpyAsync(h, C.p, size_t(nv) * sizeof(u32), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
    levels.push_back(h);
  };

  for (int pass = 0; pass < p.max_passes && !idle; ++pass) {
    const auto t_pass = Clock::now();
    Nvtx r_pass("pass %d", pass);
    const u32 nv = cur.n;
    if (!sharded) v0 = 0, v1 = nv;  // a whole-graph pass owns every row
    Bins& B = pass == 0 ? in_bins : bins;
    // sharded: the bins (and every sweep) cover the own rows only
    if (sharded) compute_bins(cur.off + v0, v1 - v0, edges, B, s, ~u64(0), v0);
    else compute_bins(cur.off, nv, edges, B, s);
    if (pass == 0) have_in_bins = true;
    size_t sp = tm.begin(LVN_STAT_RESET, s);
    pass_reset(cur, B, K.p, S.p, C.p, flags.p, s, uni.p);
    tm.end(sp, s, 4.0 * double(cur.arcs) + 29.0 * nv);
    std::vector<u32> vb;  // sharded: every rank's first row (and nv)
    if (sharded) {
      // K of every vertex from its owner; Sigma = K (singletons)
      vb.assign(cm.size() + 1, 0);
      std::vector<u64> kb(cm.size());
      {
        DBuf<u32> rb(cm.size() + 1);
        std::vector<u64> four(cm.size(), 4);
        LVN_CUDA(cudaMemcpyAsync(rb.p + cm.rank(), &v0, sizeof(u32), cudaMemcpyHostToDevice, s));
        cm.allgatherv(rb.p + cm.rank(), rb.p, four, s);
        LVN_CUDA(cudaMemcpyAsync(c.pinned, rb.p, cm.size() * sizeof(u32), cudaMemcpyDeviceToHost, s));
        LVN_CUDA(cudaStreamSynchronize(s));
        const u32* h = reinterpret_cast<const u32*>(c.pinned);
        for (int k = 0; k < cm.size(); ++k) vb[k] = h[k];
        vb[cm.size()] = nv;
      }
      for (int k = 0; k < cm.size(); ++k) kb[k] = 8ull * (vb[k + 1] - vb[k]);
      cm.allgatherv(K.p + v0, K.p, kb, s);
      LVN_CUDA(cudaMemcpyAsync(S.p, K.p, size_t(nv) * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    // uniform arc weights (every unit-weight input's first pass): the sort
    // bins key on the community alone (LVN_UNIFORM=0 disables)
    bool uniform = false;
    float uniform_w = 0.f;
    if (!no_uniform()) {
      if (sharded) {
        // uniform on every rank, with the same weight: [0] = some rank differs,
        // [1] = max weight bits, [2] = max of the complemented bits
        DBuf<u32> u3(3);
        const u32 mine = read_scalar(uni.p, s);
        u32 h3[3];
        float wf = 0.f;
        if (cur.arcs) {
          LVN_CUDA(cudaMemcpyAsync(c.pinned, cur.w, sizeof(float), cudaMemcpyDeviceToHost, s));
          LVN_CUDA(cudaStreamSynchronize(s));
          std::memcpy(&wf, c.pinned, sizeof(float));
        }
        u32 wb;
        std::memcpy(&wb, &wf, sizeof(u32));
        h3[0] = cur.arcs && mine == 0 ? 1u : 0u;
        h3[1] = cur.arcs ? wb : 0u;
        h3[2] = cur.arcs ? ~wb : 0u;
        std::memcpy(c.pinned, h3, sizeof(h3));
        LVN_CUDA(cudaMemcpyAsync(u3.p, c.pinned, sizeof(h3), cudaMemcpyHostToDevice, s));
        cm.allreduce(u3.p, 3, LVN_U32, LVN_MAX, s);
        LVN_CUDA(cudaMemcpyAsync(c.pinned, u3.p, sizeof(h3), cudaMemcpyDeviceToHost, s));
        LVN_CUDA(cudaStreamSynchronize(s));
        std::memcpy(h3, c.pinned, sizeof(h3));
        uniform = h3[0] == 0 && h3[1] == ~h3[2];
        if (uniform) std::memcpy(&uniform_w, &h3[1], sizeof(float));
      } else if (cur.arcs) {
        uniform = read_scalar(uni.p, s) != 0;
        if (uniform) uniform_w = read_scalar(cur.w, s);
      }
    }
    // kernels of this pass (sweeps, aggregation) take the constant weight
    cur.uniform = uniform ? 1 : 0;
    cur.uw = uniform_w;
    if (pass == 0) ig.g.uniform = cur.uniform, ig.g.uw = uniform_w;

    const bool shard = sharded;
    if (shard) {
      mrec.ensure(2 * u64(std::max<u32>(v1 - v0, 1)));
      mcount.ensure(cm.size() + 1);
      ++sharded_passes;
    }
    Bins& SB = B;
    MoveArgs a;
    a.g = cur;
    a.C = C.p;
    a.K = K.p;
    a.sigma = S.p;
    a.flags = flags.p;
    a.m = m;
    a.prune = p.prune;
    a.gain_acc = &rec.p->gain;
    a.counters = &rec.p->verts;
    a.err = err.p;
    a.chunk = sweep_chunk(p, nv);
    a.uniform = uniform;
    a.uniform_w = uniform_w;
    // LVN_HUB_CHUNK=k: decide the block / hub bins k vertices per launch, so
    // later hubs see earlier hubs' moves (tuning aid; +0.0003 Q on RMAT-24)
    if (const char* e = std::getenv("LVN_HUB_CHUNK")) a.hub_chunk = std::strtoull(e, nullptr, 10);
    if (const char* e = std::getenv("LVN_L2_KEEP")) a.l2_keep = std::atoi(e);
    a.hubs_first = p.sweep_order == 1;
    if (p.singleton_rule) {
      csize.ensure(nv ? nv : 1);
      fill_u32(csize.p, nv, 1u, s);
      a.csize = csize.p;
    }
    if (shard) a.moves_out = mrec.p, a.moves_n = mcount.p + cm.size();
    if (SB.count(kBinGlobal)) {
      hub_plan_build(cur, SB.of(kBinGlobal), SB.count(kBinGlobal), p.value_bits, hubs, s);
      hubs.attach(a);
    }
    // A sweep visits R consecutive vertex-id ranges in order, each with its own
    // degree bins: within a range the degree classes run low to high (the
    // reference compact order), across ranges the sweep follows vertex ids
    // like louvain_mc's, which matters for quality on skewed graphs.
    // Sharded: the own rows are swept in R = shard_rounds consecutive ranges
    // with an exchange after each, so later rounds see the other ranks' moves.
    const int R = shard ? std::max(1, std::min(p.shard_rounds ? p.shard_rounds : 2 * cm.size(), kMaxRanges))
                        : sweep_ranges(p, nv);
    std::vector<Bins> rbins(R > 1 ? R : 0);
    std::vector<u64> rbase(R + 1);
    for (int k = 0; k <= R; ++k) rbase[k] = v0 + u64(v1 - v0) * k / R;
    std::vector<BinView> views(R);
    for (int k = 0; k < R; ++k) {
      if (R > 1)
        compute_bins(cur.off + rbase[k], u32(rbase[k + 1] - rbase[k]), edges, rbins[k], s, ~u64(0),
                     u32(rbase[k]));
      views[k] = R > 1 ? rbins[k].view() : SB.view();
    }
    // pass 0's first sweep by id ranges (FirstSweep), each waiting for its chunk
    const int R0 = pass == 0 ? fs.ranges() : 1;
    std::vector<Bins> fbins(R0 > 1 ? R0 : 0);
    for (int k = 0; k < R0 && R0 > 1; ++k)
      compute_bins(cur.off + fs.vb[k], fs.vb[k + 1] - fs.vb[k], edges, fbins[k], s, ~u64(0), fs.vb[k]);
    const auto t0 = Clock::now();
    Nvtx r_move("local moving");
    int iterations = 0;
    // iteration 0 sweeps every row with arcs (all flagged); later iterations
    // sweep the flagged rows only, compacted right after the previous sweep
    // (graph-mode passes: the full lists, see graph_verts_log2)
    active.ensure(nv ? nv : 1);
    const int gl2 = graph_verts_log2();
    const bool graph_pass = !shard && R == 1 && R0 == 1 && gl2 > 0 && u64(nv) <= (u64(1) << gl2) &&
                            p.max_iterations > 1 && move_kernel_variant() == 0 && p.pick_less_period > 0;
    a.full_lists = graph_pass ? 1 : 0;
    const bool fork = !shard && fork_verts_log2() >= 0 && u64(nv) <= (u64(1) << fork_verts_log2());
    if (fork) c.ensure_aux(kForkStreams);
    a.nfork = fork ? kForkStreams : 0;
    size_t sweep_bytes = 0;
    for (int it = 0; it < p.max_iterations; ++it) {
      a.pickless = pick_less_active(it, p.pick_less_period);
      LVN_CUDA(cudaMemsetAsync(rec.p, 0, sizeof(IterRecord), s));
      size_t sp0 = 0;
      if (it == 0 && R0 > 1) {
        for (int k = 0; k < R0; ++k) {
          if (!fs.ev.empty()) LVN_CUDA(cudaStreamWaitEvent(s, fs.ev[k]));
          sp = tm.begin(LVN_STAT_MOVE, s);
          if (k == 0) sp0 = sp;
          else tm.spans[sp].count = 0;  // stats count one launch per iteration (sweep)
          move_sweep(a, fbins[k].view(), p.value_bits, s);
          tm.end(sp, s, 0.0);
        }
      }
      for (int k = 0; k < R && !(it == 0 && R0 > 1); ++k) {
        if (shard) LVN_CUDA(cudaMemsetAsync(a.moves_n, 0, sizeof(u32), s));
        sp = tm.begin(LVN_STAT_MOVE, s);
        if (k == 0) sp0 = sp;
        else tm.spans[sp].count = 0;
        if (graph_pass) c.pool.track_begin();
        move_sweep(a, views[k], p.value_bits, s);
        if (graph_pass) sweep_bytes = c.pool.track_end();
        tm.end(sp, s, 0.0);
        if (shard) {
          // every rank applies the other ranks' moves of this round (C, Sigma)
          // from their (u, to) records; marks of remote movers' neighbours are
          // OR-reduced at the end of the iteration
          std::vector<u64> four(cm.size(), 4);
          cm.allgatherv(a.moves_n, mcount.p, four, s);
          if (cm.nc) {
            // library NCCL: no host round trip. Every rank's record block has
            // the capacity of its round (one record per vertex of the round,
            // known to all from the row bounds); the apply kernel reads the
            // real counts from device memory.
            const int P = cm.size();
            std::vector<u64> bytes(P), segoff(P + 1, 0);
            for (int j = 0; j < P; ++j) {
              const u64 lo = vb[j] + u64(vb[j + 1] - vb[j]) * k / R;
              const u64 hi = vb[j] + u64(vb[j + 1] - vb[j]) * (k + 1) / R;
              bytes[j] = 8 * (hi - lo);
              segoff[j + 1] = segoff[j] + (hi - lo);
            }
            if (segoff[P]) {
              mall.ensure(2 * segoff[P]);
              segbuf.ensure(P + 1);
              // pageable source: staged before the call returns (no reuse race
              // with the next round, which does not wait for this copy)
              LVN_CUDA(cudaMemcpyAsync(segbuf.p, segoff.data(), (P + 1) * sizeof(u64), cudaMemcpyHostToDevice, s));
              cm.allgatherv(mrec.p, mall.p, bytes, s);
              apply_moves_segments(mall.p, segbuf.p, mcount.p, P, cm.rank(), segoff[P], C.p, K.p, S.p, s);
            }
            continue;
          }
          u32* hn = reinterpret_cast<u32*>(c.pinned);
          LVN_CUDA(cudaMemcpyAsync(hn, mcount.p, cm.size() * sizeof(u32), cudaMemcpyDeviceToHost, s));
          LVN_CUDA(cudaStreamSynchronize(s));
          std::vector<u64> bytes(cm.size());
          u64 total = 0, mine = 0;
          for (int j = 0; j < cm.size(); ++j) {
            if (j == cm.rank()) mine = total;
            bytes[j] = 8ull * hn[j];
            total += hn[j];
          }
          const u64 own_n = hn[cm.rank()];
          if (total) {
            mall.ensure(2 * total);
            cm.allgatherv(mrec.p, mall.p, bytes, s);
            apply_moves(mall.p, total, mine, mine + own_n, cur, C.p, K.p, S.p, flags.p, 0, s);
          }
        }
      }
      sp = sp0;
      if (shard) {
        cm.allreduce(&rec.p->gain, 1, LVN_F64, LVN_SUM, s);
        cm.allreduce(&rec.p->verts, 4, LVN_U64, LVN_SUM, s);
        if (p.prune) {
          cm.allreduce(flags.p, nv, LVN_U8, LVN_MAX, s);
          zero_outside(flags.p, nv, v0, v1, s);
        }
      }
      if (p.prune && !graph_pass)
        for (int k = 0; k < R; ++k)
          compact_active(R > 1 ? rbins[k] : SB, flags.p, active.p + rbase[k], rec.p->active + k * kBins, s);
      IterRecord* h = reinterpret_cast<IterRecord*>(c.pinned);
      LVN_CUDA(cudaMemcpyAsync(h, rec.p, sizeof(IterRecord), cudaMemcpyDeviceToHost, s));
      LVN_CUDA(cudaStreamSynchronize(s));
      tm.set_bytes(sp, 12.0 * double(h->arcs) + 32.0 * double(h->verts), h->verts, h->arcs, h->gathers);
      if (verbose())
        std::fprintf(stderr, "[lvn] pass %d it %d: %llu vertices, %llu arcs, %llu moves, gain %.6g\n", pass, it,
                     (unsigned long long)h->verts, (unsigned long long)h->arcs, (unsigned long long)h->moves,
                     h->gain);
      ++iterations;
      if (h->gain <= tolerance) break;  // louvain_compact.cpp:209
      if (graph_pass) {
        iterations += graph_iterations(a, views[0], p, tolerance, sweep_bytes, fork, rec.p, pass, tm, s);
        break;
      }
      if (p.prune)
        for (int k = 0; k < R; ++k) {
          views[k].list = active.p + rbase[k];
          for (int b = 0; b < kBins; ++b) views[k].cnt[b] = h->active[k * kBins + b];
        }
    }
    for (cudaEvent_t e : (pass == 0 ? fs.ev : std::vector<cudaEvent_t>())) LVN_CUDA(cudaStreamWaitEvent(s, e));
    t_move += since(t0);
    r_move.end();
    check_err(err.p, s);
    check_membership("after local moving", C.p, nv, nv, s);
    ++passes;
    its.push_back(iterations);
    tols.push_back(tolerance);
    vpp.push_back(nv);
    app.push_back(cur.arcs);

    if (iterations <= 1) {  // no effective movement (louvain_compact.cpp:370-374)
      ended_in_C = true;
      keep_level(nv);
      sp = tm.begin(LVN_STAT_RENUMBER, s);
      lookup(global.p, N, C.p, nv, err.p, s);
      tm.end(sp, s, 12.0 * N);
      pass_secs.push_back(since(t_pass));
      break;
    }
    sp = tm.begin(LVN_STAT_RENUMBER, s);
    const u32 count = renumber_device(C.p, nv, nv, used, rank, s, false);
    tm.end(sp, s, 12.0 * nv);
    if (double(count) / nv > p.aggregation_tolerance) {  // low shrink (louvain_compact.cpp:375-380)
      ended_in_C = true;
      keep_level(nv);
      sp = tm.begin(LVN_STAT_RENUMBER, s);
      lookup(global.p, N, C.p, nv, err.p, s);
      tm.end(sp, s, 12.0 * N);
      pass_secs.push_back(since(t_pass));
      break;
    }
    sp = tm.begin(LVN_STAT_RENUMBER, s);
    remap(C.p, nv, rank.p, s);                  // renumber_communities (louvain_compact.cpp:382)
    keep_level(nv);
    lookup(global.p, N, C.p, nv, err.p, s);     // lookup_dendrogram (louvain_compact.cpp:383)
    tm.end(sp, s, 12.0 * nv + 12.0 * N);
    const auto t1 = Clock::now();
    Nvtx r_agg("aggregation");
    OwnedCsr& next = owned[pass & 1];
    sp = tm.begin(LVN_STAT_AGGREGATE, s);
    if (shard) {
      std::vector<u32> cb;
      aggregate_sharded(cur, C.p, count, v0, v1, cm, next, cb, edges, err.p, s);
      v0 = cb[cm.rank()], v1 = cb[cm.rank() + 1];
    } else {
      self_next.ensure(count ? count : 1);
      kx_next.ensure(count ? count : 1);
      aggregate_device(cur, C.p, count, edges, next, err.p, s, false, &B, inexact.p, self_next.p);
      // exact degrees of this pass's vertices: the previous whole-graph
      // aggregation's, else (pass 0, or after a sharded aggregation) the
      // reset's row sums (sharded runs evaluate Q on the input anyway)
      sum_by_community(C.p, kx_cur.p ? kx_cur.p : K.p, nv, kx_next.p, count, s);
      std::swap(kx_cur, kx_next);
      std::swap(self_cur, self_next);
    }
    tm.end(sp, s, 12.0 * double(cur.arcs) + 16.0 * nv + 8.0 * double(next.arcs) + 8.0 * (count + 1.0),
           nv, cur.arcs);
    if (shard) {
      // the collapse: a graph below shard_min continues on rank 0 alone
      DBuf<u64> ta(1);
      LVN_CUDA(cudaMemcpyAsync(ta.p, &next.arcs, sizeof(u64), cudaMemcpyHostToDevice, s));
      cm.allreduce(ta.p, 1, LVN_U64, LVN_SUM, s);
      if (read_scalar(ta.p, s) < shard_min) {
        gather_graph(next, cm, s);
        sharded = false;
        collapsed = true;
        idle = cm.rank() != 0;
        v0 = 0, v1 = count;
      }
    }
    t_aggregate += since(t1);
    r_agg.end();
    cur = next.view();
    check_graph("aggregated graph", cur, s);
    ++aggregations;
    tolerance /= p.tolerance_drop;
    pass_secs.push_back(since(t_pass));
    // the other ping-pong buffer is free for the pass after this one
    owned[(pass + 1) & 1] = OwnedCsr();
  }
  check_err(err.p, s);

  // sharded runs: rank 0's membership (it ran the passes after the collapse alone)
  if (dist && collapsed) bcast_from0(cm, global.p, 4ull * N, s);
  // final renumber (louvain_compact.cpp:394) and modularity on the input graph (:396)
  size_t sp = tm.begin(LVN_STAT_RENUMBER, s);
  const u32 count = renumber_device(global.p, N, N, used, rank, s, true);
  tm.end(sp, s, 24.0 * N);
  double q = 0.0;
  u64 q_arcs = ig.g.arcs, q_verts = N;  // the graph Q is evaluated on
  sp = tm.begin(LVN_STAT_MODULARITY, s);
  if (input_sharded) {
    if (!have_in_bins) compute_bins(ig.g.off + v0, v1 - v0, edges, in_bins, s, ~u64(0), v0);
    q = modularity_sharded(ig.g, in_bins, global.p, count, m, cm, s);
  } else if (!dist && aggregations > 0 && read_scalar(inexact.p, s) == 0) {
    // Aggregation conserves every community's internal and total weight (the
    // super-vertex self-loop is the internal weight: test_mc.cpp:209-219), so
    // Q of the final partition (quality.cpp:30-41) is evaluated on the last
    // super-graph: its self-loops and vertex degrees in fp64 as the
    // aggregations summed them, its other arcs exact (no narrowing of a
    // non-self entry lost a bit). 25.7 M arcs instead of 3.8 G on C5.
    const u32* memb = C.p;
    if (!ended_in_C) {
      rank.ensure(cur.n ? cur.n : 1);
      iota_u32(rank.p, cur.n, s);
      memb = rank.p;
    }
    DBuf<double> tot(cur.n ? cur.n : 1), sums(2);
    modularity_exact(cur, memb, kx_cur.p, self_cur.p, tot.p, cur.n, sums.p, s, 2.0 * m);
    double* h = reinterpret_cast<double*>(c.pinned);
    LVN_CUDA(cudaMemcpyAsync(h, sums.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
    q = h[0] / (2.0 * m) - h[1];
    q_arcs = cur.arcs, q_verts = cur.n;
  } else if (!idle || !dist) {
    if (!have_in_bins) compute_bins(ig.g.off, N, edges, in_bins, s);
    q = modularity_device(ig.g, in_bins, global.p, count, m, s);
  }
  tm.end(sp, s, 12.0 * double(q_arcs) + 12.0 * q_verts, q_verts, q_arcs);
  if (dist) {
    // every rank reports rank 0's run: Q and the per-pass record
    const int MP = p.max_passes;
    const size_t words = 3 + 4 * size_t(MP);
    std::vector<double> pk(words, 0.0);
    pk[0] = q, pk[1] = passes, pk[2] = aggregations;
    for (int i = 0; i < passes && i < MP; ++i) {
      pk[3 + i] = its[i], pk[3 + MP + i] = tols[i], pk[3 + 2 * MP + i] = vpp[i], pk[3 + 3 * MP + i] = double(app[i]);
    }
    DBuf<double> dpk(words);
    std::memcpy(c.pinned, pk.data(), words * sizeof(double));
    LVN_CUDA(cudaMemcpyAsync(dpk.p, c.pinned, words * sizeof(double), cudaMemcpyHostToDevice, s));
    bcast_from0(cm, dpk.p, words * sizeof(double), s);
    LVN_CUDA(cudaMemcpyAsync(c.pinned, dpk.p, words * sizeof(double), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
    std::memcpy(pk.data(), c.pinned, words * sizeof(double));
    q = pk[0];
    if (cm.rank() != 0) {
      passes = int(pk[1]), aggregations = int(pk[2]);
      its.assign(passes, 0), tols.assign(passes, 0.0), vpp.assign(passes, 0), app.assign(passes, 0);
      pass_secs.resize(passes, 0.0);
      for (int i = 0; i < passes; ++i)
        its[i] = int(pk[3 + i]), tols[i] = pk[3 + MP + i], vpp[i] = u32(pk[3 + 2 * MP + i]),
        app[i] = u64(pk[3 + 3 * MP + i]);
    }
  }

  r->num_vertices = N;
  r->num_communities = count;
  r->modularity = q;
  r->passes = passes;
  r->aggregations = aggregations;
  const size_t k = size_t(passes);
  r->iterations_per_pass = static_cast<int*>(std::calloc(k + 1, sizeof(int)));
  r->tolerance_per_pass = static_cast<double*>(std::calloc(k + 1, sizeof(double)));
  r->pass_seconds = static_cast<double*>(std::calloc(k + 1, sizeof(double)));
  r->vertices_per_pass = static_cast<u32*>(std::calloc(k + 1, sizeof(u32)));
  r->arcs_per_pass = static_cast<u64*>(std::calloc(k + 1, sizeof(u64)));
  for (size_t i = 0; i < k; ++i) {
    r->iterations_per_pass[i] = its[i];
    r->tolerance_per_pass[i] = tols[i];
    r->pass_seconds[i] = i < pass_secs.size() ? pass_secs[i] : 0.0;
    r->vertices_per_pass[i] = vpp[i];
    r->arcs_per_pass[i] = app[i];
  }
  const auto t_d2h = Clock::now();
  if (p.membership_on_device) {
    r->membership = global.p;  // ownership moves to the result (released by lvn_result_free)
    global.p = nullptr;
    global.n = 0;
    r->membership_on_device = 1;
  } else {
    r->membership = static_cast<u32*>(c.host.get(size_t(N ? N : 1) * sizeof(u32)));
    if (N) LVN_CUDA(cudaMemcpyAsync(r->membership, global.p, size_t(N) * sizeof(u32), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
    r->membership_on_device = 0;
  }
  r->d2h_seconds = since(t_d2h);
  tm.collect(r->stats);
  r->wall_seconds = since(t_start);
  if (verbose()) c.pool.report();
  r->num_levels = int(levels.size());
  if (!levels.empty()) {
    r->levels = static_cast<u32**>(std::calloc(levels.size(), sizeof(u32*)));
    for (size_t i = 0; i < levels.size(); ++i) r->levels[i] = levels[i];
    levels.clear();
  }
  cm.settle();
  if (fs.t0) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, fs.t0, fs.t1) == cudaSuccess) r->h2d_seconds = ms * 1e-3;
  }
  r->h2d_bytes = ig.h2d_bytes;
  r->num_shards = cm.size();
  r->sharded_passes = sharded_passes;
  r->exchange_seconds = cm.seconds;
  r->local_moving = t_move;
  r->aggregation = t_aggregate;
  r->other = r->wall_seconds - t_move - t_aggregate;
}

thread_local std::string t_err;
}  // namespace
void set_error(const std::string& what) { t_err = what; }
namespace {

template <class F>
int guard(F&& f) {
  try {
    Context& c = ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    LVN_CUDA(cudaSetDevice(c.device));
    c.pool.refresh_external();  // the stream is idle between calls
    f(c);
    return kOk;
  } catch (const Error& e) {
    t_err = e.what;
    return e.code;
  } catch (const std::bad_alloc&) {
    t_err = "host allocation failed";
    return kOom;
  } catch (const std::exception& e) {
    t_err = e.what();
    return kInternal;
  }
}

struct DGraphHandle {
  OwnedCsr g;
};

}  // namespace
}  // namespace lvn

// holey-row capacity kernel (used by aggregate_device)
namespace lvn {
// capped[c] = min(ext[c] + 1, count): holey row capacity
// capped[c] = min(x[c] + plus_one, count)
__global__ void cap_budgets_k(const u64* __restrict__ x, u64* __restrict__ capped, u32 count, u32 plus_one) {
  for (u64 c = blockIdx.x * u64(blockDim.x) + threadIdx.x; c < count;
       c += u64(gridDim.x) * blockDim.x)
    capped[c] = x[c] + plus_one < count ? x[c] + plus_one : u64(count);
}
void cap_budgets(const u64* x, u64* capped, u32 count, cudaStream_t s, bool plus_one) {
  if (!count) return;
  const u64 blocks = std::min<u64>((u64(count) + 255) / 256, u64(sm_count()) * 8);
  cap_budgets_k<<<unsigned(blocks), 256, 0, s>>>(x, capped, count, plus_one ? 1u : 0u);
  LVN_LAUNCH();
}
}  // namespace lvn

// ===========================================================================
// C-ABI
// ===========================================================================
using namespace lvn;

extern "C" {

const char* lvn_version(void) { return "lvn 0.1 (sm_100a)"; }
const char* lvn_last_error(void) { return t_err.c_str(); }
unsigned long long lvn_launch_count(void) { return g_launches.load(); }

void lvn_params_default(lvn_params* p) {
  if (!p) return;
  std::memset(p, 0, sizeof(*p));
  p->max_passes = 10;
  p->max_iterations = 20;
  p->initial_tolerance = 0.01;
  p->tolerance_drop = 10.0;
  p->aggregation_tolerance = 0.8;
  p->thread_count = 0;
  p->chunk_size = 2048;
  p->prune = 1;
  p->pick_less_period = 4;
  p->switch_move = 64;
  p->switch_aggregate = 128;
  p->probing = LVN_QUADRATIC_DOUBLE;
  p->value_bits = 32;
  p->bin_thread_max = 4;
  p->bin_group_max = 256;
  p->bin_warp_max = 256;
  p->bin_block_max = 4096;
  p->membership_on_device = 0;
  p->sweep_chunk = 0;
  p->sweep_order = 0;
  p->sweep_ranges = 0;
  p->singleton_rule = 0;
  p->shard_min_arcs_log2 = 22;
  p->shard_rounds = 0;
  p->keep_levels = 0;
  p->first_range_arcs_log2 = 27;
}

int lvn_init(int num_gpus, const int* devices) {
  try {
    if (num_gpus < 0) fail(kInvalid, "num_gpus must be >= 0");
    if (num_gpus > 1) fail(kInvalid, "one device per process: shard across ranks (one process per GPU)");
    init_context(num_gpus == 1 && devices ? devices[0] : 0);
    return kOk;
  } catch (const Error& e) {
    t_err = e.what;
    return e.code;
  }
}

int lvn_finalize(void) {
  destroy_context();
  return kOk;
}

void lvn_result_free(lvn_result* r) {
  if (!r) return;
  if (r->membership) {
    if (r->membership_on_device) {
      // through guard(): the context mutex serialises the pool against calls
      // running on other threads (ctypes releases the GIL), on the right device
      (void)guard([&](Context& c) { c.pool.put(r->membership); });
    } else if (!(lvn::g_ctx && lvn::g_ctx->host.put(r->membership))) {
      (void)cudaFreeHost(r->membership);  // pinned block that outlived its context
    }
  }
  std::free(r->iterations_per_pass);
  std::free(r->tolerance_per_pass);
  std::free(r->pass_seconds);
  std::free(r->vertices_per_pass);
  std::free(r->arcs_per_pass);
  for (int i = 0; i < r->num_levels; ++i) std::free(r->levels[i]);
  std::free(r->levels);
  delete r;
}

int lvn_build_csr(uint32_t num_vertices, uint64_t num_triples, const uint32_t* sources, const uint32_t* targets,
                  const double* weights, int symmetrize, lvn_graph_out** out) {
  if (!out) {
    t_err = "null output";
    return kInvalid;
  }
  *out = nullptr;
  lvn_graph_out* res = nullptr;
  const int rc = guard([&](Context& c) {
    if (num_triples && (!sources || !targets || !weights)) fail(kInvalid, "null triple arrays");
    cudaStream_t s = c.stream;
    DBuf<u32> src(num_triples ? num_triples : 1), dst(num_triples ? num_triples : 1);
    DBuf<double> w(num_triples ? num_triples : 1);
    if (num_triples) {
      LVN_CUDA(cudaMemcpyAsync(src.p, sources, num_triples * 4, cudaMemcpyHostToDevice, s));
      LVN_CUDA(cudaMemcpyAsync(dst.p, targets, num_triples * 4, cudaMemcpyHostToDevice, s));
      LVN_CUDA(cudaMemcpyAsync(w.p, weights, num_triples * 8, cudaMemcpyHostToDevice, s));
    }
    OwnedCsr o;
    build_csr_device(num_vertices, num_triples, src.p, dst.p, w.p, symmetrize, o, s);
    res = new lvn_graph_out;
    res->num_vertices = o.n;
    res->num_arcs = o.arcs;
    res->total_weight = o.total_weight;
    res->offsets = static_cast<u64*>(std::malloc((u64(o.n) + 1) * sizeof(u64)));
    res->targets = static_cast<u32*>(std::malloc((o.arcs ? o.arcs : 1) * sizeof(u32)));
    res->weights = static_cast<float*>(std::malloc((o.arcs ? o.arcs : 1) * sizeof(float)));
    if (!res->offsets || !res->targets || !res->weights) fail(kOom, "host allocation failed");
    LVN_CUDA(cudaMemcpyAsync(res->offsets, o.off.p, (u64(o.n) + 1) * sizeof(u64), cudaMemcpyDeviceToHost, s));
    if (o.arcs) {
      LVN_CUDA(cudaMemcpyAsync(res->targets, o.tgt.p, o.arcs * sizeof(u32), cudaMemcpyDeviceToHost, s));
      LVN_CUDA(cudaMemcpyAsync(res->weights, o.w.p, o.arcs * sizeof(float), cudaMemcpyDeviceToHost, s));
    }
    LVN_CUDA(cudaStreamSynchronize(s));
  });
  if (rc) {
    lvn_graph_free(res);
    return rc;
  }
  *out = res;
  return kOk;
}

void lvn_graph_free(lvn_graph_out* g) {
  if (!g) return;
  std::free(g->offsets);
  std::free(g->targets);
  std::free(g->weights);
  delete g;
}

int lvn_louvain_sharded(const lvn_csr* g, const lvn_params* p, const lvn_comm* comm, lvn_result** out) {
  if (!out) {
    t_err = "null output";
    return kInvalid;
  }
  *out = nullptr;
  if (!comm || comm->size < 1 || comm->rank < 0 || comm->rank >= comm->size || comm->size > 1024 ||
      (comm->size > 1 && (!comm->allreduce || !comm->allgatherv))) {
    t_err = "invalid lvn_comm (rank/size out of range or missing collectives)";
    return kInvalid;
  }
  lvn_params def;
  lvn_params_default(&def);
  auto* r = new lvn_result;
  std::memset(r, 0, sizeof(*r));
  lvn::Comm cm;
  cm.c = comm;
  cm.nc = nccl_of(comm);  // the library's NCCL communicator: stream-ordered collectives
  // LVN_SHARD_SINGLE=1 (tests): a one-rank communicator still runs the
  // sharded algorithm, so every collective of the path runs at world size 1
  if (const char* e = std::getenv("LVN_SHARD_SINGLE")) cm.force = e[0] == '1';
  const int rc = guard([&](Context&) { run_louvain(g, p ? *p : def, r, &cm); });
  if (rc) {
    lvn_result_free(r);
    return rc;
  }
  *out = r;
  return kOk;
}

int lvn_partition_rows(const uint64_t* offsets, uint32_t n, int parts, uint32_t* bounds) {
  if (!offsets || !bounds || parts < 1 || parts > 1024) {
    t_err = "invalid arguments to lvn_partition_rows";
    return kInvalid;
  }
  const uint64_t A = offsets[n];
  for (int k = 0; k < parts; ++k) {
    const uint64_t target = lvn::split_target(A, parts, k);
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo) / 2;
      if (offsets[mid] >= target) hi = mid; else lo = mid + 1;
    }
    bounds[k] = lo;
  }
  bounds[parts] = n;
  return kOk;
}

int lvn_louvain(const lvn_csr* g, const lvn_params* p, lvn_result** out) {
  if (!out) {
    t_err = "null output";
    return kInvalid;
  }
  *out = nullptr;
  lvn_params def;
  lvn_params_default(&def);
  auto* r = new lvn_result;
  std::memset(r, 0, sizeof(*r));
  const int rc = guard([&](Context&) {
    Nvtx range("lvn_louvain");
    run_louvain(g, p ? *p : def, r);
  });
  if (rc) {
    lvn_result_free(r);
    return rc;
  }
  *out = r;
  return kOk;
}

int lvn_modularity(const lvn_csr* g, const uint32_t* membership, int membership_location, double* q) {
  return guard([&](Context& c) {
    if (!q) fail(kInvalid, "null output");
    check_csr_header(g);
    if (!(g->total_weight > 0.0))
      fail(kDegenerate, "modularity is undefined when the total edge weight is zero");
    cudaStream_t s = c.stream;
    InGraph ig;
    load_graph(g, s, ig, nullptr);
    DevU32 memb;
    load_u32(membership, ig.g.n, membership_location, s, memb);
    DBuf<u32> mx(1);
    reduce_max_u32(memb.p, ig.g.n, mx.p, s);
    const u64 width = ig.g.n ? u64(read_scalar(mx.p, s)) + 1 : 0;
    lvn_params d;
    lvn_params_default(&d);
    Bins b;
    compute_bins(ig.g.off, ig.g.n, edges_of(d), b, s);
    *q = modularity_device(ig.g, b, memb.p, width, g->total_weight, s);
  });
}

int lvn_vertex_weights(const lvn_csr* g, double* out_host) {
  return guard([&](Context& c) {
    if (!out_host) fail(kInvalid, "null output");
    cudaStream_t s = c.stream;
    InGraph ig;
    load_graph(g, s, ig, nullptr);
    lvn_params d;
    lvn_params_default(&d);
    Bins b;
    compute_bins(ig.g.off, ig.g.n, edges_of(d), b, s);
    DBuf<double> K(ig.g.n ? ig.g.n : 1);
    vertex_weights(ig.g, b, K.p, s);
    if (ig.g.n) LVN_CUDA(cudaMemcpyAsync(out_host, K.p, ig.g.n * sizeof(double), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
  });
}

int lvn_count_communities(const uint32_t* membership, uint64_t n, int location, uint32_t* count) {
  return guard([&](Context& c) {
    if (!count) fail(kInvalid, "null output");
    cudaStream_t s = c.stream;
    if (n == 0) {
      *count = 0;
      return;
    }
    DevU32 m;
    load_u32(membership, n, location, s, m);
    DBuf<u32> mx(1), used, rank;
    reduce_max_u32(m.p, n, mx.p, s);
    const u64 width = u64(read_scalar(mx.p, s)) + 1;
    *count = renumber_device(m.p, n, width, used, rank, s, false);
  });
}

int lvn_renumber(uint32_t* membership, uint64_t n, int location, uint32_t* count) {
  return guard([&](Context& c) {
    cudaStream_t s = c.stream;
    u32 k = 0;
    if (n) {
      DevU32 m;
      load_u32(membership, n, location, s, m);
      DBuf<u32> mx(1), used, rank;
      reduce_max_u32(m.p, n, mx.p, s);
      const u64 width = u64(read_scalar(mx.p, s)) + 1;
      k = renumber_device(m.p, n, width, used, rank, s, true);
      if (location == LVN_HOST)
        LVN_CUDA(cudaMemcpyAsync(membership, m.p, n * sizeof(u32), cudaMemcpyDeviceToHost, s));
      LVN_CUDA(cudaStreamSynchronize(s));
    }
    if (count) *count = k;
  });
}

int lvn_lookup_dendrogram(uint32_t* membership, uint64_t n, const uint32_t* level, uint64_t nl,
                          int location) {
  return guard([&](Context& c) {
    cudaStream_t s = c.stream;
    if (!n) return;
    DevU32 m, l;
    load_u32(membership, n, location, s, m);
    load_u32(level, nl, location, s, l);
    DBuf<u32> err(1);
    LVN_CUDA(cudaMemsetAsync(err.p, 0, sizeof(u32), s));
    lookup(m.p, n, l.p, nl, err.p, s);
    check_err(err.p, s);
    if (location == LVN_HOST)
      LVN_CUDA(cudaMemcpyAsync(membership, m.p, n * sizeof(u32), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
  });
}

int lvn_community_csr(const uint32_t* membership, uint32_t n, uint32_t count, int location,
                      uint64_t* offsets, uint32_t* members) {
  return guard([&](Context& c) {
    if (!offsets || (n && !members)) fail(kInvalid, "null output");
    cudaStream_t s = c.stream;
    DevU32 m;
    load_u32(membership, n, location, s, m);
    if (n) {
      DBuf<u32> mx(1);
      reduce_max_u32(m.p, n, mx.p, s);
      if (read_scalar(mx.p, s) >= count) fail(kInvalid, "membership id out of range");
    }
    DBuf<u32> msize(count ? count : 1), cursor(count ? count : 1), mem(n ? n : 1);
    DBuf<u64> budget(count + 1), coff(count + 1);
    DGraph none;
    none.n = n;
    community_counts(none, m.p, count, msize.p, budget.p, s);
    exclusive_scan_u32_to_u64(msize.p, coff.p, count, s);
    community_scatter(m.p, n, coff.p, count, cursor.p, mem.p, s);
    if (count) {
      DBuf<u32> mx(1);
      reduce_max_u32(msize.p, count, mx.p, s);
      segmented_sort_u32(mem.p, nullptr, coff.p, count, read_scalar(mx.p, s), s);
    }
    LVN_CUDA(cudaMemcpyAsync(offsets, coff.p, (u64(count) + 1) * sizeof(u64), cudaMemcpyDeviceToHost, s));
    if (n) LVN_CUDA(cudaMemcpyAsync(members, mem.p, u64(n) * sizeof(u32), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
  });
}

int lvn_aggregate(const lvn_csr* g, const uint32_t* membership, int membership_location,
                  int canonical, const lvn_params* p, lvn_graph_out** out) {
  if (!out) {
    t_err = "null output";
    return kInvalid;
  }
  *out = nullptr;
  lvn_graph_out* res = nullptr;
  const int rc = guard([&](Context& c) {
    lvn_params def;
    lvn_params_default(&def);
    const lvn_params& pp = p ? *p : def;
    validate(pp);
    cudaStream_t s = c.stream;
    set_probing_aggregate(pp.probing, s);
    InGraph ig;
    load_graph(g, s, ig, nullptr);
    DevU32 m;
    load_u32(membership, ig.g.n, membership_location, s, m);
    // contiguity check (louvain_mc.cpp:106-112): max id + 1 == distinct count
    u32 count = 0;
    if (ig.g.n) {
      DBuf<u32> mx(1), used, rank;
      reduce_max_u32(m.p, ig.g.n, mx.p, s);
      const u64 width = u64(read_scalar(mx.p, s)) + 1;
      count = renumber_device(m.p, ig.g.n, width, used, rank, s, false);
      if (count != width) fail(kInvalid, "membership ids must be contiguous");
    }
    DBuf<u32> err(1);
    LVN_CUDA(cudaMemsetAsync(err.p, 0, sizeof(u32), s));
    // the engine's pass view of the graph: degree bins and the uniform-weight
    // test of the pass reset, so this API takes the aggregation path a pass
    // of the engine would (by external arcs for clustered unit-weight graphs)
    Bins gb;
    compute_bins(ig.g.off, ig.g.n, edges_of(pp), gb, s);
    if (ig.g.arcs && !no_uniform()) {
      DBuf<double> k2(ig.g.n ? ig.g.n : 1);
      DBuf<u32> uni(1);
      pass_reset(ig.g, gb, k2.p, nullptr, nullptr, nullptr, s, uni.p);
      if (read_scalar(uni.p, s) != 0) ig.g.uniform = 1, ig.g.uw = read_scalar(ig.g.w, s);
    }
    OwnedCsr o;
    aggregate_device(ig.g, m.p, count, edges_of(pp), o, err.p, s, canonical != 0, &gb);
    check_err(err.p, s);
    res = new lvn_graph_out;
    res->num_vertices = o.n;
    res->num_arcs = o.arcs;
    res->total_weight = o.total_weight;
    res->offsets = static_cast<u64*>(std::malloc((u64(o.n) + 1) * sizeof(u64)));
    res->targets = static_cast<u32*>(std::malloc((o.arcs ? o.arcs : 1) * sizeof(u32)));
    res->weights = static_cast<float*>(std::malloc((o.arcs ? o.arcs : 1) * sizeof(float)));
    if (!res->offsets || !res->targets || !res->weights) fail(kOom, "host allocation failed");
    LVN_CUDA(cudaMemcpyAsync(res->offsets, o.off.p, (u64(o.n) + 1) * sizeof(u64), cudaMemcpyDeviceToHost, s));
    if (o.arcs) {
      LVN_CUDA(cudaMemcpyAsync(res->targets, o.tgt.p, o.arcs * sizeof(u32), cudaMemcpyDeviceToHost, s));
      LVN_CUDA(cudaMemcpyAsync(res->weights, o.w.p, o.arcs * sizeof(float), cudaMemcpyDeviceToHost, s));
    }
    LVN_CUDA(cudaStreamSynchronize(s));
  });
  if (rc) {
    lvn_graph_free(res);
    return rc;
  }
  *out = res;
  return kOk;
}

namespace lvn {
namespace {
// lvn_evaluate_moves (probe = false) and lvn_probe_moves (probe = true)
int evaluate_moves_impl(const lvn_csr* g, const uint32_t* membership, const double* vertex_w,
                        const double* community_w, double m, const lvn_params* p, int force_kernel,
                        uint32_t* to, double* gain, bool probe) {
  return guard([&](Context& c) {
    lvn_params def;
    lvn_params_default(&def);
    const lvn_params& pp = p ? *p : def;
    validate(pp);
    if (!to || !gain || !vertex_w || !community_w) fail(kInvalid, "null argument");
    if (!(m > 0.0)) fail(kDegenerate, "m must be > 0");
    cudaStream_t s = c.stream;
    set_probing_move(pp.probing, s);
    InGraph ig;
    load_graph(g, s, ig, nullptr);
    const u32 n = ig.g.n;
    DevU32 mb;
    load_u32(membership, n, LVN_HOST, s, mb);
    DBuf<double> K(n ? n : 1), S(n ? n : 1), og(n ? n : 1);
    DBuf<u32> ot(n ? n : 1);
    if (n) {
      LVN_CUDA(cudaMemcpyAsync(K.p, vertex_w, n * sizeof(double), cudaMemcpyHostToDevice, s));
      LVN_CUDA(cudaMemcpyAsync(S.p, community_w, n * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    BinEdges e = edges_of(pp);
    if (force_kernel >= 1) e.thread_max = 0;
    if (force_kernel >= 2) e.group_max = 0;
    if (force_kernel >= 3) e.warp_max = 0;
    if (force_kernel >= 4) e.block_max = 0;
    Bins b;
    compute_bins(ig.g.off, n, e, b, s);
    // isolated vertices stay (louvain_compact.cpp:424)
    if (n) {
      LVN_CUDA(cudaMemcpyAsync(ot.p, mb.p, n * sizeof(u32), cudaMemcpyDeviceToDevice, s));
      LVN_CUDA(cudaMemsetAsync(og.p, 0, n * sizeof(double), s));
    }
    DBuf<IterRecord> rec(1);
    DBuf<u32> err(1);
    LVN_CUDA(cudaMemsetAsync(rec.p, 0, sizeof(IterRecord), s));
    LVN_CUDA(cudaMemsetAsync(err.p, 0, sizeof(u32), s));
    MoveArgs a;
    a.g = ig.g;
    a.C = mb.p;
    a.K = K.p;
    a.sigma = S.p;
    a.m = m;
    a.dry = probe ? 0 : 1;
    a.probe = probe ? 1 : 0;
    a.value_f32 = pp.value_bits == 32 ? 1 : 0;
    a.prune = 0;
    DBuf<u8> flags(n ? n : 1);
    a.flags = flags.p;
    if (probe && n) {
      // uniform-weight detection exactly as the pass reset does it (scratch K,
      // Sigma, C; only the flag is kept)
      DBuf<double> k2(n), s2(n);
      DBuf<u32> c2(n), uni(1);
      pass_reset(ig.g, b, k2.p, s2.p, c2.p, flags.p, s, uni.p);
      if (ig.g.arcs && !no_uniform() && read_scalar(uni.p, s) != 0) {
        a.uniform = 1;
        a.uniform_w = read_scalar(ig.g.w, s);
        a.g.uniform = 1;
        a.g.uw = a.uniform_w;
      }
    }
    a.out_to = ot.p;
    a.out_gain = og.p;
    a.gain_acc = &rec.p->gain;
    a.counters = &rec.p->verts;
    a.err = err.p;
    HubPlan hubs;
    if (b.count(kBinGlobal)) {
      hub_plan_build(ig.g, b.of(kBinGlobal), b.count(kBinGlobal), pp.value_bits, hubs, s);
      hubs.attach(a);
    }
    move_sweep(a, b.view(), pp.value_bits, s);
    if (n) {
      LVN_CUDA(cudaMemcpyAsync(to, ot.p, n * sizeof(u32), cudaMemcpyDeviceToHost, s));
      LVN_CUDA(cudaMemcpyAsync(gain, og.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    LVN_CUDA(cudaStreamSynchronize(s));
  });
}
}  // namespace
}  // namespace lvn

int lvn_evaluate_moves(const lvn_csr* g, const uint32_t* membership, const double* vertex_w,
                       const double* community_w, double m, const lvn_params* p, int force_kernel,
                       uint32_t* to, double* gain) {
  return lvn::evaluate_moves_impl(g, membership, vertex_w, community_w, m, p, force_kernel, to, gain, false);
}

int lvn_probe_moves(const lvn_csr* g, const uint32_t* membership, const double* vertex_w,
                    const double* community_w, double m, const lvn_params* p, int force_kernel,
                    uint32_t* to, double* gain) {
  return lvn::evaluate_moves_impl(g, membership, vertex_w, community_w, m, p, force_kernel, to, gain, true);
}

// ---- device-resident graphs ----------------------------------------------------
struct lvn_dgraph {
  lvn::OwnedCsr g;
};

int lvn_generate(const lvn_gen_params* gp, lvn_dgraph** out) {
  if (!out || !gp) {
    t_err = "null argument";
    return kInvalid;
  }
  *out = nullptr;
  auto* h = new lvn_dgraph;
  const int rc = guard([&](Context& c) {
    GenSpec sp;
    sp.kind = gp->kind;
    sp.n = gp->n;
    sp.edges = gp->edges;
    sp.scale = gp->scale;
    sp.blocks = gp->blocks;
    sp.a = gp->a;
    sp.b = gp->b;
    sp.c = gp->c;
    sp.mu = gp->mu;
    sp.p = gp->p;
    sp.avg_degree = gp->avg_degree;
    sp.seed = gp->seed;
    generate(sp, h->g, c.stream);
  });
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return kOk;
}

int lvn_dgraph_upload(const lvn_csr* host, lvn_dgraph** out) {
  if (!out) {
    t_err = "null output";
    return kInvalid;
  }
  *out = nullptr;
  auto* h = new lvn_dgraph;
  const int rc = guard([&](Context& c) {
    if (!host || host->location != LVN_HOST) fail(kInvalid, "host graph expected");
    InGraph ig;
    load_graph(host, c.stream, ig, nullptr);
    h->g.n = ig.g.n;
    h->g.arcs = ig.g.arcs;
    h->g.off = std::move(ig.off);
    h->g.tgt = std::move(ig.tgt);
    h->g.w = std::move(ig.w);
    h->g.total_weight = host->total_weight;
  });
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return kOk;
}

int lvn_dgraph_view(const lvn_dgraph* g, lvn_csr* view) {
  if (!g || !view) {
    t_err = "null argument";
    return kInvalid;
  }
  view->num_vertices = g->g.n;
  view->num_arcs = g->g.arcs;
  view->offsets = g->g.off.p;
  view->targets = g->g.tgt.p;
  view->weights = g->g.w.p;
  view->total_weight = g->g.total_weight;
  view->location = LVN_DEVICE;
  return kOk;
}

int lvn_dgraph_download(const lvn_dgraph* g, uint64_t* offsets, uint32_t* targets, float* weights) {
  return guard([&](Context& c) {
    if (!g) fail(kInvalid, "null graph");
    cudaStream_t s = c.stream;
    if (offsets)
      LVN_CUDA(cudaMemcpyAsync(offsets, g->g.off.p, (u64(g->g.n) + 1) * sizeof(u64), cudaMemcpyDeviceToHost, s));
    if (targets && g->g.arcs)
      LVN_CUDA(cudaMemcpyAsync(targets, g->g.tgt.p, g->g.arcs * sizeof(u32), cudaMemcpyDeviceToHost, s));
    if (weights && g->g.arcs)
      LVN_CUDA(cudaMemcpyAsync(weights, g->g.w.p, g->g.arcs * sizeof(float), cudaMemcpyDeviceToHost, s));
    LVN_CUDA(cudaStreamSynchronize(s));
  });
}

void lvn_dgraph_free(lvn_dgraph* g) {
  if (!g) return;
  try {
    Context& c = ctx();
    std::lock_guard<std::mutex> lk(c.mu);
    (void)cudaStreamSynchronize(c.stream);
    delete g;
  } catch (...) {
  }
}

int lvn_device_alloc(size_t bytes, void** ptr) {
  return guard([&](Context&) {
    if (!ptr) fail(kInvalid, "null output");
    LVN_CUDA(cudaMalloc(ptr, bytes ? bytes : 1));
  });
}

int lvn_device_free(void* ptr) {
  return guard([&](Context& c) {
    LVN_CUDA(cudaStreamSynchronize(c.stream));
    LVN_CUDA(cudaFree(ptr));
  });
}

int lvn_memcpy(void* dst, const void* src, size_t bytes, int kind) {
  return guard([&](Context& c) {
    const cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice
                             : kind == 2 ? cudaMemcpyDeviceToHost
                                         : cudaMemcpyDeviceToDevice;
    LVN_CUDA(cudaMemcpyAsync(dst, src, bytes, k, c.stream));
    LVN_CUDA(cudaStreamSynchronize(c.stream));
  });
}

}  // extern "C"
