// Shared internals of liblvn.so: types, error plumbing, device pool, small
// device helpers. Everything here is B200 (sm_100a) only.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

namespace lvn {

using u8 = std::uint8_t;
using u16 = std::uint16_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;
using ull = unsigned long long;

constexpr u32 kEmpty = 0xFFFFFFFFu;  // empty-slot / invalid id (graph.hpp:15, compact_hashtable.hpp:26)
constexpr ull kEmptySlot64 = 0xFFFFFFFF00000000ull;  // packed (key=kEmpty, value=0.0f)

// status codes of include/lvn.h
enum Status { kOk = 0, kInvalid = 1, kDegenerate = 2, kInternal = 3, kCuda = 4, kOom = 5 };

struct Error {
  int code;
  std::string what;
};

// lvn_last_error() text of this thread (engine.cu)
void set_error(const std::string& what);

[[noreturn]] inline void fail(int code, const std::string& what) { throw Error{code, what}; }

inline void cuda_check(cudaError_t e, const char* expr, const char* file, int line) {
  if (e != cudaSuccess) {
    const int code = (e == cudaErrorMemoryAllocation) ? kOom : kCuda;
    fail(code, std::string(expr) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                   std::to_string(line) + ")");
  }
}
extern std::atomic<unsigned long long> g_launches;  // kernels launched by this library

// LVN_SYNC_DEBUG=1: synchronise after every launch and name the launch site
void launch_check(const char* file, int line);

#define LVN_CUDA(x) ::lvn::cuda_check((x), #x, __FILE__, __LINE__)
#define LVN_LAUNCH() ::lvn::launch_check(__FILE__, __LINE__)

// device error word bits (checked by the host once per pass)
enum DevErr : u32 { kErrTable = 1u, kErrLookup = 2u, kErrRange = 4u };

// ---------------------------------------------------------------------------
// Device view of a CSR graph (graph.hpp:38-54)
// ---------------------------------------------------------------------------
struct DGraph {
  u32 n = 0;
  u64 arcs = 0;
  const u64* off = nullptr;
  const u32* tgt = nullptr;
  const float* w = nullptr;
  // every arc weight is uw (detected by the pass reset): the kernels that
  // only sum weights take uw instead of reading w (4 B per arc less traffic)
  int uniform = 0;
  float uw = 0.f;
};

// ---------------------------------------------------------------------------
// Device memory. Everything is stream-ordered on the engine stream:
// requests below 64 MB come from the device memory pool (cudaMallocAsync /
// cudaFreeAsync, release threshold unlimited); larger ones (graph arrays,
// holey rows, tables) are rounded up to 1/16 of their power of two and kept in
// a best-fit cache of their own, so the multi-GB buffers of consecutive runs
// land on the same blocks instead of fragmenting the pool.
// ---------------------------------------------------------------------------
class Pool {
 public:
  void bind(int device, cudaStream_t s);
  void* get(size_t bytes);
  void put(void* p);
  void trim();         // return cached memory to the driver
  void release_all();  // free every outstanding allocation (context teardown)
  void report();       // pool occupancy on stderr (LVN_VERBOSE)
  // device memory this pool can still hand out: device total minus the
  // memory held outside the pool (as of the last refresh) minus the pool's
  // live allocations, plus its cached big blocks, minus a 1 GB margin
  size_t available();
  // re-measure the memory held outside the pool (CUDA context, caller
  // buffers such as a borrowed device CSR, other processes on the GPU) with
  // cudaMemGetInfo; called at the entry of a run while the stream is idle
  // (mid-run, cudaMemGetInfo stalls the host for tens of ms)
  void refresh_external();
  // Graph capture of a sweep: transient buffers come from a caller-owned
  // arena (no allocation nodes in the captured body; the arena outlives the
  // graph), sized from the bytes the same sweep requested uncaptured
  // (track_begin / track_end).
  void arena_begin(void* base, size_t bytes);
  void arena_end();
  void track_begin();
  size_t track_end();

 private:
  unsigned char* arena_ = nullptr;
  size_t arena_cap_ = 0, arena_used_ = 0;
  bool arena_on_ = false, tracking_ = false;
  size_t tracked_ = 0;
  void* raw(size_t bytes);
  cudaMemPool_t pool_ = nullptr;
  cudaStream_t stream_ = nullptr;
  std::unordered_set<void*> used_;
  std::unordered_map<void*, size_t> big_used_;
  std::multimap<size_t, void*> big_free_;
  size_t cache_budget_ = size_t(16) << 30;  // bytes of free big blocks kept across a miss
  size_t total_ = 0;                        // device memory (at bind)
  size_t external_ = 0;                     // held outside the pool (refresh_external)
};

// Pinned host blocks for results handed to the caller (membership): device
// to host copies run at full link speed and without first-touch page faults
// once a block has been used; lvn_result_free returns the block here.
class HostCache {
 public:
  void* get(size_t bytes);
  bool put(void* p);  // false: not a block of this cache
  ~HostCache();

 private:
  std::mutex mu_;
  std::multimap<size_t, void*> free_;
  std::unordered_map<void*, size_t> used_;
};

// Engine context: one device, one stream, pinned scratch for small readbacks.
struct Context {
  int device = 0;
  int sms = 148;
  size_t smem_optin = 227 * 1024;
  cudaStream_t stream = nullptr;
  cudaStream_t copy = nullptr;  // host -> device input chunks (overlapped with the first sweep)
  // forked streams + events of a captured sweep with concurrent degree bins
  std::vector<cudaStream_t> aux;
  std::vector<cudaEvent_t> aux_ev;
  void ensure_aux(int n);
  Pool pool;
  HostCache host;
  u64* pinned = nullptr;  // 8192 u64 of pinned host scratch
  std::mutex mu;
};

Context& ctx();  // lazily initialised on device 0 (or the lvn_init device)
void init_context(int device);
void destroy_context();

// RAII typed device buffer from the pool
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p, n = o.n;
      o.p = nullptr, o.n = 0;
    }
    return *this;
  }
  void alloc(size_t count) {
    release();
    n = count;
    p = static_cast<T*>(ctx().pool.get((count ? count : 1) * sizeof(T)));
  }
  void ensure(size_t count) {
    if (count > n || !p) alloc(count);
  }
  void release() {
    if (p) ctx().pool.put(p);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  T* get() const { return p; }
};

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------
__host__ __device__ inline u32 ceil_log2_u64(u64 x) {
#ifdef __CUDA_ARCH__
  return x <= 1 ? 0u : 64u - u32(__clzll((long long)(x - 1)));
#else
  return x <= 1 ? 0u : 64u - u32(__builtin_clzll(x - 1));
#endif
}

// L2 eviction priority for the random gathers of a sweep (C[t], Sigma[c]):
// evict_last keeps those arrays resident while the streamed rows (loaded
// evict-first) pass through L2.
__device__ __forceinline__ ull l2_keep_policy(int mode = 1) {
  ull p;
  if (mode == 0) asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  else if (mode == 2) asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  else asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ u32 ld_keep(const u32* a, ull pol) {
  u32 v;
  asm("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_keep(const double* a, ull pol) {
  double v;
  asm("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
  return v;
}

// weight of arc a (streamed: read once per sweep)
__device__ __forceinline__ float arc_w(const DGraph& g, u64 a) { return g.uniform ? g.uw : __ldcs(g.w + a); }

// multiplicative hash into a power-of-two table of 2^log_size slots
__device__ __forceinline__ u32 slot_hash(u32 key, u32 log_size) {
  return log_size ? (key * 0x9E3779B1u) >> (32u - log_size) : 0u;
}

// Eq. 2, evaluated operation for operation like delta_modularity
// (quality.hpp:34-37) with round-to-nearest intrinsics so no FMA contraction
// changes the bits.
__device__ __forceinline__ double delta_q(double k_to_c, double k_to_d, double k_i, double sigma_c,
                                          double sigma_d, double m) {
  const double a = __ddiv_rn(__dsub_rn(k_to_c, k_to_d), m);
  const double num = __dmul_rn(k_i, __dsub_rn(__dadd_rn(k_i, sigma_c), sigma_d));
  const double den = __dmul_rn(__dmul_rn(2.0, m), m);
  return __dsub_rn(a, __ddiv_rn(num, den));
}

// best-candidate order: greater gain, ties to the lowest id (compact_hashtable.hpp:152)
__device__ __forceinline__ bool better(double g, u32 c, double bg, u32 bc) {
  return g > bg || (g == bg && c < bc);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ ull warp_sum(ull v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

int sm_count();

}  // namespace lvn
