// Device exclusive prefix sums (reduce -> spine -> downsweep), the device
// counterpart of exclusive_scan (prefix_sum.hpp:27-68): out[i] = sum of
// in[0..i), out[n] = total. Integer addition is associative, so the result is
// bit-identical to the sequential scan regardless of tiling.
//
// Bytes: read n inputs twice (reduce + downsweep), write n+1 outputs.
#include "kernels.cuh"

namespace lvn {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;
constexpr int kTile = kThreads * kItems;

__device__ __forceinline__ int pad(int i) { return i + (i >> 5); }

template <class T>
__device__ T block_exclusive(T v, T* total) {
  __shared__ T warp_tot[kThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T t = lane < kThreads / 32 ? warp_tot[lane] : T(0);
    T ti = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, ti, o);
      if (lane >= o) ti += y;
    }
    if (lane < kThreads / 32) warp_tot[lane] = ti - t;  // exclusive warp offsets
    if (lane == kThreads / 32 - 1) *total = ti;
  }
  __syncthreads();
  const T r = warp_tot[wid] + inc - v;
  __syncthreads();
  return r;
}

template <class TIn, class TOut>
__global__ void __launch_bounds__(kThreads) scan_reduce(const TIn* __restrict__ in, u64 n,
                                                        TOut* __restrict__ part) {
  const u64 base = u64(blockIdx.x) * kTile;
  TOut s = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const u64 k = base + u64(i) * kThreads + threadIdx.x;
    if (k < n) s += TOut(in[k]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ TOut ws[kThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    TOut t = 0;
    for (int w = 0; w < kThreads / 32; ++w) t += ws[w];
    part[blockIdx.x] = t;
  }
}

// single block: exclusive scan of the per-tile sums in place, total -> *total
template <class TOut>
__global__ void __launch_bounds__(kThreads) scan_spine(TOut* part, u64 nb, TOut* total) {
  const u64 per = (nb + kThreads - 1) / kThreads;
  const u64 lo = threadIdx.x * per;
  const u64 hi = lo + per < nb ? lo + per : nb;
  TOut s = 0;
  for (u64 i = lo; i < hi; ++i) s += part[i];
  __shared__ TOut tot;
  TOut run = block_exclusive<TOut>(s, &tot);
  for (u64 i = lo; i < hi; ++i) {
    const TOut v = part[i];
    part[i] = run;
    run += v;
  }
  if (threadIdx.x == 0) *total = tot;
}

template <class TIn, class TOut>
__global__ void __launch_bounds__(kThreads) scan_down(const TIn* __restrict__ in, u64 n,
                                                      const TOut* __restrict__ part,
                                                      TOut* __restrict__ out) {
  __shared__ TOut sm[kTile + kTile / 32];
  const u64 base = u64(blockIdx.x) * kTile;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int j = i * kThreads + threadIdx.x;
    const u64 k = base + j;
    sm[pad(j)] = k < n ? TOut(in[k]) : TOut(0);
  }
  __syncthreads();
  TOut v[kItems];
  TOut s = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    v[i] = sm[pad(threadIdx.x * kItems + i)];
    s += v[i];
  }
  __shared__ TOut tot;
  TOut run = block_exclusive<TOut>(s, &tot) + part[blockIdx.x];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    sm[pad(threadIdx.x * kItems + i)] = run;
    run += v[i];
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int j = i * kThreads + threadIdx.x;
    const u64 k = base + j;
    if (k < n) out[k] = sm[pad(j)];
  }
}

template <class TIn, class TOut>
void scan_impl(const TIn* in, TOut* out, u64 n, cudaStream_t s) {
  if (n == 0) {
    LVN_CUDA(cudaMemsetAsync(out, 0, sizeof(TOut), s));
    return;
  }
  const u64 nb = (n + kTile - 1) / kTile;
  DBuf<TOut> part(nb);
  scan_reduce<TIn, TOut><<<unsigned(nb), kThreads, 0, s>>>(in, n, part.p);
  LVN_LAUNCH();
  scan_spine<TOut><<<1, kThreads, 0, s>>>(part.p, nb, out + n);
  LVN_LAUNCH();
  scan_down<TIn, TOut><<<unsigned(nb), kThreads, 0, s>>>(in, n, part.p, out);
  LVN_LAUNCH();
  // `part` returns to the pool; the pool hands memory back out only to later
  // stream-ordered work on the same stream, so reuse is safe.
}

__global__ void max_u32_kernel(const u32* __restrict__ in, u64 n, u32* out) {
  u32 m = 0;
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
    m = max(m, in[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace

void exclusive_scan_u32(const u32* in, u32* out, u64 n, cudaStream_t s) { scan_impl(in, out, n, s); }
void exclusive_scan_u64(const u64* in, u64* out, u64 n, cudaStream_t s) { scan_impl(in, out, n, s); }
void exclusive_scan_u32_to_u64(const u32* in, u64* out, u64 n, cudaStream_t s) {
  scan_impl(in, out, n, s);
}

void reduce_max_u32(const u32* in, u64 n, u32* out, cudaStream_t s) {
  LVN_CUDA(cudaMemsetAsync(out, 0, sizeof(u32), s));
  if (n == 0) return;
  const u64 blocks = std::min<u64>((n + 255) / 256, u64(sm_count()) * 8);
  max_u32_kernel<<<unsigned(blocks), 256, 0, s>>>(in, n, out);
  LVN_LAUNCH();
}

}  // namespace lvn
