// Device CSR construction from an edge list: build_csr (graph.cpp:15-87) as a
// sort-and-reduce on the GPU.
//
//   1. expand: every triple (u, v, w) becomes the arc u->v, plus v->u when
//      symmetrizing and u != v (graph.cpp:23-26); endpoints and weights are
//      validated on the device (out of range, non-finite or negative weights
//      set the error word: std::invalid_argument in the reference);
//   2. order: two stable radix sorts, by weight bits then by (source, target),
//      give every row sorted by (target, weight) -- the order std::sort puts
//      the reference's (target, weight) pairs in (graph.cpp:55);
//   3. merge: one thread per run of equal (source, target) sums the weights
//      sequentially in fp64 in that order and narrows once to f32
//      (graph.cpp:57-63, 80), so the CSR is bit-identical to the reference's
//      for any weights; row lengths are counted per source and scanned.
// total_weight = (fp64 sum of the f32 arc weights) / 2 (graph.cpp:76-84).
#include <cub/device/device_radix_sort.cuh>

#include <cmath>

#include "kernels.cuh"

namespace lvn {
namespace {

constexpr ull kDrop = ~0ull;  // dropped slot (the mirror of a self-loop): sorts last

unsigned grid_of(u64 n) { return unsigned(std::max<u64>(1, std::min<u64>((n + 255) / 256, u64(sm_count()) * 16))); }

__global__ void bc_expand(const u32* __restrict__ src, const u32* __restrict__ dst, const double* __restrict__ w,
                          u64 T, u32 n, int sym, ull* __restrict__ key, ull* __restrict__ wbits, u32* err) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < T; i += u64(gridDim.x) * blockDim.x) {
    const u32 u = src[i], v = dst[i];
    const double x = w[i];
    if (u >= n || v >= n || !isfinite(x) || x < 0.0) atomicOr(err, u32(kErrRange));
    // -0.0 counts as 0.0 for the order (and the sum)
    const ull b = ull(__double_as_longlong(x + 0.0));
    const u64 o = sym ? 2 * i : i;
    key[o] = (ull(u) << 32) | v;
    wbits[o] = b;
    if (sym) {
      key[o + 1] = u != v ? ((ull(v) << 32) | u) : kDrop;
      wbits[o + 1] = b;
    }
  }
}

__global__ void bc_heads(const ull* __restrict__ key, u64 m, u32* __restrict__ head) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < m; i += u64(gridDim.x) * blockDim.x)
    head[i] = key[i] != kDrop && (i == 0 || key[i] != key[i - 1]) ? 1u : 0u;
}

__global__ void bc_starts(const u32* __restrict__ head, const u64* __restrict__ rid, u64 m, u64* __restrict__ start) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < m; i += u64(gridDim.x) * blockDim.x)
    if (head[i]) start[rid[i]] = i;
}

__global__ void bc_merge(const ull* __restrict__ key, const ull* __restrict__ wbits, const u64* __restrict__ start,
                         u64 runs, u64 m, u32* __restrict__ tgt, float* __restrict__ w, u32* __restrict__ deg,
                         double* __restrict__ tw) {
  double acc = 0.0;
  for (u64 r = blockIdx.x * u64(blockDim.x) + threadIdx.x; r < runs; r += u64(gridDim.x) * blockDim.x) {
    const u64 a = start[r];
    const ull k = key[a];
    double s = 0.0;
    for (u64 i = a; i < m && key[i] == k; ++i) s += __longlong_as_double((long long)wbits[i]);
    const float f = float(s);
    tgt[r] = u32(k);
    w[r] = f;
    atomicAdd(&deg[u32(k >> 32)], 1u);
    acc += double(f);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc != 0.0) atomicAdd(tw, acc);
}

template <class K, class V>
void sort_pairs(DBuf<K>& k, DBuf<V>& v, u64 m, int end_bit, cudaStream_t s) {
  DBuf<K> k2(m ? m : 1);
  DBuf<V> v2(m ? m : 1);
  size_t bytes = 0;
  LVN_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k.p, k2.p, v.p, v2.p, m, 0, end_bit, s));
  DBuf<unsigned char> tmp(bytes ? bytes : 1);
  LVN_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, k.p, k2.p, v.p, v2.p, m, 0, end_bit, s));
  std::swap(k.p, k2.p);
  std::swap(v.p, v2.p);
}

}  // namespace

void build_csr_device(u32 n, u64 T, const u32* src, const u32* dst, const double* w, int symmetrize,
                      OwnedCsr& out, cudaStream_t s) {
  if (n == kEmpty) fail(kInvalid, "vertex count collides with the reserved sentinel id");
  const u64 m = symmetrize ? 2 * T : T;
  DBuf<ull> key(m ? m : 1), wb(m ? m : 1);
  DBuf<u32> err(1);
  LVN_CUDA(cudaMemsetAsync(err.p, 0, sizeof(u32), s));
  if (T) {
    bc_expand<<<grid_of(T), 256, 0, s>>>(src, dst, w, T, n, symmetrize, key.p, wb.p, err.p);
    LVN_LAUNCH();
  }
  u32 h_err = 0;
  LVN_CUDA(cudaMemcpyAsync(&h_err, err.p, sizeof(u32), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  if (h_err) fail(kInvalid, "edge endpoint out of range, or an edge weight that is not finite and non-negative");
  // stable LSD order: weight bits (non-negative doubles order like their bits), then (source, target)
  sort_pairs(wb, key, m, 64, s);
  sort_pairs(key, wb, m, 64, s);
  DBuf<u32> head(m ? m : 1);
  DBuf<u64> rid(m + 1);
  if (m) {
    bc_heads<<<grid_of(m), 256, 0, s>>>(key.p, m, head.p);
    LVN_LAUNCH();
  }
  exclusive_scan_u32_to_u64(head.p, rid.p, m, s);
  u64 runs = 0;
  LVN_CUDA(cudaMemcpyAsync(&runs, rid.p + m, sizeof(u64), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  DBuf<u64> start(runs ? runs : 1);
  if (m) {
    bc_starts<<<grid_of(m), 256, 0, s>>>(head.p, rid.p, m, start.p);
    LVN_LAUNCH();
  }
  out.n = n;
  out.arcs = runs;
  out.tgt.alloc(runs ? runs : 1);
  out.w.alloc(runs ? runs : 1);
  out.off.alloc(u64(n) + 1);
  DBuf<u32> deg(n ? n : 1);
  DBuf<double> tw(1);
  LVN_CUDA(cudaMemsetAsync(deg.p, 0, size_t(n ? n : 1) * sizeof(u32), s));
  LVN_CUDA(cudaMemsetAsync(tw.p, 0, sizeof(double), s));
  if (runs) {
    bc_merge<<<grid_of(runs), 256, 0, s>>>(key.p, wb.p, start.p, runs, m, out.tgt.p, out.w.p, deg.p, tw.p);
    LVN_LAUNCH();
  }
  exclusive_scan_u32_to_u64(deg.p, out.off.p, n, s);
  double h_tw = 0.0;
  LVN_CUDA(cudaMemcpyAsync(&h_tw, tw.p, sizeof(double), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  out.total_weight = h_tw / 2.0;
}

}  // namespace lvn
