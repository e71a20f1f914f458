// Device side of the row-sharded engine (lvn_louvain_sharded).
//
// Storage: rank r keeps only its own rows [v0, v1) of the current graph, as a
// CSR over ALL n vertices whose other rows are empty (offsets n+1 entries,
// targets / weights of the own rows only), so every single-GPU kernel (bins,
// pass reset, sweeps, modularity rows) runs on it unchanged.
//
// Aggregation by own rows (the reference's per-community merge,
// louvain_compact.cpp:214-310, distributed):
//   1. partial_super_edges: every own arc (u, v, w) becomes the entry
//      (C[u] << kb | C[v], w as f64; kb = ceil(log2(count + 1)), so the radix
//      sort covers 2 kb bits, not 64); entries are radix-sorted by key and
//      summed per key in fp64 -> this rank's partial super-edges, sorted.
//   2. the host routes the sorted entries to the owner of their row
//      (community ranges [cb[k], cb[k+1])) with one all-to-all (NCCL).
//   3. merge_super_rows: the owner stably sorts what it received (rank order
//      kept among equal keys), sums each key in fp64 in that order, narrows
//      once to f32 (louvain_mc.cpp:95) and builds its super-rows, every row
//      sorted by target (the canonical layout), as the next pass's local CSR.
// Integer weights therefore give the same super-graph bit for bit as the
// single-GPU aggregation; partial sums never pass through f32.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cuda/std/functional>

#include <cstdlib>

#include "kernels.cuh"
#include "shard.hpp"

namespace lvn {
namespace {

unsigned grid_for(u64 n, int threads, int per_sm) {
  return unsigned(std::max<u64>(1, std::min<u64>((n + threads - 1) / threads, u64(sm_count()) * per_sm)));
}

__global__ void local_offsets_k(const u64* __restrict__ off, u32 n, u32 v0, u32 v1, u64* __restrict__ out) {
  const u64 a0 = off[v0], a1 = off[v1];
  for (u64 u = blockIdx.x * u64(blockDim.x) + threadIdx.x; u <= n; u += u64(gridDim.x) * blockDim.x) {
    const u64 o = off[u];
    out[u] = (o < a0 ? a0 : o > a1 ? a1 : o) - a0;
  }
}

__global__ void entries_k(DGraph g, const u32* __restrict__ C, u32 v0, u32 v1, u32 kb, u64 e0, u64 e1,
                          ull* __restrict__ keys, double* __restrict__ vals) {
  // one thread per own arc of [e0, e1) (own-arc index); its row by a binary
  // search over the own offsets
  const u64 base = g.off[v0];
  for (u64 a = e0 + blockIdx.x * u64(blockDim.x) + threadIdx.x; a < e1; a += u64(gridDim.x) * blockDim.x) {
    u32 lo = v0, hi = v1;  // last row u with off[u] <= base + a
    while (hi - lo > 1) {
      const u32 mid = lo + (hi - lo) / 2;
      if (g.off[mid] <= base + a) lo = mid; else hi = mid;
    }
    keys[a - e0] = (ull(C[lo]) << kb) | C[g.tgt[base + a]];
    vals[a - e0] = double(arc_w(g, base + a));
  }
}

// first index of a sorted key array whose row (key >> 32) reaches each bound
__global__ void route_k(const ull* __restrict__ keys, u64 n, const u32* __restrict__ cb, int parts, u32 kb,
                        u64* __restrict__ cut) {
  for (int k = threadIdx.x; k <= parts; k += blockDim.x) {
    const ull target = ull(cb[k]) << kb;
    u64 lo = 0, hi = n;
    while (lo < hi) {
      const u64 mid = lo + (hi - lo) / 2;
      if (keys[mid] >= target) hi = mid; else lo = mid + 1;
    }
    cut[k] = k == parts ? n : lo;
  }
}

__global__ void row_counts_k(const ull* __restrict__ keys, u64 n, u32 kb, u32* __restrict__ cnt) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
    atomicAdd(&cnt[u32(keys[i] >> kb)], 1u);
}

__global__ void emit_k(const ull* __restrict__ keys, const double* __restrict__ vals, u64 n, u32 kb,
                       u32* __restrict__ tgt, float* __restrict__ w, double* __restrict__ tw) {
  double acc = 0.0;
  const ull mask = (ull(1) << kb) - 1;
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x) {
    tgt[i] = u32(keys[i] & mask);
    const float f = float(vals[i]);
    w[i] = f;
    acc += double(f);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0 && acc != 0.0) atomicAdd(tw, acc);
}

// sort (keys, vals) by key (stable) and sum equal keys in fp64 in that order;
// returns the number of distinct keys, left at the front of keys / vals
u64 sort_reduce(DBuf<ull>& keys, DBuf<double>& vals, u64 n, int bits, cudaStream_t s) {
  if (!n) return 0;
  DBuf<ull> k2(n);
  DBuf<double> v2(n);
  size_t bytes = 0;
  LVN_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, k2.p, vals.p, v2.p, n, 0, bits, s));
  size_t rbytes = 0;
  DBuf<u64> nout(1);
  LVN_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, rbytes, k2.p, keys.p, v2.p, vals.p, nout.p, cuda::std::plus<>{},
                                          n, s));
  DBuf<unsigned char> tmp(std::max(bytes, rbytes));
  LVN_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys.p, k2.p, vals.p, v2.p, n, 0, bits, s));
  LVN_CUDA(cub::DeviceReduce::ReduceByKey(tmp.p, rbytes, k2.p, keys.p, v2.p, vals.p, nout.p, cuda::std::plus<>{}, n,
                                          s));
  g_launches += 4;
  LVN_CUDA(cudaMemcpyAsync(ctx().pinned, nout.p, sizeof(u64), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  return ctx().pinned[0];
}

}  // namespace

void shard_offsets(const u64* off, u32 n, u32 v0, u32 v1, u64* out, cudaStream_t s) {
  local_offsets_k<<<grid_for(u64(n) + 1, 256, 8), 256, 0, s>>>(off, n, v0, v1, out);
  LVN_LAUNCH();
}

u32 key_bits(u32 count) { return std::max(1u, ceil_log2_u64(u64(count) + 1)); }

// Own arcs in slices of at most kSlice entries: each slice sorted and reduced
// on its own, the reduced slices appended and reduced once more, so the sort
// buffers scale with a slice, not with the rank's arcs (C5 on 2 ranks: 1.9 G
// arcs -> 8.6 GB of slice buffers instead of 61 GB)
u64 slice_arcs() {  // LVN_SHARD_SLICE_LOG2 (tests: exercise the multi-slice merge on small graphs)
  static const u64 v = [] {
    const char* e = std::getenv("LVN_SHARD_SLICE_LOG2");
    const int l = e ? std::atoi(e) : 28;
    return u64(1) << (l >= 4 && l <= 40 ? l : 28);
  }();
  return v;
}

u64 partial_super_edges(const DGraph& g, const u32* C, u32 v0, u32 v1, u32 kb, DBuf<ull>& keys, DBuf<double>& vals,
                        cudaStream_t s) {
  const u64 A = g.arcs;  // own arcs only: the other rows are empty
  const u64 kSlice = slice_arcs();
  if (!A || v1 <= v0) {
    keys.ensure(1);
    vals.ensure(1);
    return 0;
  }
  if (A <= kSlice) {
    keys.ensure(A);
    vals.ensure(A);
    entries_k<<<grid_for(A, 256, 16), 256, 0, s>>>(g, C, v0, v1, kb, 0, A, keys.p, vals.p);
    LVN_LAUNCH();
    return sort_reduce(keys, vals, A, int(2 * kb), s);
  }
  DBuf<ull> acc_k;
  DBuf<double> acc_v;
  u64 n = 0;
  DBuf<ull> sk(kSlice);
  DBuf<double> sv(kSlice);
  for (u64 e0 = 0; e0 < A; e0 += kSlice) {
    const u64 e1 = std::min(A, e0 + kSlice);
    entries_k<<<grid_for(e1 - e0, 256, 16), 256, 0, s>>>(g, C, v0, v1, kb, e0, e1, sk.p, sv.p);
    LVN_LAUNCH();
    const u64 m = sort_reduce(sk, sv, e1 - e0, int(2 * kb), s);
    if (n + m > acc_k.n) {  // grow the accumulator (keeps what it holds)
      const u64 cap = std::max<u64>(n + m, 2 * acc_k.n);
      DBuf<ull> nk(cap);
      DBuf<double> nv(cap);
      if (n) {
        LVN_CUDA(cudaMemcpyAsync(nk.p, acc_k.p, n * sizeof(ull), cudaMemcpyDeviceToDevice, s));
        LVN_CUDA(cudaMemcpyAsync(nv.p, acc_v.p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      }
      acc_k = std::move(nk);
      acc_v = std::move(nv);
    }
    LVN_CUDA(cudaMemcpyAsync(acc_k.p + n, sk.p, m * sizeof(ull), cudaMemcpyDeviceToDevice, s));
    LVN_CUDA(cudaMemcpyAsync(acc_v.p + n, sv.p, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
    n += m;
  }
  sk.release();
  sv.release();
  const u64 m = sort_reduce(acc_k, acc_v, n, int(2 * kb), s);
  keys = std::move(acc_k);
  vals = std::move(acc_v);
  return m;
}

void super_row_counts(const ull* keys, u64 n, u32 count, u32 kb, u32* cnt, cudaStream_t s) {
  LVN_CUDA(cudaMemsetAsync(cnt, 0, size_t(count ? count : 1) * sizeof(u32), s));
  if (!n) return;
  row_counts_k<<<grid_for(n, 256, 16), 256, 0, s>>>(keys, n, kb, cnt);
  LVN_LAUNCH();
}

void route_entries(const ull* keys, u64 n, const u32* cb, int parts, u32 kb, u64* cut, cudaStream_t s) {
  route_k<<<1, 256, 0, s>>>(keys, n, cb, parts, kb, cut);
  LVN_LAUNCH();
}

void merge_super_rows(DBuf<ull>& keys, DBuf<double>& vals, u64 n, u32 count, u32 kb, OwnedCsr& out, double* tw,
                      cudaStream_t s) {
  const u64 m = sort_reduce(keys, vals, n, int(2 * kb), s);
  out.n = count;
  out.arcs = m;
  out.off.alloc(u64(count) + 1);
  DBuf<u32> cnt(count ? count : 1);
  super_row_counts(keys.p, m, count, kb, cnt.p, s);
  exclusive_scan_u32_to_u64(cnt.p, out.off.p, count, s);
  out.tgt.alloc(m ? m : 1);
  out.w.alloc(m ? m : 1);
  LVN_CUDA(cudaMemsetAsync(tw, 0, sizeof(double), s));
  if (m) {
    emit_k<<<grid_for(m, 256, 16), 256, 0, s>>>(keys.p, vals.p, m, kb, out.tgt.p, out.w.p, tw);
    LVN_LAUNCH();
  }
}

__global__ void row_lengths_k(const u64* __restrict__ off, u32 n, u32* __restrict__ len) {
  for (u64 u = blockIdx.x * u64(blockDim.x) + threadIdx.x; u < n; u += u64(gridDim.x) * blockDim.x)
    len[u] = u32(off[u + 1] - off[u]);
}

void row_lengths(const u64* off, u32 n, u32* len, cudaStream_t s) {
  if (!n) return;
  row_lengths_k<<<grid_for(n, 256, 8), 256, 0, s>>>(off, n, len);
  LVN_LAUNCH();
}

__global__ void holey_entries_k(const u64* __restrict__ hoff, const u32* __restrict__ htgt,
                                const double* __restrict__ hw64, const u32* __restrict__ fill,
                                const u64* __restrict__ eoff, u32 count, u32 kb, ull* __restrict__ keys,
                                double* __restrict__ vals) {
  const u32 lane = threadIdx.x & 31;
  const u64 warps = u64(gridDim.x) * (blockDim.x >> 5);
  for (u64 c = (blockIdx.x * u64(blockDim.x) + threadIdx.x) >> 5; c < count; c += warps) {
    const u64 src = hoff[c], dst = eoff[c];
    for (u32 j = lane; j < fill[c]; j += 32) {
      keys[dst + j] = (ull(c) << kb) | htgt[src + j];
      vals[dst + j] = hw64[src + j];
    }
  }
}

u64 holey_entries(const u64* hoff, const u32* htgt, const double* hw64, const u32* fill, u32 count, u32 kb,
                  DBuf<ull>& keys, DBuf<double>& vals, cudaStream_t s) {
  DBuf<u64> eoff(u64(count) + 1);
  exclusive_scan_u32_to_u64(fill, eoff.p, count, s);
  u64 n = 0;
  LVN_CUDA(cudaMemcpyAsync(&n, eoff.p + count, sizeof(u64), cudaMemcpyDeviceToHost, s));
  LVN_CUDA(cudaStreamSynchronize(s));
  keys.ensure(n ? n : 1);
  vals.ensure(n ? n : 1);
  if (count) {
    holey_entries_k<<<grid_for(u64(count) * 32, 256, 8), 256, 0, s>>>(hoff, htgt, hw64, fill, eoff.p, count, kb,
                                                                       keys.p, vals.p);
    LVN_LAUNCH();
  }
  return n;
}

__global__ void zero_outside_k(u8* __restrict__ f, u32 n, u32 v0, u32 v1) {
  for (u64 u = blockIdx.x * u64(blockDim.x) + threadIdx.x; u < n; u += u64(gridDim.x) * blockDim.x)
    if (u < v0 || u >= v1) f[u] = 0;
}

void zero_outside(u8* flags, u32 n, u32 v0, u32 v1, cudaStream_t s) {
  if (!n) return;
  zero_outside_k<<<grid_for(n, 256, 8), 256, 0, s>>>(flags, n, v0, v1);
  LVN_LAUNCH();
}

}  // namespace lvn
