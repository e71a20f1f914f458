// Renumbering, dendrogram lookup and the community -> vertex CSR.
//
//  mark_used + exclusive scan + remap = renumber_communities
//      (louvain_mc.cpp:125-143): used flags, scan -> rank in ascending old-id
//      order, gather. count_communities (quality.cpp:43-56) is the scan total.
//  lookup = lookup_dendrogram (louvain_mc.cpp:145-160), range-checked.
//  community_counts / community_scatter = build_community_csr +
//      community_total_degrees (engine_detail.cpp:44-75).
//  segmented_sort_u32: canonical row order (members ascending, targets
//      ascending) for the bit-exact parity outputs.
//
// Bytes: renumber / lookup / count = 12 B per vertex each.
#include "kernels.cuh"

namespace lvn {
namespace {

__global__ void mark_used_k(const u32* __restrict__ C, u64 n, u32* __restrict__ used) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
    used[C[i]] = 1;
}

__global__ void remap_k(u32* __restrict__ C, u64 n, const u32* __restrict__ rank) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
    C[i] = rank[C[i]];
}

__global__ void lookup_k(u32* __restrict__ g, u64 n, const u32* __restrict__ level, u64 nl,
                         u32* err) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n;
       i += u64(gridDim.x) * blockDim.x) {
    const u32 c = g[i];
    if (c >= nl) {
      atomicOr(err, u32(kErrLookup));
      continue;
    }
    g[i] = level[c];
  }
}

__global__ void counts_k(DGraph g, const u32* __restrict__ C, u32* __restrict__ members,
                         ull* __restrict__ budget) {
  for (u64 v = blockIdx.x * u64(blockDim.x) + threadIdx.x; v < g.n;
       v += u64(gridDim.x) * blockDim.x) {
    const u32 c = C[v];
    // warp-aggregate equal communities: one atomic per distinct id per warp
    const u32 act = __activemask();
    const u32 peers = __match_any_sync(act, c);
    const u64 d = g.off ? g.off[v + 1] - g.off[v] : 0;
    const int leader = __ffs(peers) - 1;
    const int lane = threadIdx.x & 31;
    // sum the peers' degrees (every peer walks the same mask, so the
    // shuffles are converged within the peer group)
    u32 rest = peers;
    u64 total = 0;
    while (rest) {
      const int src = __ffs(rest) - 1;
      total += __shfl_sync(peers, d, src);
      rest &= rest - 1;
    }
    if (lane == leader) {
      atomicAdd(&members[c], u32(__popc(peers)));
      atomicAdd(&budget[c], ull(total));
    }
  }
}

__global__ void scatter_k(const u32* __restrict__ C, u32 n, const u64* __restrict__ coff,
                          u32* __restrict__ cursor, u32* __restrict__ members) {
  for (u64 v = blockIdx.x * u64(blockDim.x) + threadIdx.x; v < n;
       v += u64(gridDim.x) * blockDim.x) {
    const u32 c = C[v];
    const u32 act = __activemask();
    const u32 peers = __match_any_sync(act, c);
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(peers) - 1;
    u32 base = 0;
    if (lane == leader) base = atomicAdd(&cursor[c], u32(__popc(peers)));
    base = __shfl_sync(peers, base, leader);
    const u32 rank = __popc(peers & ((1u << lane) - 1u));
    members[coff[c] + base + rank] = u32(v);
  }
}

__global__ void iota_k(u32* p, u64 n) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
    p[i] = u32(i);
}

__global__ void fill_k(u32* p, u64 n, u32 v) {
  for (u64 i = blockIdx.x * u64(blockDim.x) + threadIdx.x; i < n; i += u64(gridDim.x) * blockDim.x)
    p[i] = v;
}

// ---- segmented sort ----------------------------------------------------------------
constexpr int kSortThreads = 512;
constexpr u32 kSmemSortMax = 4096;

__device__ __forceinline__ void cas_pair(u32& ka, float& va, u32& kb, float& vb, bool up) {
  if ((ka > kb) == up) {
    const u32 tk = ka;
    ka = kb;
    kb = tk;
    const float tv = va;
    va = vb;
    vb = tv;
  }
}

__global__ void __launch_bounds__(kSortThreads) seg_sort_small(u32* keys, float* vals,
                                                               const u64* __restrict__ off,
                                                               u32 nseg) {
  __shared__ u32 sk[kSmemSortMax];
  __shared__ float sv[kSmemSortMax];
  for (u32 sgi = blockIdx.x; sgi < nseg; sgi += gridDim.x) {
    const u64 lo = off[sgi];
    const u32 len = u32(off[sgi + 1] - lo);
    if (len <= 1 || len > kSmemSortMax) continue;
    u32 P = 1;
    while (P < len) P <<= 1;
    for (u32 i = threadIdx.x; i < P; i += kSortThreads) {
      sk[i] = i < len ? keys[lo + i] : kEmpty;
      sv[i] = (vals && i < len) ? vals[lo + i] : 0.0f;
    }
    __syncthreads();
    for (u32 k = 2; k <= P; k <<= 1)
      for (u32 j = k >> 1; j > 0; j >>= 1) {
        for (u32 i = threadIdx.x; i < P; i += kSortThreads) {
          const u32 ixj = i ^ j;
          if (ixj > i) cas_pair(sk[i], sv[i], sk[ixj], sv[ixj], (i & k) == 0);
        }
        __syncthreads();
      }
    for (u32 i = threadIdx.x; i < len; i += kSortThreads) {
      keys[lo + i] = sk[i];
      if (vals) vals[lo + i] = sv[i];
    }
    __syncthreads();
  }
}

// segments longer than the smem tile: bitonic network over a padded global
// scratch copy, one block per segment
__global__ void __launch_bounds__(1024) seg_sort_large(u32* keys, float* vals,
                                                       const u64* __restrict__ off, u32 nseg,
                                                       u32* sk_all, float* sv_all, u64 pmax) {
  u32* sk = sk_all + blockIdx.x * pmax;
  float* sv = sv_all + blockIdx.x * pmax;
  for (u32 sgi = blockIdx.x; sgi < nseg; sgi += gridDim.x) {
    const u64 lo = off[sgi];
    const u64 len = off[sgi + 1] - lo;
    if (len <= kSmemSortMax) continue;
    u64 P = 1;
    while (P < len) P <<= 1;
    for (u64 i = threadIdx.x; i < P; i += blockDim.x) {
      sk[i] = i < len ? keys[lo + i] : kEmpty;
      sv[i] = (vals && i < len) ? vals[lo + i] : 0.0f;
    }
    __syncthreads();
    for (u64 k = 2; k <= P; k <<= 1)
      for (u64 j = k >> 1; j > 0; j >>= 1) {
        for (u64 i = threadIdx.x; i < P; i += blockDim.x) {
          const u64 ixj = i ^ j;
          if (ixj > i) {
            u32 a = sk[i], b = sk[ixj];
            const bool up = (i & k) == 0;
            if ((a > b) == up) {
              sk[i] = b;
              sk[ixj] = a;
              const float t = sv[i];
              sv[i] = sv[ixj];
              sv[ixj] = t;
            }
          }
        }
        __syncthreads();
      }
    for (u64 i = threadIdx.x; i < len; i += blockDim.x) {
      keys[lo + i] = sk[i];
      if (vals) vals[lo + i] = sv[i];
    }
    __syncthreads();
  }
}

unsigned grid_for(u64 n, int threads, int per_sm = 8) {
  const u64 b = (n + threads - 1) / threads;
  return unsigned(std::max<u64>(1, std::min<u64>(b, u64(sm_count()) * per_sm)));
}

}  // namespace

void mark_used(const u32* C, u64 n, u32* used, u64 width, cudaStream_t s) {
  LVN_CUDA(cudaMemsetAsync(used, 0, width * sizeof(u32), s));
  if (!n) return;
  mark_used_k<<<grid_for(n, 256), 256, 0, s>>>(C, n, used);
  LVN_LAUNCH();
}

void remap(u32* C, u64 n, const u32* rank, cudaStream_t s) {
  if (!n) return;
  remap_k<<<grid_for(n, 256), 256, 0, s>>>(C, n, rank);
  LVN_LAUNCH();
}

void lookup(u32* global, u64 n, const u32* level, u64 nl, u32* err, cudaStream_t s) {
  if (!n) return;
  lookup_k<<<grid_for(n, 256), 256, 0, s>>>(global, n, level, nl, err);
  LVN_LAUNCH();
}

void community_counts(const DGraph& g, const u32* C, u32 count, u32* members, u64* budget,
                      cudaStream_t s) {
  LVN_CUDA(cudaMemsetAsync(members, 0, size_t(count) * sizeof(u32), s));
  LVN_CUDA(cudaMemsetAsync(budget, 0, size_t(count) * sizeof(u64), s));
  if (!g.n) return;
  counts_k<<<grid_for(g.n, 256), 256, 0, s>>>(g, C, members, reinterpret_cast<ull*>(budget));
  LVN_LAUNCH();
}

void community_scatter(const u32* C, u32 n, const u64* coff, u32 count, u32* cursor, u32* members,
                       cudaStream_t s) {
  LVN_CUDA(cudaMemsetAsync(cursor, 0, size_t(count) * sizeof(u32), s));
  if (!n) return;
  scatter_k<<<grid_for(n, 256), 256, 0, s>>>(C, n, coff, cursor, members);
  LVN_LAUNCH();
}

void segmented_sort_u32(u32* keys, float* vals, const u64* off, u32 nseg, u64 max_seg,
                        cudaStream_t s) {
  if (!nseg || max_seg <= 1) return;
  seg_sort_small<<<grid_for(nseg, 1, 16), kSortThreads, 0, s>>>(keys, vals, off, nseg);
  LVN_LAUNCH();
  if (max_seg > kSmemSortMax) {
    u64 pmax = 1;
    while (pmax < max_seg) pmax <<= 1;
    const unsigned blocks = unsigned(std::min<u64>(nseg, 16));
    DBuf<u32> sk(pmax * blocks);
    DBuf<float> sv(pmax * blocks);
    seg_sort_large<<<blocks, 1024, 0, s>>>(keys, vals, off, nseg, sk.p, sv.p, pmax);
    LVN_LAUNCH();
    LVN_CUDA(cudaStreamSynchronize(s));  // scratch lifetime
  }
}

void iota_u32(u32* p, u64 n, cudaStream_t s) {
  if (!n) return;
  iota_k<<<grid_for(n, 256), 256, 0, s>>>(p, n);
  LVN_LAUNCH();
}

void fill_u32(u32* p, u64 n, u32 v, cudaStream_t s) {
  if (!n) return;
  fill_k<<<grid_for(n, 256), 256, 0, s>>>(p, n, v);
  LVN_LAUNCH();
}

__global__ void sum_by_community_k(const u32* __restrict__ C, const double* __restrict__ v, u64 n,
                                   double* __restrict__ out) {
  for (u64 u = blockIdx.x * u64(blockDim.x) + threadIdx.x; u < n; u += u64(gridDim.x) * blockDim.x)
    if (v[u] != 0.0) atomicAdd(&out[C[u]], v[u]);
}

void sum_by_community(const u32* C, const double* v, u64 n, double* out, u32 count, cudaStream_t s) {
  LVN_CUDA(cudaMemsetAsync(out, 0, size_t(count ? count : 1) * sizeof(double), s));
  if (!n) return;
  const u64 blocks = std::min<u64>((n + 255) / 256, u64(sm_count()) * 8);
  sum_by_community_k<<<unsigned(blocks), 256, 0, s>>>(C, v, n, out);
  LVN_LAUNCH();
}

}  // namespace lvn
