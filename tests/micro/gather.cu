// Microbenchmark (tuning aid, not product): random 4 B / 8 B gathers from an
// L2-resident array through the different load paths, in G elements/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather gather.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE, class T>
__device__ __forceinline__ T ld(const T* p) {
  T v;
  if (MODE == 0) v = *p;
  if (MODE == 1) v = __ldcg(p);
  if (MODE == 2) v = __ldg(p);
  if (MODE == 3) {
    if (sizeof(T) == 4) asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(*(unsigned*)&v) : "l"(p));
    else asm volatile("ld.global.L1::no_allocate.u64 %0, [%1];" : "=l"(*(unsigned long long*)&v) : "l"(p));
  }
  if (MODE == 4) v = __ldcv(p);
  return v;
}

template <int MODE, class T, int U>
__global__ void k(const T* __restrict__ a, const unsigned* __restrict__ idx, unsigned long long n, T* out) {
  T acc = 0;
  const unsigned long long stride = (unsigned long long)(gridDim.x) * blockDim.x * U;
  for (unsigned long long i = (blockIdx.x * (unsigned long long)(blockDim.x) + threadIdx.x) * U; i < n; i += stride) {
    unsigned j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) j[u] = __ldcs(idx + i + u);
    T v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld<MODE>(a + j[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == T(12345)) out[0] = acc;
}

__global__ void fill_idx(unsigned* idx, unsigned long long n, unsigned range, unsigned seed, int coalesced) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)(blockDim.x) + threadIdx.x; i < n; i += (unsigned long long)(gridDim.x) * blockDim.x) {
    unsigned x = unsigned(i) * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    idx[i] = coalesced ? unsigned(i % range) : x % range;
  }
}

template <int MODE, class T>
float run(const T* a, const unsigned* idx, unsigned long long n, T* out, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  k<MODE, T, 4><<<sms * 8, 256>>>(a, idx, n, out);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<MODE, T, 4><<<sms * 8, 256>>>(a, idx, n, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return 5.0f * n / (ms * 1e6f);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const unsigned long long n = 1ull << 28;
  unsigned* idx;
  cudaMalloc(&idx, n * 4);
  double* out;
  cudaMalloc(&out, 64);
  for (unsigned range : {10000000u, 1000000u, 100000u}) {
    void* a;
    cudaMalloc(&a, size_t(range) * 8);
    cudaMemset(a, 0, size_t(range) * 8);
    fill_idx<<<sms * 8, 256>>>(idx, n, range, 7, 0);
    printf("range %u (u32 %.0f MB): default %.1f  cg %.1f  nc %.1f  no_alloc %.1f  cv %.1f  G/s\n", range, range * 4 / 1e6,
           run<0>((const unsigned*)a, idx, n, (unsigned*)out, sms), run<1>((const unsigned*)a, idx, n, (unsigned*)out, sms),
           run<2>((const unsigned*)a, idx, n, (unsigned*)out, sms), run<3>((const unsigned*)a, idx, n, (unsigned*)out, sms),
           run<4>((const unsigned*)a, idx, n, (unsigned*)out, sms));
    printf("range %u (f64 %.0f MB): default %.1f  cg %.1f  nc %.1f  no_alloc %.1f  G/s\n", range, range * 8 / 1e6,
           run<0>((const double*)a, idx, n, out, sms), run<1>((const double*)a, idx, n, out, sms),
           run<2>((const double*)a, idx, n, out, sms), run<3>((const double*)a, idx, n, out, sms));
    cudaFree(a);
  }
  {
    void* a;
    cudaMalloc(&a, size_t(1) << 30);
    fill_idx<<<sms * 8, 256>>>(idx, n, 1u << 28, 7, 1);
    printf("coalesced u32: default %.1f G/s\n", run<0>((const unsigned*)a, idx, n, (unsigned*)out, sms));
  }
  return 0;
}
