// Microbenchmark (tuning aid, not product): per-SM throughput of the warp
// primitives the local-moving kernels are built from on this B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o warp_ops warp_ops.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int OP>
__global__ void k(unsigned* out, unsigned seed) {
  unsigned a = threadIdx.x * 2654435761u + seed, b = a ^ 0x55u, c = a + 7, d = a * 3;
  unsigned long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < ITERS; ++i) {
    if (OP == 0) {  // 4 independent shfl chains
      a = __shfl_xor_sync(0xffffffffu, a, 1) + 1; b = __shfl_xor_sync(0xffffffffu, b, 2) + 1;
      c = __shfl_xor_sync(0xffffffffu, c, 4) + 1; d = __shfl_xor_sync(0xffffffffu, d, 8) + 1;
    } else if (OP == 1) {  // match.any
      a = __match_any_sync(0xffffffffu, a & 7) + a; b = __match_any_sync(0xffffffffu, b & 7) + b;
      c = __match_any_sync(0xffffffffu, c & 7) + c; d = __match_any_sync(0xffffffffu, d & 7) + d;
    } else if (OP == 2) {  // redux.max full mask
      a = __reduce_max_sync(0xffffffffu, a) + a; b = __reduce_max_sync(0xffffffffu, b) + b;
      c = __reduce_max_sync(0xffffffffu, c) + c; d = __reduce_max_sync(0xffffffffu, d) + d;
    } else if (OP == 3) {  // integer min/max/sel ALU baseline
      a = min(a, b) + 1; b = max(b, c) ^ 3; c = min(c, d) + 5; d = max(d, a) ^ 9;
    } else if (OP == 4) {  // ballot
      a += __ballot_sync(0xffffffffu, a & 1); b += __ballot_sync(0xffffffffu, b & 1);
      c += __ballot_sync(0xffffffffu, c & 1); d += __ballot_sync(0xffffffffu, d & 1);
    } else if (OP == 5) {  // dadd
      double x = __int_as_float(a), y = __int_as_float(b);
      x = x * 1.0000001 + y; y = y * 0.999 + x;
      a = __float_as_int(float(x)); b = __float_as_int(float(y));
      c += a; d ^= b;
    }
  }
  unsigned long long t1 = clock64();
  if (a + b + c + d == 0x12345) out[0] = 1;
  if (threadIdx.x == 0) out[1 + blockIdx.x] = unsigned(t1 - t0);
}

template <int OP>
void run(const char* name, int warps_per_block) {
  unsigned* out;
  cudaMalloc(&out, 4 * 4096);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  k<OP><<<sms, warps_per_block * 32>>>(out, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<OP><<<sms, warps_per_block * 32>>>(out, 2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  unsigned cyc;
  cudaMemcpy(&cyc, out + 1, 4, cudaMemcpyDeviceToHost);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double winst = double(warps_per_block) * ITERS * 4;  // warp-ops per SM
  printf("%-10s warps/SM %2d: %.3f warp-ops/clk/SM (%u cycles, %.3f ms)\n", name, warps_per_block,
         winst / cyc, cyc, ms);
  cudaFree(out);
}

int main() {
  for (int w : {8, 32}) {
    run<0>("shfl", w);
    run<1>("match.any", w);
    run<2>("redux.max", w);
    run<3>("imnmx", w);
    run<4>("ballot", w);
    run<5>("dfma", w);
  }
}
