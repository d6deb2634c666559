// DFMA dependent-chain latency and chains-per-SMSP needed to saturate the
// FP64 pipe on this GPU (clock64 timing inside one SM).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void chain(double* out, long long* cyc, int iters) {
  double r[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) r[c] = threadIdx.x * 1e-3 + c;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) r[c] = fma(-r[c], r[c], r[c]);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += r[c];
  if (s == -1.0) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64); cudaMalloc(&c, 8 * 1024);
  const int iters = 20000;
  for (int warps : {1, 4, 8, 16, 32}) {
    for (int ch : {1, 2, 4, 8}) {
      long long h = 0;
      switch (ch) {
        case 1: chain<1><<<1, warps * 32>>>(o, c, iters); break;
        case 2: chain<2><<<1, warps * 32>>>(o, c, iters); break;
        case 4: chain<4><<<1, warps * 32>>>(o, c, iters); break;
        case 8: chain<8><<<1, warps * 32>>>(o, c, iters); break;
      }
      cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      double per = double(h) / iters;  // cycles per iteration of the chain loop
      double dfma_per_cycle_sm = double(warps) * ch / per;  // warp-DFMA per cycle per SM
      printf("warps/SM %2d chains %d: %.2f cycles/iter  %.3f warp-DFMA/clk/SM (%.1f%% of 2.0)\n",
             warps, ch, per, dfma_per_cycle_sm, 50.0 * dfma_per_cycle_sm);
    }
  }
  return 0;
}
