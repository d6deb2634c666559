// Probe: FP64 pipe throughput of the physics recurrence (u = fma(-y,y,y);
// y = fma(k,u,e)) vs a plain fma chain, at the step kernel's occupancy
// (5 CTAs x 128 threads per SM, 2 chains per thread) and at 8 chains per thread.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH, bool LOGISTIC>
__global__ void __launch_bounds__(128) loop_k(double* out, double seed, int iters) {
  double y[CH], e[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) { y[c] = 0.3 + 1e-6 * (threadIdx.x + c); e[c] = 1e-3 * c; }
  const double k = 3.984375, m = 0.999999, a = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (LOGISTIC) {
        const double u = __fma_rn(-y[c], y[c], y[c]);
        y[c] = __fma_rn(k, u, e[c]);
      } else {
        const double u = __fma_rn(y[c], m, a);
        y[c] = __fma_rn(u, m, a);
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += y[c];
  if (s == -1.0) out[threadIdx.x] = s;
}

template <int CH, bool LOG>
double run(int sms, int ctas_per_sm) {
  double* out; cudaMalloc(&out, 1024 * sizeof(double));
  const int iters = 8192 / CH * 2;
  dim3 grid(sms * ctas_per_sm), block(128);
  loop_k<CH, LOG><<<grid, block>>>(out, 1.0, iters);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    loop_k<CH, LOG><<<grid, block>>>(out, 1.0, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  const double flops = 4.0 * CH * (double)iters * grid.x * block.x;  // 2 FMA per iteration
  cudaFree(out);
  return flops / (best * 1e-3) / 1e12;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"plain_2ch_5cta\": %.2f, \"logistic_2ch_5cta\": %.2f, \"plain_8ch_5cta\": %.2f, "
         "\"logistic_8ch_5cta\": %.2f, \"logistic_2ch_4cta\": %.2f, \"logistic_2ch_3cta\": %.2f, "
         "\"logistic_4ch_5cta\": %.2f, \"logistic_4ch_4cta\": %.2f, \"logistic_4ch_3cta\": %.2f, "
         "\"logistic_3ch_4cta\": %.2f, \"logistic_2ch_6cta\": %.2f, \"logistic_2ch_10cta\": %.2f}\n",
         run<2, false>(sms, 5), run<2, true>(sms, 5), run<8, false>(sms, 5), run<8, true>(sms, 5),
         run<2, true>(sms, 4), run<2, true>(sms, 3), run<4, true>(sms, 5), run<4, true>(sms, 4),
         run<4, true>(sms, 3), run<3, true>(sms, 4), run<2, true>(sms, 6), run<2, true>(sms, 10));
  return 0;
}
