// Microbenchmark: FP64 / FP32 FMA pipe peak and HBM copy bandwidth on the
// local GPU.  Used to fill the FP64/FP32 roofline denominators that
// MEASURED_PEAKS.json does not carry.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CHAINS, int ITERS>
__global__ void fma_loop(T* out, T seed) {
  T r[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) r[c] = seed + T(threadIdx.x + c);
  const T m = T(0.999999), a = T(1e-7);
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) r[c] = fma(r[c], m, a);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += r[c];
  if (s == T(-1)) out[threadIdx.x] = s;  // never true; keeps the loop alive
}

__global__ void copy_k(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}

template <typename T>
double run_fma(int sms) {
  constexpr int CH = 8, IT = 4096;
  T* out; cudaMalloc(&out, 1024 * sizeof(T));
  dim3 grid(sms * 8), block(256);
  fma_loop<T, CH, IT><<<grid, block>>>(out, T(1));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_loop<T, CH, IT><<<grid, block>>>(out, T(1));
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * CH * IT * (double)grid.x * block.x;
  cudaFree(out);
  return flops / (best * 1e-3) / 1e12;
}

// back-to-back launches for ~4 s (power-capped steady state), like the driver's
// sustained bf16 figure
template <typename T>
double run_fma_sustained(int sms, double seconds) {
  constexpr int CH = 8, IT = 4096;
  T* out; cudaMalloc(&out, 1024 * sizeof(T));
  dim3 grid(sms * 8), block(256);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int launches = 0;
  float ms = 0;
  cudaEventRecord(e0);
  while (ms < seconds * 1e3f) {
    for (int i = 0; i < 50; ++i) fma_loop<T, CH, IT><<<grid, block>>>(out, T(1));
    launches += 50;
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double flops = 2.0 * CH * IT * (double)grid.x * block.x * launches;
  cudaFree(out);
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double f64 = run_fma<double>(sms), f32 = run_fma<float>(sms);
  double f64s = run_fma_sustained<double>(sms, 4.0);
  size_t n = (size_t(1) << 31) / sizeof(double4);  // 2 GiB per buffer
  double4 *a, *b; cudaMalloc(&a, n * sizeof(double4)); cudaMalloc(&b, n * sizeof(double4));
  cudaMemset(a, 0, n * sizeof(double4));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(e0);
    copy_k<<<sms * 8, 256>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
  }
  double gbs = 2.0 * n * sizeof(double4) / (best * 1e-3) / 1e9;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"fp64_fma_tflops\": %.2f, \"fp64_fma_tflops_sustained\": %.2f, \"fp32_fma_tflops\": %.2f, \"copy_gbs\": %.1f, \"clock_khz\": %d}\n",
         p.name, sms, f64, f64s, f32, gbs, p.clockRate);
  return 0;
}
