// Probe: does a memory-streaming kernel keep its bandwidth while an FP64-FMA
// bound persistent kernel occupies part of every SM?  Variants of the stream
// kernel: pure copy, copy + 7 FP64 ops per element, copy + 7 FP32 ops.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fp32_hog(float* out, int iters) {
  float r0 = threadIdx.x, r1 = r0 + 1;
  const float m = 0.999999f, a = 1e-7f;
  for (int i = 0; i < iters; ++i) { r0 = fmaf(r0, m, a); r1 = fmaf(r1, m, a); }
  if (r0 + r1 == -1.0f) out[0] = r0;
}

__global__ void fp64_hog(double* out, int iters) {
  double r0 = threadIdx.x, r1 = r0 + 1;
  const double m = 0.999999, a = 1e-7;
  for (int i = 0; i < iters; ++i) { r0 = fma(r0, m, a); r1 = fma(r1, m, a); }
  if (r0 + r1 == -1.0) out[0] = r0;
}

template <int MODE>
__global__ void stream_k(const double* __restrict__ a, double* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) {
    double v = a[i];
    if (MODE == 1) { double s = v + 1.0; s = s + v; s = s + 2.0; s = s * 0.5; s = fma(s, 0.25, v); s = s + 3.0; v = s + v; }
    if (MODE == 3) { unsigned q = (unsigned)i; for (int j = 0; j < 8; ++j) q = q * 2654435761u + (unsigned)j; if (q == 7u) v = 1.0; }
    if (MODE == 2) { float s = (float)1.0f; float t = __int_as_float((int)i); s = s + t; s = s * t; s = fmaf(s, t, 1.f); s = s + 2.f; s = s * t; s = s + t; if (s == 12345.f) v = 0; }
    b[i] = v;
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  size_t n = (size_t(1) << 31) / 8;  // 2 GiB
  double *a, *b, *o; cudaMalloc(&a, n * 8); cudaMalloc(&b, n * 8); cudaMalloc(&o, 64);
  cudaMemset(a, 0, n * 8);
  cudaStream_t s0, s1; int lo, hi; cudaDeviceGetStreamPriorityRange(&lo, &hi);
  cudaStreamCreateWithPriority(&s0, cudaStreamNonBlocking, lo);
  cudaStreamCreateWithPriority(&s1, cudaStreamNonBlocking, hi);
  cudaEvent_t e0, e1, f0, f1; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&f0); cudaEventCreate(&f1);
  int hog_kind = 64;
  auto run = [&](int mode, int hog_ctas, const char* name) {
    float best = 1e9, hog = 0;
    for (int r = 0; r < 4; ++r) {
      cudaDeviceSynchronize();
      if (hog_ctas) { cudaEventRecord(f0, s1); if (hog_kind == 64) fp64_hog<<<sms * hog_ctas, 256, 0, s1>>>(o, 400000); else fp32_hog<<<sms * hog_ctas, 256, 0, s1>>>((float*)o, 800000); cudaEventRecord(f1, s1); }
      cudaEventRecord(e0, s0);
      if (mode == 0) stream_k<0><<<sms * 4, 256, 0, s0>>>(a, b, n);
      if (mode == 1) stream_k<1><<<sms * 4, 256, 0, s0>>>(a, b, n);
      if (mode == 2) stream_k<2><<<sms * 4, 256, 0, s0>>>(a, b, n);
      if (mode == 3) stream_k<3><<<sms * 4, 256, 0, s0>>>(a, b, n);
      cudaEventRecord(e1, s0);
      cudaDeviceSynchronize();
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      if (hog_ctas) cudaEventElapsedTime(&hog, f0, f1);
    }
    printf("hog%d %-22s hog_ctas=%d stream %.3f ms = %.0f GB/s   hog %.1f ms\n", hog_kind, name, hog_ctas, best, 2.0 * n * 8 / best / 1e6, hog);
  };
  for (int k : {64, 32}) { hog_kind = k; for (int h : {0, 2, 3}) { run(0, h, "copy"); run(1, h, "copy+7 fp64"); run(2, h, "copy+7 fp32"); run(3, h, "copy+8 imad"); } }
  return 0;
}
