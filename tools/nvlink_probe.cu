// NVLink copy-rate probe for the chunk migration (diagnostic; one process, 2 GPUs).
// Measures SM-driven copies between GPU 0 and GPU 1 with peer access enabled:
//   pull  : each GPU reads the peer's buffer and writes its own (what Runtime::migrate does)
//   push  : each GPU reads its own buffer and writes the peer's
// one direction (GPU 0 only) and both directions at once (both GPUs, the migration case),
// with 1 or 4 16-byte loads in flight per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlink_probe tools/nvlink_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                             \
    }                                                                           \
  } while (0)

template <int U>
__global__ void copy_k(const double2* __restrict__ s, double2* __restrict__ d, long long n2) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(s + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) d[i + u * stride] = v[u];
  }
  for (; i < n2; i += stride) d[i] = __ldcs(s + i);
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    std::printf("{\"error\": \"needs 2 GPUs\"}\n");
    return 0;
  }
  const size_t bytes = size_t(1) << 30;
  const long long n2 = bytes / 16;
  double2 *a[2], *b[2];
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&a[g], bytes));
    CK(cudaMalloc(&b[g], bytes));
    CK(cudaMemset(a[g], 1, bytes));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  const int grid = 2 * 148 * 8, block = 256;
  std::printf("{\"bytes_per_copy\": %zu, \"results\": [\n", bytes);
  bool first = true;
  for (int mode = 0; mode < 2; ++mode)        // 0 pull, 1 push
    for (int both = 0; both < 2; ++both)      // one direction / both at once
      for (int unroll = 1; unroll <= 4; unroll += 3) {
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
          for (int g = 0; g < 2; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaDeviceSynchronize());
          }
          for (int g = 0; g < 1 + both; ++g) {
            CK(cudaSetDevice(g));
            const double2* src = mode == 0 ? a[1 - g] : a[g];
            double2* dst = mode == 0 ? b[g] : b[1 - g];
            CK(cudaEventRecord(e0[g], st[g]));
            if (unroll == 1) copy_k<1><<<grid, block, 0, st[g]>>>(src, dst, n2);
            else copy_k<4><<<grid, block, 0, st[g]>>>(src, dst, n2);
            CK(cudaEventRecord(e1[g], st[g]));
          }
          float worst = 0.f;
          for (int g = 0; g < 1 + both; ++g) {
            CK(cudaSetDevice(g));
            CK(cudaEventSynchronize(e1[g]));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
            if (ms > worst) worst = ms;
          }
          if (rep > 0 && worst < best) best = worst;
        }
        std::printf("%s  {\"mode\": \"%s\", \"directions\": %d, \"loads_in_flight\": %d, "
                    "\"ms\": %.3f, \"GBps_per_gpu\": %.1f}",
                    first ? "" : ",\n", mode == 0 ? "pull" : "push", 1 + both, unroll, best,
                    bytes / (best * 1e-3) / 1e9);
        first = false;
      }
  std::printf("\n]}\n");
  return 0;
}
