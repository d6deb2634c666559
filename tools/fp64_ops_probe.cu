// FP64 pipe throughput per instruction kind on one SM (clock64 timing):
// DFMA vs DADD vs DMUL, 16 warps x 8 independent chains (throughput regime).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_ops_probe.cu -o tools/fp64_ops_probe
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void probe(double* out, long long* cyc, int iters) {
  double r[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) r[c] = threadIdx.x * 1e-3 + c * 0.1;
  const double k = 0.999;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (OP == 0) r[c] = __fma_rn(r[c], k, 1e-9);
      else if (OP == 1) r[c] = __dadd_rn(r[c], k);
      else r[c] = __dmul_rn(r[c], k);
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += r[c];
  if (s == -1.0) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64); cudaMalloc(&c, 8 * 1024);
  const int iters = 20000, warps = 16;
  const char* names[3] = {"DFMA", "DADD", "DMUL"};
  for (int op = 0; op < 3; ++op) {
    long long h = 0;
    if (op == 0) probe<0><<<1, warps * 32>>>(o, c, iters);
    if (op == 1) probe<1><<<1, warps * 32>>>(o, c, iters);
    if (op == 2) probe<2><<<1, warps * 32>>>(o, c, iters);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double per_cycle = double(warps) * 8 * iters / double(h);  // warp-instr per clock per SM
    printf("%s: %.3f warp-instr/clk/SM (%.1f thread-ops/clk/SM)\n", names[op], per_cycle,
           per_cycle * 32);
  }
  return 0;
}
