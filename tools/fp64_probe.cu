// fp64_probe.cu -- measures the FP64 pipe on the local GPU (roofline denominator).
// MEASUREMENT TOOL: MEASURED_PEAKS.json carries no FP64 figure, so bench.py
// calls this once per run.  DFMA counts 2 flops, DADD 1.
#include <cuda_runtime.h>
#include <cstdio>

template <int KIND>
__global__ void __launch_bounds__(256) k_probe(double *out, int iters, double b, double c) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-3, a2 = a0 + 2e-3, a3 = a0 + 3e-3;
  double a4 = a0 + 4e-3, a5 = a0 + 5e-3, a6 = a0 + 6e-3, a7 = a0 + 7e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (KIND == 0) {
        a0 = __fma_rn(a0, b, c); a1 = __fma_rn(a1, b, c); a2 = __fma_rn(a2, b, c); a3 = __fma_rn(a3, b, c);
        a4 = __fma_rn(a4, b, c); a5 = __fma_rn(a5, b, c); a6 = __fma_rn(a6, b, c); a7 = __fma_rn(a7, b, c);
      } else {
        a0 = __dadd_rn(a0, c); a1 = __dadd_rn(a1, c); a2 = __dadd_rn(a2, c); a3 = __dadd_rn(a3, c);
        a4 = __dadd_rn(a4, c); a5 = __dadd_rn(a5, c); a6 = __dadd_rn(a6, c); a7 = __dadd_rn(a7, c);
      }
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[blockIdx.x] = s;
}

extern "C" double fp64_probe_flops(int kind, int sms) {
  double *out;
  cudaMalloc(&out, 1 << 20);
  int blocks = sms * 8, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    if (kind == 0) k_probe<0><<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
    else k_probe<1><<<blocks, 256>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  cudaFree(out);
  double ops = (double)blocks * 256 * iters * 4 * 8 * (kind == 0 ? 2.0 : 1.0);
  return ops / (best * 1e-3);
}
