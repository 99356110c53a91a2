// Dependent-chain latency of fp64 / fp32 ops on one thread (cycles per op).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu && ./lat_probe
#include <cstdio>
__global__ void k(double *o, float *of, long long *cyc, double a, double b, float fa, float fb) {
  double x = a; float y = fa;
  long long t0 = clock64();
  for (int i = 0; i < 1024; ++i) x = x + b;
  long long t1 = clock64();
  for (int i = 0; i < 1024; ++i) x = x * b;
  long long t2 = clock64();
  for (int i = 0; i < 1024; ++i) x = fma(x, b, a);
  long long t3 = clock64();
  for (int i = 0; i < 1024; ++i) y = y + fb;
  long long t4 = clock64();
  for (int i = 0; i < 256; ++i) x = a / x;
  long long t5 = clock64();
  o[0] = x; of[0] = y;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}
int main() {
  double *o; float *of; long long *c;
  cudaMallocManaged(&o, 8); cudaMallocManaged(&of, 4); cudaMallocManaged(&c, 40);
  for (int r = 0; r < 2; ++r) { k<<<1, 1>>>(o, of, c, 1.0000001, 1.0000000001, 1.0f, 1e-7f); cudaDeviceSynchronize(); }
  printf("cycles/op: DADD %.1f DMUL %.1f DFMA %.1f FADD %.1f DDIV %.1f\n", c[0] / 1024.0, c[1] / 1024.0,
         c[2] / 1024.0, c[3] / 1024.0, c[4] / 256.0);
}
