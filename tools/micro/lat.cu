// Dependent-chain latencies on the B200 (cycles per op): DMUL, DADD, DFMA, DDIV, 64-bit SHFL,
// LDS.64, and the refactor/trisolve step pattern dsub(a, dmul(l, y)).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, double seed, int n) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  double a = seed + threadIdx.x, b = 1.0000001;
  long long t0, t1;
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dmul_rn(a, b);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, 1e-9);
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = __ddiv_rn(a, b);
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_sync(0xffffffffu, a, (i + 1) & 31);
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { a = sm[idx]; idx = ((int)a) & 1023; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / n;
  double l = 0.999;
  t0 = clock64();
  for (int i = 0; i < n; ++i) { const double y = __shfl_sync(0xffffffffu, a, i & 31); a = __dsub_rn(a, __dmul_rn(l, y)); }
  t1 = clock64(); if (threadIdx.x == 0) cyc[6] = (t1 - t0) / n;
  out[threadIdx.x] = a;
}
int main() {
  double *o; long long *c;
  cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64);
  k<<<1, 32>>>(o, c, 1.0, 1000);
  k<<<1, 32>>>(o, c, 1.0, 4096);
  cudaDeviceSynchronize();
  printf("cycles/op (1 warp): dmul %lld dadd %lld dfma %lld ddiv %lld shfl64 %lld lds64-chase %lld step(shfl+dmul+dsub) %lld\n",
         c[0], c[1], c[2], c[3], c[4], c[5], c[6]);
  return 0;
}
