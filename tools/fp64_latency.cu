// Latency of dependent FP64 ops for one warp on sm_100a (measurement tool only).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double *out, long long *cyc, double x0, int n) {
  double x = x0 + threadIdx.x * 1e-9, y = 1.000001;
  long long t0, t1;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-12);
  t1 = clock64(); if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / x + 0.5;
  t1 = clock64(); if (threadIdx.x == 0) cyc[1] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + 0.25;
  t1 = clock64(); if (threadIdx.x == 0) cyc[2] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * 1.0000001;
  t1 = clock64(); if (threadIdx.x == 0) cyc[3] = (t1 - t0) / n;
  __shared__ double sm[64];
  sm[threadIdx.x] = x; __syncwarp();
  t0 = clock64();
  int j = threadIdx.x;
  for (int i = 0; i < n; ++i) { double v = sm[j]; j = ((int)v & 1) ^ threadIdx.x; sm[threadIdx.x] = v + 1.0; }
  t1 = clock64(); if (threadIdx.x == 0) cyc[4] = (t1 - t0) / n;
  t0 = clock64();
  for (int i = 0; i < n; ++i) x = x / y + 1e-3;
  t1 = clock64(); if (threadIdx.x == 0) cyc[5] = (t1 - t0) / n;
  out[threadIdx.x] = x + sm[j];
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  lat<<<1, 32>>>(o, c, 1.5, 1000); cudaDeviceSynchronize();
  lat<<<1, 32>>>(o, c, 1.5, 10000); cudaDeviceSynchronize();
  long long h[6]; cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  printf("cycles per dependent op: dfma %lld  rcp-div(1/x) %lld  sqrt %lld  shfl+dmul %lld  lds+sts %lld  div(x/y) %lld\n", h[0], h[1], h[2], h[3], h[4], h[5]);
  return 0;
}
