// FP64 peak microbenchmarks for B200 (sm_100a): register-resident DMMA
// (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4) and SIMT DFMA.  Measurement
// tool only; not linked into the product.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int NACC>
__global__ void dmma_loop(double *out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed * 0.5 + threadIdx.x * 1e-4;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double *out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = 1.0 - 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
static double run(K kern, int blocks, int threads, int iters, double flop_per_thread_iter) {
  double *d; CK(cudaMalloc(&d, 8));
  for (int w = 0; w < 3; ++w) kern<<<blocks, threads>>>(d, iters, 1.0);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); kern<<<blocks, threads>>>(d, iters, 1.0); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  cudaFree(d);
  double flops = (double)blocks * threads * iters * flop_per_thread_iter;
  return flops / (best * 1e-3) / 1e12;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int iters = 1 << 16;
  // one DMMA = 8*8*4 FMA = 512 flop per warp -> 16 flop per thread
  for (int wpb : {4, 8, 16}) for (int bps : {1, 2}) {
    double t4 = run(dmma_loop<4>, sms * bps, 32 * wpb, iters / 4, 16.0 * 4);
    double t8 = run(dmma_loop<8>, sms * bps, 32 * wpb, iters / 4, 16.0 * 8);
    printf("{\"kind\":\"dmma\",\"warps_per_block\":%d,\"blocks\":%d,\"tflops_acc4\":%.3f,\"tflops_acc8\":%.3f}\n",
           wpb, sms * bps, t4, t8);
  }
  for (int wpb : {4, 8, 16}) for (int bps : {1, 2}) {
    double t = run(dfma_loop<8>, sms * bps, 32 * wpb, iters / 4, 2.0 * 8);
    printf("{\"kind\":\"dfma\",\"warps_per_block\":%d,\"blocks\":%d,\"tflops\":%.3f}\n", wpb, sms * bps, t);
  }
  return 0;
}
