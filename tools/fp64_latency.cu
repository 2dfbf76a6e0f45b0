// Dependent-chain latency (cycles per op) of the FP64 operations on the panel factor's pivot chain
// (measurement tool only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_latency tools/fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 256;

template <int OP>
__global__ void chain(double x0, double *out, long long *cyc) {
  double x = x0 + threadIdx.x * 1e-3;
  const double c = 1.0000001, e = 0.9999999;
  __syncwarp();
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    if (OP == 0) x = fma(x, c, -1e-9);                             // DFMA
    if (OP == 1) x = sqrt(x) + 0.5;                                // sqrt (+ DADD)
    if (OP == 2) x = c / x;                                        // IEEE division
    if (OP == 3) x = 1.0 / x;                                      // IEEE reciprocal
    if (OP == 4) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) * e;  // shfl (+ DMUL)
    if (OP == 5) x = rsqrt(x) + 0.5;                               // rsqrt (+ DADD)
    if (OP == 6) x = __drcp_rn(x);                                 // __drcp_rn
    if (OP == 7) x = x * c;                                        // DMUL
    if (OP == 8) {                                                 // DMMA.8x8x4, accumulator chain
      double c0 = x, c1 = x;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0), "+d"(c1) : "d"(c), "d"(e));
      x = c0;
    }
    if (OP == 9) {                                                 // DMMA, then an LDS of the next operand
      __shared__ double sh[64];
      sh[threadIdx.x] = x;
      __syncwarp();
      double b = sh[(threadIdx.x + 1) & 31];
      double c0 = 0.0, c1 = 0.0;
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0), "+d"(c1) : "d"(c), "d"(b));
      x = c0 * 1e-3 + 1.0;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int OP>
void run(double *o, long long *c, const char *name, double x0 = 2.0) {
  chain<OP><<<1, 32>>>(x0, o, c);
  chain<OP><<<1, 32>>>(x0, o, c);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-22s %6.1f cycles / op\n", name, (double)h / N);
}

int main() {
  double *o;
  long long *c;
  cudaMalloc(&o, 32 * 8);
  cudaMalloc(&c, 8);
  run<0>(o, c, "dfma");
  run<7>(o, c, "dmul");
  run<1>(o, c, "sqrt + dadd");
  run<2>(o, c, "div");
  run<3>(o, c, "1.0 / x");
  run<6>(o, c, "__drcp_rn");
  run<5>(o, c, "rsqrt + dadd");
  run<4>(o, c, "shfl + dmul");
  run<8>(o, c, "dmma (acc chain)");
  run<9>(o, c, "sts+lds+dmma+dfma");
  return 0;
}
