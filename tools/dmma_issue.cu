// DMMA.8x8x4 issue rate vs warps per SM partition, register-resident (measurement tool only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_issue tools/dmma_issue.cu
// One CTA on one SM; `acc` independent accumulators per warp; prints cycles per DMMA per warp and
// the SM's DMMA rate (DMMAs per cycle; the FP64 peak is 0.25 / cycle / SM = 128 flop/clk).
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void k(double *out, long long *cyc, int iters) {
  double c[ACC][2];
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = threadIdx.x * 1e-3;
  double a = 1.0 + threadIdx.x * 1e-6, b = 1.0 - threadIdx.x * 1e-6;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int ACC>
void run(int threads) {
  double *o;
  long long *c, h;
  cudaMalloc(&o, 4096 * 8);
  cudaMalloc(&c, 8);
  const int iters = 2000;
  k<ACC><<<1, threads>>>(o, c, 100);
  k<ACC><<<1, threads>>>(o, c, iters);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double per_warp = (double)h / (iters * ACC);
  printf("warps %2d (per SMSP %d) acc %2d: %.1f cycles per DMMA per warp, SM rate %.3f DMMA/clk\n", threads / 32,
         threads / 128 > 0 ? threads / 128 : 1, ACC, per_warp, (threads / 32) / per_warp);
  cudaFree(o);
  cudaFree(c);
}

int main() {
  for (int th : {32, 128, 256, 512}) {
    run<1>(th);
    run<2>(th);
    run<4>(th);
    run<8>(th);
    run<16>(th);
  }
  return 0;
}
