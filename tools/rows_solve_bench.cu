// Cycle cost of the panel kernel's row solve (rows below the diagonal block: each thread forward-
// substitutes its row against the 32 kept columns T) under variants (measurement tool only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/rows_solve_bench tools/rows_solve_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int PB = 32, LDT = 2 * PB + 2, LDS32 = 36;

__device__ __forceinline__ double mdiv(double a, double b, double y) {
  const double q = a * y;
  const double r = fma(-q, b, a);
  return fma(r, y, q);
}

// VAR 0: as in frchol_panel_kernel (thread = row, window of 4 columns shifted every 4 steps)
// VAR 1: two threads per row (lanes l and l+16 of a warp), each updating half of the columns;
//        the quotient is computed by both (redundant), no communication needed
template <int VAR>
__global__ void solve(const double *__restrict__ Tg, const double *__restrict__ Wg, double *out, long long *cyc) {
  __shared__ __align__(16) double TT[PB * LDT];
  __shared__ double dd[PB], rd[PB];
  extern __shared__ __align__(16) double Ws[];   // [128][LDS32]
  const int tid = threadIdx.x;
  for (int i = tid; i < PB * LDT; i += blockDim.x) TT[i] = Tg[i];
  for (int i = tid; i < 128 * LDS32; i += blockDim.x) Ws[i] = Wg[i];
  if (tid < PB) { dd[tid] = TT[tid * LDT + tid]; rd[tid] = 1.0 / dd[tid]; }
  __syncthreads();
  const int nacc = PB;
  long long t0 = clock64();
  if (VAR == 0) {
    double *wr = Ws + tid * LDS32;
    double v[PB];
#pragma unroll
    for (int j = 0; j < PB; ++j) v[j] = wr[j];
    for (int m = 0; 4 * m < nacc; ++m) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = 4 * m + u;
        const double *tc = TT + j * LDT + 4 * m;
        const double lj = mdiv(v[u], dd[j], rd[j]);
        wr[j] = lj;
#pragma unroll
        for (int q = u + 1; q < PB; ++q) v[q] -= lj * tc[q];
      }
#pragma unroll
      for (int q = 0; q < PB - 4; ++q) v[q] = v[q + 4];
#pragma unroll
      for (int q = PB - 4; q < PB; ++q) v[q] = 0.0;
    }
  } else {
    // 256 threads: row = tid >> 1 ... here 128 threads cover 64 rows x 2 halves
    const int row = (tid >> 5) * 16 + (tid & 15), half = (tid >> 4) & 1;
    double *wr = Ws + row * LDS32;
    double v[PB / 2 + 4];
    // v[q] for q < 16: columns of my half (half 0: 0..15, half 1: 16..31); pivot column j needs v_j:
    // half 0 owns j < 16, half 1 owns j >= 16; the owner shuffles l_j to its partner (lane ^ 16)
#pragma unroll
    for (int q = 0; q < PB / 2; ++q) v[q] = wr[half * 16 + q];
#pragma unroll
    for (int j = 0; j < PB; ++j) {
      const bool own = (j >> 4) == half;
      double lj = 0.0;
      if (own) lj = mdiv(v[j & 15], dd[j], rd[j]);
      lj = __shfl_sync(0xffffffffu, lj, (tid & 31) ^ (own ? 0 : 16));
      if (own) wr[j] = lj;
      const double *tc = TT + j * LDT + half * 16;
#pragma unroll
      for (int q = 0; q < PB / 2; ++q)
        if (half * 16 + q > j) v[q] -= lj * tc[q];
    }
  }
  long long t1 = clock64();
  __syncthreads();
  out[tid] = Ws[tid];
  if (tid == 0) cyc[0] = t1 - t0;
}

template <int VAR>
void run(const double *T, const double *W, double *o, long long *c, const char *name) {
  cudaFuncSetAttribute(solve<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * LDS32 * 8);
  solve<VAR><<<1, 128, 128 * LDS32 * 8>>>(T, W, o, c);
  solve<VAR><<<1, 128, 128 * LDS32 * 8>>>(T, W, o, c);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %7lld cycles  %6.1f per column\n", name, h, h / 32.0);
}

int main() {
  static double hT[PB * LDT], hW[128 * LDS32];
  for (int j = 0; j < PB; ++j)
    for (int i = 0; i < LDT; ++i) hT[j * LDT + i] = (i == j) ? 2.0 + j * 0.01 : (i > j && i < PB ? 0.01 * (i - j) : 0.0);
  for (int i = 0; i < 128 * LDS32; ++i) hW[i] = 1.0 + (i % 7) * 0.1;
  double *T, *W, *o;
  long long *c;
  cudaMalloc(&T, sizeof(hT));
  cudaMalloc(&W, sizeof(hW));
  cudaMalloc(&o, 256 * 8);
  cudaMalloc(&c, 8);
  cudaMemcpy(T, hT, sizeof(hT), cudaMemcpyHostToDevice);
  cudaMemcpy(W, hW, sizeof(hW), cudaMemcpyHostToDevice);
  run<0>(T, W, o, c, "thread per row (panel kernel)");
  run<1>(T, W, o, c, "two threads per row (halves, shuffle)");
  return 0;
}
