// Cycle cost of one column step of the panel kernel's diagonal factor (warp-level, 32 x 32 block)
// under variants, to locate its latency (measurement tool only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/diag_chain_bench tools/diag_chain_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int PB = 32;

// VAR 0: as in frchol_panel_kernel (sqrt, division, shuffle of l_{k+1}, smem broadcast, bulk update)
// VAR 1: no bulk update (critical chain only)
// VAR 2: division replaced by multiplication with 1/d computed once (rcp)
// VAR 3: sqrt + division replaced by rsqrt + multiply
// VAR 4: VAR 0 without the keep branch (always keep)
template <int VAR>
__global__ void diag(const double *__restrict__ A, double *out, long long *cyc, double tol) {
  __shared__ __align__(16) double lbuf[2][2 * PB];
  __shared__ double Ld[PB * 33];
  const int lane = threadIdx.x;
  double w[PB];
#pragma unroll
  for (int c = 0; c < PB; ++c) w[c] = c <= lane ? A[lane * PB + c] : 0.0;
  lbuf[0][lane] = lbuf[1][lane] = lbuf[0][lane + 32] = lbuf[1][lane + 32] = 0.0;
  __syncwarp();
  int nacc = 0;
  double mn = 1e300;
  long long t0 = clock64();
  for (int m = 0; 4 * m < PB; ++m) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = 4 * m + u;
      const double pv = __shfl_sync(0xffffffffu, w[u], k);
      const bool keep = VAR == 4 ? true : (pv > tol);
      mn = fmin(mn, pv);
      if (keep) {
        double l;
        if (VAR == 3) {
          const double iv = rsqrt(pv);
          l = (lane == k) ? pv * iv : ((lane > k) ? w[u] * iv : 0.0);
        } else if (VAR == 5) {   // Markstein: exact quotient from y = RN(1/d), no lane-dependent division
          const double d = sqrt(pv);
          const double y = 1.0 / d;
          const double q = w[u] * y;
          const double r = fma(-q, d, w[u]);
          const double qq = fma(r, y, q);
          l = (lane == k) ? d : ((lane > k) ? qq : 0.0);
        } else if (VAR == 2) {
          const double d = sqrt(pv);
          const double iv = 1.0 / d;
          l = (lane == k) ? d : ((lane > k) ? w[u] * iv : 0.0);
        } else {
          const double d = sqrt(pv);
          l = (lane == k) ? d : ((lane > k) ? w[u] / d : 0.0);
        }
        const double lk1 = __shfl_sync(0xffffffffu, l, (k + 1) & 31);
        w[u + 1] -= l * lk1;
        double *lb = lbuf[u & 1];
        lb[lane] = l;
        Ld[lane * 33 + nacc] = l;
        __syncwarp();
        if (VAR != 1) {
#pragma unroll
          for (int q = u + 2; q < PB; ++q) w[q] -= l * lb[4 * m + q];
        }
        ++nacc;
      }
    }
#pragma unroll
    for (int q = 0; q < PB - 4; ++q) w[q] = w[q + 4];
#pragma unroll
    for (int q = PB - 4; q < PB; ++q) w[q] = 0.0;
  }
  long long t1 = clock64();
  double s = mn;
  for (int c = 0; c < PB; ++c) s += w[c] + Ld[lane * 33 + c];
  out[lane] = s;
  if (lane == 0) cyc[0] = t1 - t0;
}

template <int VAR>
void run(const double *A, double *o, long long *c, const char *name) {
  diag<VAR><<<1, 32>>>(A, o, c, 1e-9);
  diag<VAR><<<1, 32>>>(A, o, c, 1e-9);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-34s %7lld cycles  %5.1f per column\n", name, h, h / 32.0);
}

int main() {
  // SPD 32 x 32: A = B B' + 32 I with B entries in [-1, 1]
  double hA[PB * PB], B[PB * PB];
  unsigned s = 12345;
  for (int i = 0; i < PB * PB; ++i) {
    s = s * 1664525u + 1013904223u;
    B[i] = ((s >> 8) / 16777216.0) * 2 - 1;
  }
  for (int i = 0; i < PB; ++i)
    for (int j = 0; j < PB; ++j) {
      double v = i == j ? 32.0 : 0.0;
      for (int k = 0; k < PB; ++k) v += B[i * PB + k] * B[j * PB + k];
      hA[i * PB + j] = v;
    }
  double *A, *o;
  long long *c;
  cudaMalloc(&A, sizeof(hA));
  cudaMalloc(&o, 256 * 8);
  cudaMalloc(&c, 8);
  cudaMemcpy(A, hA, sizeof(hA), cudaMemcpyHostToDevice);
  run<0>(A, o, c, "as in the panel kernel");
  run<1>(A, o, c, "critical chain only (no bulk)");
  run<2>(A, o, c, "multiply by 1/d");
  run<3>(A, o, c, "rsqrt + multiply");
  run<4>(A, o, c, "no keep branch");
  run<5>(A, o, c, "Markstein (exact) quotient");
  return 0;
}
