// Cycle cost per column of the panel kernel's diagonal factor as it is now (predicated accept /
// drop, branch-free rsqrt-based sqrt and Markstein quotient, next pivot shuffled before the bulk
// update) and variants (measurement tool only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/diag_chain_bench2 tools/diag_chain_bench2.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int PB = 32, LDT = 2 * PB + 2, LDW = PB + 1;

__device__ __forceinline__ void rsqrt_sqrt(double x, double &y, double &d) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
  const double e = fma(-x, y0 * y0, 1.0);
  y = fma(y0 * e, fma(0.375, e, 0.5), y0);
  const double g = x * y;
  d = fma(fma(-g, g, x), 0.5 * y, g);
}
__device__ __forceinline__ double mdiv(double a, double b, double y) {
  const double q = a * y;
  const double r = fma(-q, b, a);
  return fma(r, y, q);
}

// VAR 0: as in the kernel.  1: no bulk update (chain + stores only).  2: no smem stores (Ld, TT,
// pos ..) besides lbuf.  3: the window shift replaced by an unrolled full loop over 32 columns
template <int VAR>
__global__ void diag(const double *__restrict__ A, double *out, long long *cyc, double tol) {
  __shared__ __align__(16) double lbuf[2][2 * PB];
  __shared__ double Ld[PB * LDW];
  __shared__ __align__(16) double TT[PB * LDT];
  __shared__ double ddiag[PB], rdiag[PB];
  __shared__ int pos[PB], kidx[PB];
  const int lane = threadIdx.x;
  const int bw = PB, mode = 0;
  double w[PB];
#pragma unroll
  for (int c = 0; c < PB; ++c) w[c] = c <= lane ? A[lane * PB + c] : 0.0;
  lbuf[0][lane] = lbuf[1][lane] = lbuf[0][lane + 32] = lbuf[1][lane + 32] = 0.0;
  __syncwarp();
  int nacc = 0;
  double mn_acc = 1e300, mx_drop = 0.0, mn_piv = 1e300;
  double pn = __shfl_sync(0xffffffffu, w[0], 0);
  double dreg = 0.0, yreg = 0.0;
  int preg = 0, kreg = -1;
  long long t0 = clock64();
  for (int m = 0; 4 * m < bw; ++m) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int k = 4 * m + u;
      const bool live = k < bw;
      const double pv = pn;
      const bool keep = live && (mode == 0 ? (pv > tol) : (pv > 0.0));
      if (live) mn_piv = fmin(mn_piv, pv);
      double y, d;
      rsqrt_sqrt(pv, y, d);
      const double lq = mdiv(w[u], d, y);
      const double l = !keep ? 0.0 : (lane == k) ? d : ((lane > k && lane < bw) ? lq : 0.0);
      pn = __shfl_sync(0xffffffffu, fma(-l, l, w[u + 1]), (k + 1) & 31);
      const double lk1 = __shfl_sync(0xffffffffu, l, (k + 1) & 31);
      w[u + 1] = fma(-l, lk1, w[u + 1]);
      double *lb = lbuf[u & 1];
      lb[lane] = l;
      if (VAR < 2) {
        Ld[lane * LDW + nacc] = l;
        TT[nacc * LDT + lane] = l;
        if (lane == 0) {
          pos[nacc] = k;
          ddiag[nacc] = d;
          rdiag[nacc] = y;
          if (keep) kidx[k] = nacc;
        }
      }
      __syncwarp();
      if (VAR != 1) {
#pragma unroll
        for (int q = u + 2; q < PB; ++q) w[q] = fma(-l, lb[4 * m + q], w[q]);
      }
      if (VAR == 4) {
        Ld[lane * LDW + nacc] = l;
        TT[nacc * LDT + lane] = l;
      }
      if (VAR == 5) {
        if (lane == 0) {
          pos[nacc] = k;
          ddiag[nacc] = d;
          rdiag[nacc] = y;
          if (keep) kidx[k] = nacc;
        }
      }
      if (VAR == 6) {   // every lane stores the same (warp-uniform) values: no divergent branch
        Ld[lane * LDW + nacc] = l;
        TT[nacc * LDT + lane] = l;
        pos[nacc] = k;
        ddiag[nacc] = d;
        rdiag[nacc] = y;
        kidx[k] = keep ? nacc : -1;
      }
      if (VAR == 8) {   // as 6 without Ld (the L output can come from TT)
        TT[nacc * LDT + lane] = l;
        pos[nacc] = k;
        ddiag[nacc] = d;
        rdiag[nacc] = y;
        kidx[k] = keep ? nacc : -1;
      }
      if (VAR == 7) {   // Ld, TT per column; d, y, pos, kidx held by the lane of their index, stored per group
        Ld[lane * LDW + nacc] = l;
        TT[nacc * LDT + lane] = l;
        if (keep && lane == nacc) { dreg = d; yreg = y; preg = k; }
        if (lane == k) kreg = keep ? nacc : -1;
      }
      if (VAR == 3) {
        Ld[lane * LDW + nacc] = l;
        TT[nacc * LDT + lane] = l;
        if (lane == 0) {
          pos[nacc] = k;
          ddiag[nacc] = d;
          rdiag[nacc] = y;
          if (keep) kidx[k] = nacc;
        }
      }
      if (keep) mn_acc = fmin(mn_acc, pv);
      else if (live) mx_drop = fmax(mx_drop, fabs(pv));
      nacc += keep ? 1 : 0;
    }
    if (VAR == 7) {
      if (lane < nacc) { ddiag[lane] = dreg; rdiag[lane] = yreg; pos[lane] = preg; }
      if ((lane >> 2) == m) kidx[lane] = kreg;
    }
#pragma unroll
    for (int q = 0; q < PB - 4; ++q) w[q] = w[q + 4];
#pragma unroll
    for (int q = PB - 4; q < PB; ++q) w[q] = 0.0;
  }
  long long t1 = clock64();
  double s = mn_acc + mx_drop + mn_piv + nacc;
  for (int c = 0; c < PB; ++c) s += w[c] + Ld[lane * LDW + c] + TT[c * LDT + lane];
  s += ddiag[lane % 32] + rdiag[lane % 32] + pos[lane] + kidx[lane];
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
  run<0>(A, o, c, "as in the kernel");
  run<1>(A, o, c, "no bulk update");
  run<2>(A, o, c, "no metadata stores");
  run<3>(A, o, c, "metadata stores after the bulk update");
  run<4>(A, o, c, "after: Ld, TT only");
  run<5>(A, o, c, "after: lane-0 block only");
  run<6>(A, o, c, "after: all lanes store the uniform values");
  run<7>(A, o, c, "Ld, TT; the rest in registers, per group");
  run<8>(A, o, c, "TT + uniform metadata (no Ld)");
  return 0;
}
