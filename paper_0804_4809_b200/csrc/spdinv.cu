// a5 (M = inv(L'L)): triangular inverse of the Cholesky factor by
// recursive doubling.  With C = [C11 0; C21 C22] lower triangular,
//   C^-1 = [C11^-1 0; -C22^-1 C21 C11^-1  C22^-1],
// so after inverting the 32 x 32 diagonal blocks, each level h = 32, 64, ...
// combines all pairs of h-blocks with two batched DMMA GEMMs -- O(log r)
// dependent steps (the "O(log r)" remark of P:80 for the SPD inverse).
// The factor is padded to r_pad = round_up(r, 32) with an identity block so
// every block boundary is a multiple of 32 (the padding inverts to identity
// and is never read back).
#include "common.cuh"
#include "gemm_host.h"
#include "kernels.h"

namespace gi {

__global__ void pad_identity_kernel(double *C, long long ldc, int r, int r_pad) {
  const int i = r + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < r_pad) C[(long long)i * ldc + i] = 1.0;
}

// Inverse of each 32 x 32 lower-triangular diagonal block; thread j owns column j.
__global__ void trtri_diag_kernel(const double *__restrict__ C, long long ldc, double *__restrict__ Ci,
                                  long long ldi) {
  __shared__ double c[32][33];
  const int b0 = blockIdx.x * 32;
  const int j = threadIdx.x;
  for (int i = 0; i < 32; ++i) c[i][j] = C[(long long)(b0 + i) * ldc + b0 + j];
  __syncthreads();
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    double v;
    if (i < j) {
      v = 0.0;
    } else {
      double a = (i == j) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k)
        if (k >= j) a -= c[i][k] * x[k];
      v = a / c[i][i];
    }
    x[i] = v;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i >= j) Ci[(long long)(b0 + i) * ldi + b0 + j] = x[i];
}

cudaError_t trtri_lower(double *C, long long ldc, int r, double *Ci, long long ldi, double *T, cudaStream_t st) {
  const int r_pad = (r + 31) / 32 * 32;
  if (r_pad == 0) return cudaSuccess;
  if (r_pad > r) pad_identity_kernel<<<1, 32, 0, st>>>(C, ldc, r, r_pad);
  trtri_diag_kernel<<<r_pad / 32, 32, 0, st>>>(C, ldc, Ci, ldi);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  for (int h = 32; h < r_pad; h *= 2) {
    // pairs p: block1 rows/cols [2ph, 2ph+h), block2 [(2p+1)h, (2p+1)h + h2)
    const int nfull = r_pad / (2 * h);                 // pairs with h2 == h
    const int rem = r_pad - nfull * 2 * h;             // leftover: partial pair if rem > h
    struct Group { int p0, count, h2; };
    Group groups[2];
    int ng = 0;
    if (nfull > 0) groups[ng++] = {0, nfull, h};
    if (rem > h) groups[ng++] = {nfull, 1, rem - h};
    for (int gi_ = 0; gi_ < ng; ++gi_) {
      const Group gr = groups[gi_];
      const long long off1 = (long long)gr.p0 * 2 * h;  // block1 origin (row = col)
      const long long bstr_c = 2LL * h * (ldc + 1), bstr_i = 2LL * h * (ldi + 1);
      // T1 = C21 * Cinv11   (h2 x h), T: batch stride h2*h, ld h
      GemmOp op1;
      op1.A = Mat{C + (off1 + h) * ldc + off1, ldc, gr.h2, h, gr.count, bstr_c};
      op1.a_kmajor = true;
      op1.B = Mat{Ci + off1 * ldi + off1, ldi, h, h, gr.count, bstr_i};
      op1.b_kmajor = false;
      op1.C = T;
      op1.ldc = h;
      op1.c_bstride = (long long)gr.h2 * h;
      op1.M = gr.h2;
      op1.N = h;
      op1.K = h;
      op1.batch = gr.count;
      op1.k_lo_mode = 2;                               // Cinv11 lower: B(k, n) = 0 for k < n
      e = gemm(op1, st);
      if (e != cudaSuccess) return e;
      // Cinv21 = -Cinv22 * T1   (h2 x h)
      GemmOp op2;
      op2.A = Mat{Ci + (off1 + h) * ldi + off1 + h, ldi, gr.h2, gr.h2, gr.count, bstr_i};
      op2.a_kmajor = true;
      op2.B = Mat{T, h, gr.h2, h, gr.count, (long long)gr.h2 * h};
      op2.b_kmajor = false;
      op2.C = Ci + (off1 + h) * ldi + off1;
      op2.ldc = ldi;
      op2.c_bstride = bstr_i;
      op2.alpha = -1.0;
      op2.M = gr.h2;
      op2.N = h;
      op2.K = gr.h2;
      op2.batch = gr.count;
      op2.k_hi_mode = 1;                               // Cinv22 lower: A(m, k) = 0 for k > m
      e = gemm(op2, st);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

}  // namespace gi
