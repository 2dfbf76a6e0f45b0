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

#include <stdlib.h>

#include <algorithm>
#include <vector>

namespace gi {

__global__ void pad_identity_kernel(double *C, long long ldc, int r, int r_pad) {
  const int i = r + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < r_pad) C[(long long)i * ldc + i] = 1.0;
}

// Inverse of each 32 x 32 lower-triangular diagonal block; thread j owns column j.  Right-looking forward
// substitution: x_i = a_i * (1 / C_ii) (the 32 reciprocals computed once, in parallel), then a_k -= C_ki x_i
// for k > i -- the dependent chain per row is one multiply and one FMA (the left-looking form had a dependent
// sum of up to 31 FMAs and a division per row: ~13 us per launch at r = 1024, now ~2 us).
__global__ void trtri_diag_kernel(const double *__restrict__ C, long long ldc, double *__restrict__ Ci,
                                  long long ldi) {
  __shared__ double c[32][33];
  __shared__ double rd[32];
  const int b0 = blockIdx.x * 32;
  const int j = threadIdx.x;
  for (int i = 0; i < 32; ++i) c[i][j] = C[(long long)(b0 + i) * ldc + b0 + j];
  __syncthreads();
  rd[j] = 1.0 / c[j][j];
  __syncthreads();
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = i == j ? 1.0 : 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    x[i] = i >= j ? x[i] * rd[i] : 0.0;
#pragma unroll
    for (int k = i + 1; k < 32; ++k) x[k] = fma(-c[k][i], x[i], x[k]);
  }
#pragma unroll
  for (int i = 0; i < 32; ++i)
    if (i >= j) Ci[(long long)(b0 + i) * ldi + b0 + j] = x[i];
}

// The level GEMMs of the recursive doubling, in launch order (op1, op2 per group and level).
std::vector<GemmOp> trtri_ops(double *C, long long ldc, int r, double *Ci, long long ldi, double *T) {
  std::vector<GemmOp> ops;
  const int r_pad = (r + 31) / 32 * 32;
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
      ops.push_back(op1);
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
      ops.push_back(op2);
    }
  }
  return ops;
}

GemmPlan trtri_plan(const GemmOp &op) {
  static const int on = [] {
    const char *e = getenv("GENINV_CHAIN_SPLIT");
    return e ? atoi(e) : 1;
  }();
  return on ? balanced_plan(op, 8, num_sms()) : GemmPlan();
}
int trtri_splits(const GemmOp &op) { return trtri_plan(op).splits; }

int trtri_launches(int r, long long ldc, long long ldi, long long part_elems) {
  const int r_pad = (r + 31) / 32 * 32;
  if (r_pad == 0) return 0;
  int n = (r_pad > r ? 1 : 0) + 1;
  for (const GemmOp &op : trtri_ops(nullptr, ldc, r, nullptr, ldi, nullptr)) {
    int S = trtri_splits(op);
    while (S > 1 && (long long)S * op.batch * op.M * op.N > part_elems) --S;
    n += S > 1 ? 2 : 1;
  }
  return n;
}

long long trtri_part_elems(int r, long long ldc, long long ldi) {
  long long need = 0;
  for (const GemmOp &op : trtri_ops(nullptr, ldc, r, nullptr, ldi, nullptr)) {
    const int S = trtri_splits(op);
    if (S > 1) need = std::max(need, (long long)S * op.batch * op.M * op.N);
  }
  return need;
}

// Batched fixed-order split-K sum: out_b = alpha * sum_z P[z][b]  (P: split stride sstride, batch stride
// M * N, ld N; out: batch stride obs, ld ldo).
__global__ void splitk_reduce_batched_kernel(const double *__restrict__ P, long long sstride, int splits,
                                             double *__restrict__ out, long long ldo, long long obs, double alpha,
                                             int M, int N, int batch) {
  const long long per = (long long)M * N, total = per * batch;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / per);
    const long long e = idx - b * per;
    const int i = (int)(e / N), j = (int)(e % N);
    double v = 0.0;
    for (int z = 0; z < splits; ++z) v += P[z * sstride + idx];
    out[b * obs + (long long)i * ldo + j] = alpha * v;
  }
}

cudaError_t trtri_lower(double *C, long long ldc, int r, double *Ci, long long ldi, double *T, double *part,
                        long long part_elems, cudaStream_t st) {
  const int r_pad = (r + 31) / 32 * 32;
  if (r_pad == 0) return cudaSuccess;
  if (r_pad > r) pad_identity_kernel<<<1, 32, 0, st>>>(C, ldc, r, r_pad);
  trtri_diag_kernel<<<r_pad / 32, 32, 0, st>>>(C, ldc, Ci, ldi);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  for (GemmOp op : trtri_ops(C, ldc, r, Ci, ldi, T)) {
    const GemmPlan pl = trtri_plan(op);
    op.tile = pl.tile;
    int S = part ? pl.splits : 1;
    const long long per = (long long)op.M * op.N;
    while (S > 1 && (long long)S * op.batch * per > part_elems) --S;
    if (S <= 1) {
      if ((e = gemm(op, st)) != cudaSuccess) return e;
      continue;
    }
    double *out = op.C;
    const long long ldo = op.ldc, obs = op.c_bstride;
    const double alpha = op.alpha;
    op.C = part;
    op.ldc = op.N;
    op.c_bstride = per;
    op.splits = S;
    op.split_stride = per * op.batch;
    if ((e = gemm(op, st)) != cudaSuccess) return e;
    const long long total = per * op.batch;
    const int blocks = (int)std::min<long long>((total + 255) / 256, (long long)num_sms() * 8);
    splitk_reduce_batched_kernel<<<blocks, 256, 0, st>>>(part, per * op.batch, S, out, ldo, obs, alpha, op.M, op.N,
                                                         op.batch);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace gi
