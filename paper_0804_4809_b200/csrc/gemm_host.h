// Host-side description of one FP64 tensor-core GEMM launch (see gemm.cuh).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gi {

struct Mat {               // row-major device matrix (or batch of equally-shaped blocks)
  const double *ptr = nullptr;
  long long ld = 0, rows = 0, cols = 0;
  int batch = 1;
  long long bstride = 0;   // elements between batch items
};

enum Tile { TILE_128x128 = 0, TILE_128x32 = 1, TILE_64x64 = 2 };   // TILE_128x32: N = 32 panel updates (256 x 32 when both operands are K-major, see upd_tile_bm)

struct GemmOp {
  Mat A;  bool a_kmajor = true;  int a_mn0 = 0, a_k0 = 0;
  Mat B;  bool b_kmajor = true;  int b_mn0 = 0, b_k0 = 0;
  double *C = nullptr; long long ldc = 0, c_bstride = 0;
  const double *C0 = nullptr; long long ldc0 = 0, c0_bstride = 0;
  double alpha = 1.0;
  int M = 0, N = 0, K = 0;
  const int *K_dev = nullptr;   // device-side K (overrides K; K is then the upper bound)
  int k_lo_mode = 0, k_hi_mode = 0;  // per-tile k-range of a triangular operand (see GemmArgs)
  const int *k_lo_dev = nullptr;
  int batch = 1;
  bool lower = false, mirror = false;
  int splits = 1; long long split_stride = 0;
  int kchunk = 0;                // > 0: two-level accumulation in chunks of kchunk k-slabs (alpha 1, no C0 /
                                 //   mirror; 128 x 128 tiles) -- the Gram's accuracy over millions of rows
  Tile tile = TILE_128x128;
};

// Enqueue one GEMM on `st`.  Returns cudaSuccess or the launch / encode error.
int upd_tile_bm();   // rows of the panel update's tiles (TILE_128x32 with K-major operands): 256, or 128
cudaError_t gemm(const GemmOp &op, cudaStream_t st);

// Sum split-K partial slices in a fixed order:  out = C0 + alpha * sum_z P[z]
// (C0 may be null).  lower: only elements with j <= i (square M == N).
// (lower && mirror: also out[j][i] = out[i][j], the symmetric store of a lower-only reduction.)
cudaError_t splitk_reduce(const double *P, long long split_stride, int splits, long long ldp, double *out,
                          long long ldo, const double *C0, long long ldc0, double alpha, int M, int N, bool lower,
                          cudaStream_t st, bool mirror = false);

int num_sms();   // SM count of the current device (cached per device)

// Opt `fn` in to `bytes` of dynamic shared memory on the CURRENT device (the attribute is per device /
// context: done once per (kernel, device), thread-safe).
cudaError_t smem_optin(const void *fn, int bytes);

// Tile size and split-K count of a chain product from a schedule simulation (see gemm.cu).
struct GemmPlan {
  int splits = 1;
  Tile tile = TILE_128x128;
};
GemmPlan balanced_plan(const GemmOp &op, int max_splits, int sms);
int balanced_splits(const GemmOp &op, int max_splits, int sms);   // balanced_plan(...).splits

}  // namespace gi
