// FP64 products emulated on the INT8 tensor cores (Ozaki splitting, tcgen05.mma.kind::i8); see emu.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gi {

// K rounded up to 16 bytes (the slice arrays' row length; TMA needs 16-byte row strides).
int emu_kpad(int K);

// rows x K FP64 block (row stride ldx) -> S digit slices [S][rows][emu_kpad(K)] (digit 1 signed int8,
// the others unsigned, see emu.cu) and one
// power-of-two exponent per row; *flag |= 1 for a row outside the exact-scaling range.
cudaError_t emu_split(const double *X, long long ldx, int rows, int K, int S, int8_t *slices, int *exps, int *flag,
                      cudaStream_t st);

// The COLUMNS of the rows x cols block G (row stride ld) -> digit planes [S][cols][emu_kpad(rows)] and
// one exponent per column (the K-major operand of G'G for a K-chunk of rows); colmax: workspace of
// cols uint64.
cudaError_t emu_split_cols(const double *G, long long ld, int rows, int cols, int S, int8_t *slices, int *exps,
                           unsigned long long *colmax, int *flag, cudaStream_t st);

// C (M x N, row stride ldc) = A B' from the slices of A (M rows) and B (N rows) over K, groups
// t + u <= T (S = 7, T = 9: 34 int8 products, FP64-level accuracy).  K <= 4096.  scratch: FP64
// workspace of emu_scratch_elems(M, N) (the running sums, one tile per CTA).
long long emu_scratch_elems(int M, int N);
// lower: only the tiles of a square output's lower triangle (M == N); accumulate: C += A B'.
cudaError_t emu_gemm_nt(const int8_t *As, const int *ea, int M, const int8_t *Bs, const int *eb, int N, int K, int S,
                        int T, double *C, long long ldc, double *scratch, cudaStream_t st, int lower = 0,
                        int accumulate = 0);

}  // namespace gi
