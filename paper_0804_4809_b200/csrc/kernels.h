// Host entry points of the geninv step kernels (frchol.cu, spdinv.cu, batched.cu).
#pragma once
#include <cuda_runtime.h>

namespace gi {

constexpr int PB = 32;  // panel width of the blocked full-rank Cholesky

// Device-side diagnostics of one factorisation run.
struct FactorStats {
  double min_acc;    // min accepted pivot
  double max_drop;   // max |dropped pivot|
  double min_pivot;  // min pivot
  double tol;        // tolerance used
  int flags;         // bit0: non-finite diagonal, bit1: non-SPD pivot (mode 1), bit2: accepted pivot < 2^-1022
  int pad;           // spare (the one-CTA small path stores the rank here)
};

// a2: tol = tol_abs >= 0 ? tol_abs : tol_rel * min{A_ii > 0} (0 if none); also
// initialises the stats block and flags a non-finite diagonal.
cudaError_t tolerance(const double *A, long long lda, int s, double tol_rel, double tol_abs, FactorStats *st,
                      cudaStream_t stream);

// a3: blocked left-looking rank-revealing Cholesky with one-panel lookahead.
// L (s x s, ldl) must be zero on entry; rk: device int[ceil(s/PB)+1] (rk[p] =
// rank before panel p, rk[npanels] = final rank); piv: device int[s]; Wp:
// workspace of wp_elems doubles (>= 40 * s * PB).  mode 0: drop iff pivot <=
// tol (paper); mode 1: SPD (accept iff pivot > 0, flag bit1 otherwise).  The
// big updates run on `upd` (a second stream) concurrently with the previous
// one or two panels (lookahead depth by s), alternating between the streams
// upd and upd2 (consecutive updates are independent); ev: 8 events owned by the caller.
cudaError_t frchol(const double *A, long long lda, int s, double *L, long long ldl, int *piv, int *rk,
                   FactorStats *st, int mode, double *Wp, long long wp_elems, cudaStream_t stream,
                   cudaStream_t upd, cudaStream_t upd2, cudaEvent_t *ev);

// Kernel launches frchol makes for size s (panels + lookahead updates).
int frchol_launches(int s);

// a5 pieces: Cinv = C^-1 for lower-triangular C (r x r, ldc) padded to
// r_pad = round_up(r, 32) with an identity block; C and Cinv are r_pad x r_pad
// buffers (ld), C zero outside its r x r lower triangle, Cinv zero on entry.
// T: workspace of r_pad * r_pad doubles.
cudaError_t trtri_lower(double *C, long long ldc, int r, double *Cinv, long long ldi, double *T, double *part,
                        long long part_elems, cudaStream_t stream);
// Doubles of split-K partial workspace trtri_lower uses for (r, ldc, ldi) (0: no split).
long long trtri_part_elems(int r, long long ldc, long long ldi);
// Kernel launches trtri_lower makes with that workspace.
int trtri_launches(int r, long long ldc, long long ldi, long long part_elems);

// a9: batched small geninv, one CTA per matrix (min(m,n) <= 64, max(m,n) <= 128).  rank[b] >= 0, or
// -2 (non-finite G) / -3 (L'L not SPD) / -9 (an accepted pivot below 2^-1022) with G+_b = NaN.  stats (optional, device, one per matrix):
// tol, decision margins and flags (bit0 non-finite, bit1 not SPD, bit2 pivot < 2^-1022) of each matrix.
cudaError_t batched_geninv(const double *G, int m, int n, long long ld, long long strideG, long long batch,
                           double *Gp, long long ldp, long long strideGp, int *rank, double tol_rel,
                           double tol_abs, cudaStream_t stream, FactorStats *stats = nullptr);

}  // namespace gi
