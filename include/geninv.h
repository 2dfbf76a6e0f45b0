/*
 * geninv.h -- C ABI of the B200-native (sm_100a) FP64 geninv library.
 *
 * Computes the Moore-Penrose inverse G+ of a real m x n matrix G with
 * Courrieu's full-rank-Cholesky method (arXiv 0804.4809, "Fast Computation
 * of Moore-Penrose Inverse Matrices"; PAPER.md line numbers cited as P:NN):
 *
 *   a0  if m < n: work with G G' (transpose branch), else G' G
 *   a1  A = G'G (or GG'), s x s with s = min(m, n)
 *   a2  tol = 1e-9 * min{A_ii : A_ii > 0}   (0 if none)
 *   a3  rank-revealing full-rank Cholesky A = L L', natural column
 *       order, a column is kept iff its pivot > tol (strict)        P:118-133, Eq.(1)
 *   a4  B = L'L;  a5  M = inv(B) (SPD: Cholesky, triangular inverse,
 *       product)
 *   a6  K = L M, X = K K'  (= L M M L', Theorem 1)
 *   a7  G+ = X G'  (m >= n)   or   G+ = G' X  (m < n)
 *   a8  row-sharded Gram: A = sum_p G_p' G_p (caller all-reduces A)
 *   a9  batched: many independent small G, one CTA per matrix
 *
 * Conventions (all entry points):
 *   - FP64 (double), ROW-MAJOR storage: element (i, j) of a matrix with
 *     leading dimension ld is at ptr[i * ld + j].
 *   - Pointers named *_dev / G / Gp / A are DEVICE pointers on the handle's
 *     device unless stated; *_host are host pointers (pinned memory gives
 *     overlapped copies; pageable memory works but is slower).
 *   - The caller owns G (never written), G+ and every output buffer; the
 *     handle owns its workspace (about 7 s^2 doubles + split-K partials),
 *     grown on demand and freed by geninv_destroy.  G and G+ must not alias.
 *   - Work is enqueued on the handle's stream (geninv_set_stream).  Calls
 *     that return a host-side rank / info synchronise that stream.
 *   - Errors are status codes; nothing throws across the ABI.  A handle is
 *     not thread-safe; separate handles are independent.
 *   - Alignment: any leading dimension ld >= n and any (8-byte aligned)
 *     base pointer is accepted.  The tensor-core path reads G, F and L with
 *     TMA, which needs 16-byte-aligned bases and even leading dimensions: an
 *     operand without them is first copied (stream-ordered, device to device)
 *     into a handle-owned aligned buffer -- one extra m x n doubles of device
 *     memory and one copy; aligned operands are read in place.  Outputs
 *     (G+, W, M, X) are written with plain stores: any ldp works.
 */
#ifndef GENINV_H_
#define GENINV_H_

#include <stdint.h>

#if defined(__GNUC__)
#define GENINV_API __attribute__((visibility("default")))
#else
#define GENINV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  GENINV_OK = 0,
  GENINV_EINVAL = 1,      /* bad size / leading dimension / null pointer */
  GENINV_ENONFINITE = 2,  /* non-finite diagonal of A (NaN/Inf in G) */
  GENINV_ENOTSPD = 3,     /* a5: a pivot <= 0 in the Cholesky of L'L (reading R8) */
  GENINV_ECUDA = 4,       /* CUDA runtime / launch error */
  GENINV_ENOMEM = 5,      /* device allocation failed */
  GENINV_EALIGN = 6,      /* reserved: no longer returned (unaligned operands are staged, see above) */
  GENINV_ESTATE = 7,      /* geninv_apply_d before geninv_from_gram_d, or shape mismatch */
  GENINV_ENCCL = 8,       /* geninv_sharded_d: libnccl.so.2 not loadable or ncclAllReduce failed */
  GENINV_ERANGE = 9       /* an accepted pivot below 2^-1022 (subnormal, ~2.2e-308): |G| is too
                             small for the branch-free sqrt / reciprocal of the factorisations --
                             scale G by a power of two (G+ scales by its inverse) */
} geninv_status;

/* Tolerance policy (SPEC ToleranceConfig).  NULL opts = the paper's policy. */
typedef struct {
  double tol_rel; /* relative factor, default 1e-9 */
  double tol_abs; /* < 0: paper policy tol = tol_rel * min positive diag; >= 0: this absolute tol */
} geninv_opts;

/* Diagnostics of one factorisation (device values copied back to the host). */
typedef struct {
  double tol;        /* the tolerance actually used */
  int64_t rank;      /* detected rank r */
  int32_t transposed;/* 1 if the m < n branch was taken */
  int32_t status;    /* geninv_status of the call */
  double min_acc;    /* smallest accepted pivot c_k (before sqrt); +inf if none */
  double max_drop;   /* largest |c_k| over dropped columns; 0 if none */
  double min_pivot;  /* smallest c_k over all columns */
  int32_t order;     /* a7 product order used by geninv_d: 0 = X G' / G' X with X = K K';
                        1 = K (K' G') / (G' K) K' (low rank) */
  int32_t not_psd_hint; /* 1 if a tentative pivot fell below -s * tol (SPEC's definiteness rule): the
                           paper drops it like any pivot <= tol, so it is not an error -- G'G never
                           produces one beyond rounding, a user-supplied non-PSD A (geninv_from_gram_d,
                           geninv_frchol_d) does */
} geninv_info;

typedef struct geninv_handle_s *geninv_handle;

/* Create a handle bound to CUDA device `device` with its own non-blocking stream. */
GENINV_API geninv_status geninv_create(geninv_handle *h, int device);
/* Use `stream` (a cudaStream_t passed as void*) for all later work; NULL = the legacy default
 * stream.  Until this is called the handle uses its own non-blocking stream. */
GENINV_API geninv_status geninv_set_stream(geninv_handle h, void *stream);
GENINV_API geninv_status geninv_destroy(geninv_handle h);
/* Arithmetic of the two big contractions (opt-in).  mode 0 (default): FP64 tensor
 * cores (DMMA).  mode 1: the output product (a7, both branches, X order) and the Gram (a1, s >= 3072;
 * not for geninv_host_d's accumulating chunks) emulated on the INT8 tensor cores (tcgen05.mma.kind::i8):
 * every line of the operands is scaled by a power of two and split into 7 int8 digits, the 34 digit
 * products with t + u <= 9 are exact int32 sums in TMEM, accumulated in FP64 -- an error below
 * ~2.4e-17 sum_k |x_ik g_jk|, under an FP64 GEMM's own rounding bound.  a7 for
 * s = min(m, n) <= 16384, the Gram for 3072 <= s <= 16384; lines outside 2^(+-900) or with NaN / Inf
 * fall back to DMMA.  Environment GENINV_EMULATE=1
 * sets mode 1 for handles that never call this. */
GENINV_API geninv_status geninv_set_emulation(geninv_handle h, int mode);
GENINV_API const char *geninv_strerror(geninv_status st);

/* ---- whole path, single matrix (a0-a7) ------------------------------------
 * G: m x n device, ld >= n.  Gp: n x m device, ldp >= m, overwritten.
 * rank (host, may be NULL) receives r; info (host, may be NULL) diagnostics.
 * Zero G -> rank 0 and G+ = 0 (reading R2).  Synchronises the stream.
 * Small matrices (min(m, n) <= 64, max(m, n) <= 128) run the whole path in one
 * CTA (the batched kernel, a9; G read in place at any alignment); that path does not keep X in the handle
 * (geninv_copy_x then returns GENINV_ESTATE).  For low rank, where
 * 4 r s l < s (s + 1) r + 2 s^2 l (s = min(m, n), l = max(m, n)), geninv_d skips
 * X and evaluates G+ = K (K' G') (m >= n) or (G' K) K' (m < n) with K = L M,
 * in chunks of the long side (info->order = 1; X is then not kept either). */
GENINV_API geninv_status geninv_d(geninv_handle h, const double *G, int64_t m, int64_t n, int64_t ld, double *Gp,
                       int64_t ldp, int64_t *rank, const geninv_opts *opts, geninv_info *info);

/* Asynchronous variant: nothing is copied back and the stream is not synchronised.  rank_dev
 * (device int64) receives r, or -GENINV_ENONFINITE / -GENINV_ENOTSPD / -GENINV_ERANGE; G+ is then
 * unspecified.
 * Without the rank on the host, the inverse runs at the full size s with an identity block past
 * the detected rank (M = diag(M_r, I); K = L M and X = K K' are exactly the rank-r results), so
 * it costs up to (s/r)^3 more inverse flops than geninv_d.  Always the X G' / G' X order. */
GENINV_API geninv_status geninv_d_async(geninv_handle h, const double *G, int64_t m, int64_t n, int64_t ld, double *Gp,
                             int64_t ldp, int64_t *rank_dev, const geninv_opts *opts);

/* Same computation with HOST buffers G_host (m x n, ld) and Gp_host (n x m, ldp):
 * the library stages G to the device in row chunks (copies overlapped with the
 * Gram), and streams G+ back overlapped with the output product.  Device
 * buffers for G and G+ chunks live in the handle's workspace. */
GENINV_API geninv_status geninv_host_d(geninv_handle h, const double *G_host, int64_t m, int64_t n, int64_t ld,
                            double *Gp_host, int64_t ldp, int64_t *rank, const geninv_opts *opts,
                            geninv_info *info);

/* ---- batched small matrices (a9) ------------------------------------------
 * `batch` independent m x n matrices: matrix b at G + b*strideG (device, ld >= n),
 * G+ of matrix b written at Gp + b*strideGp (n x m, ldp >= m).  rank_dev:
 * device int32[batch]: the rank of each matrix, or -GENINV_ENONFINITE (-2) /
 * -GENINV_ENOTSPD (-3) / -GENINV_ERANGE (-9) for a matrix with non-finite entries / a non-SPD L'L /
 * an accepted pivot below 2^-1022,
 * whose G+ is then filled with NaN.  Requires min(m, n) <= 64 and
 * max(m, n) <= 128 (GENINV_EINVAL otherwise).  Does not synchronise. */
GENINV_API geninv_status geninv_batched_d(geninv_handle h, const double *G, int64_t m, int64_t n, int64_t ld, int64_t strideG,
                               int64_t batch, double *Gp, int64_t ldp, int64_t strideGp, int32_t *rank_dev,
                               const geninv_opts *opts);

/* ---- minimum-norm least-squares solve ---------------------
 * W = G+ F, the paper's use of G+ for RBF synaptic weights (P:22, P:32-34 with
 * the "W = G+ W" typo read as W = G+ F, reading R10), without forming
 * G+: N branch (m >= n) W = X (G' F), T branch (m < n) W = G' (X F), with
 * X = L M M L' from steps a1-a6.  G: m x n (ld >= n), F: m x k (ldf >= k),
 * W: n x k (ldw >= k), all device, row-major; W is written.
 * rank / info as for geninv_d.  Synchronises.  The s x k intermediate lives
 * in the handle's workspace. */
GENINV_API geninv_status geninv_solve_d(geninv_handle h, const double *G, int64_t m, int64_t n, int64_t ld,
                             const double *F, int64_t k, int64_t ldf, double *W, int64_t ldw, int64_t *rank,
                             const geninv_opts *opts, geninv_info *info);

/* ---- sharded multi-GPU step (a8, north star: "G is row-sharded") ----------
 * One process per GPU.  trans == 0 (tall G, C4): G_local = this rank's rows
 * (m_local x n, ld), Gp_local = this rank's column block of G+ (n x m_local,
 * ldp >= m_local).  trans == 1 (wide G, C3): G_local = this rank's
 * columns (m x n_local passed as m_local = m, n = n_local), Gp_local = its row
 * block of G+ (n_local x m, ldp >= m).  The local Gram A_p is summed over the
 * ranks with one ncclAllReduce (FP64, sum) on the handle's stream; the
 * factorisation and inverse run replicated (deterministic: every rank gets the
 * same r and X); the output needs no further communication.  nccl_comm is an
 * ncclComm_t (e.g. torch ProcessGroupNCCL._comm_ptr()); NCCL is resolved at
 * run time from the already-loaded libnccl.so.2 (GENINV_ENCCL if absent).
 * Collective call: every rank of the communicator must call it.  Before the
 * all-reduce of A the ranks exchange (status, s) in one small MAX all-reduce,
 * so a local failure on any rank (bad arguments, ENOMEM, a CUDA error in its
 * Gram) or s differing between ranks returns that status (EINVAL for the shape)
 * on EVERY rank instead of blocking the others.
 * Synchronises; rank / info as for geninv_d. */
GENINV_API geninv_status geninv_sharded_d(geninv_handle h, void *nccl_comm, const double *G_local, int64_t m_local,
                               int64_t n, int64_t ld, int32_t trans, double *Gp_local, int64_t ldp, int64_t *rank,
                               const geninv_opts *opts, geninv_info *info);

/* ---- split form (row sharding, a8) -----------------------------------------
 * geninv_gram_d: A (s x s, lda >= s, device, caller-owned) = G'G if trans == 0
 *   (s = n), G G' if trans == 1 (s = m).  Lower triangle (and diagonal) written.
 *   For row shards with trans == 0 the caller sums A over ranks (all-reduce)
 *   before geninv_from_gram_d.  Does not synchronise.
 * geninv_from_gram_d: steps a2-a6 on the (summed) A: tol, full-rank Cholesky,
 *   M = inv(L'L), X = (LM)(LM)' kept in the handle.  Synchronises; rank/info out.
 * geninv_apply_d: step a7 with the handle's X: trans == 0: Gp (n x m_local) =
 *   X G_local'  (a column block of G+ for a row shard); trans == 1: Gp = G' X.
 *   Does not synchronise. */
GENINV_API geninv_status geninv_gram_d(geninv_handle h, const double *G, int64_t m, int64_t n, int64_t ld, int32_t trans,
                            double *A, int64_t lda);
GENINV_API geninv_status geninv_from_gram_d(geninv_handle h, const double *A, int64_t s, int64_t lda, int64_t *rank,
                                 const geninv_opts *opts, geninv_info *info);
GENINV_API geninv_status geninv_apply_d(geninv_handle h, const double *G, int64_t m, int64_t n, int64_t ld, int32_t trans,
                             double *Gp, int64_t ldp);

/* ---- single steps, exposed for step-level parity tests ----------------------
 * geninv_frchol_d (a2+a3): on A (s x s lower, lda): tol per opts, then the
 *   full-rank Cholesky.  L (s x s, ldl, device) receives the s x r factor in
 *   its first r columns (zeros above pivots and in columns >= r); piv_dev
 *   (device int32[s]) the pivot row of each kept column.  Synchronises.
 * geninv_spd_inverse_d (a5): M (r x r, ldm) = inv(B) for SPD B (r x r lower,
 *   ldb) via Cholesky, triangular inverse and C^-T C^-1; GENINV_ENOTSPD on a
 *   pivot <= 0.  Synchronises.
 * geninv_copy_x: copies the handle's X = L M M L' (s x s, from the last
 *   geninv_d / geninv_from_gram_d) into the device buffer X (ldx >= s) and
 *   synchronises; X == NULL only reports s.  GENINV_ESTATE before any call. */
GENINV_API geninv_status geninv_frchol_d(geninv_handle h, const double *A, int64_t s, int64_t lda, double *L, int64_t ldl,
                              int32_t *piv_dev, int64_t *rank, const geninv_opts *opts, geninv_info *info);
GENINV_API geninv_status geninv_spd_inverse_d(geninv_handle h, const double *B, int64_t r, int64_t ldb, double *M,
                                   int64_t ldm);
GENINV_API geninv_status geninv_copy_x(geninv_handle h, double *X, int64_t ldx, int64_t *s);

/* Number of kernels this handle has launched so far (launch accounting for bench.py). */
GENINV_API int64_t geninv_launch_count(geninv_handle h);

#ifdef __cplusplus
}
#endif
#endif /* GENINV_H_ */
