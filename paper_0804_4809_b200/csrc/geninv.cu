// Host orchestrator + C ABI (include/geninv.h) of the sm_100a geninv library.
//
// Plans the step sequence of PAPER.md P:105-140 for (m, n), owns the
// workspace and the stream, and enqueues the kernels:
//   a1 gram (gemm.cu, lower tiles, split-K + fixed-order reduction)
//   a2 tolerance, a3 frchol (frchol.cu)         -- one host sync to read r
//   a4 B = L'L, a5 POTRF (frchol mode 1) + TRTRI (spdinv.cu) + C^-T C^-1
//   a6 K = L M, X = K K'  (flop-minimal reassociation of P:137/P:139, R9)
//   a7 G+ = X G' or G' X
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <vector>

#include "../../include/geninv.h"
#include "emu.h"
#include "gemm_host.h"
#include "kernels.h"

using namespace gi;

struct geninv_handle_s {
  int device = 0;
  cudaStream_t own = nullptr, st = nullptr, st2 = nullptr, upd = nullptr, upd2 = nullptr;
  // CUDA graphs of the launch-bound factorisation chain (replayed while the shapes/pointers match)
  struct GraphSlot {
    cudaGraphExec_t exec = nullptr;
    long long key[10] = {};
    long long nlaunch = 0;   // kernels in the graph (counted while capturing)
  } g_factor, g_build, g_async;
  cudaStream_t gstream = nullptr;   // private non-blocking stream the graphs are captured / launched on
  cudaEvent_t ev_g[2] = {};
  cudaEvent_t ev[4] = {};
  cudaEvent_t ev_fr[8] = {};  // frchol lookahead events
  // s x s workspaces (leading dimension ld >= round_up(s, 32))
  int s_cap = 0;
  long long ld = 0;
  double *A = nullptr, *L = nullptr, *Bm = nullptr, *Cf = nullptr, *Ci = nullptr, *Mm = nullptr, *Kb = nullptr,
         *X = nullptr, *T = nullptr;
  double *Wp = nullptr;
  long long wp_elems = 0;
  double *part = nullptr;  // Gram split-K partials
  size_t part_bytes = 0;
  int *rk = nullptr, *piv = nullptr, *rk2 = nullptr, *piv2 = nullptr;
  FactorStats *fs = nullptr, *fs2 = nullptr;
  // host-buffer path staging
  double *Gdev = nullptr, *Gpchunk[2] = {nullptr, nullptr};
  size_t gdev_bytes = 0, chunk_bytes = 0;
  // least-squares solve (f1): the s x k intermediate G'F or X F
  double *T1 = nullptr;
  size_t t1_bytes = 0;
  // aligned copies of caller operands the TMA path cannot read in place (stage_operand)
  double *stage[2] = {nullptr, nullptr};
  double *coll = nullptr;   // geninv_sharded_d: the small pre-check all-reduce buffer
  size_t stage_bytes[2] = {0, 0};
  // a7 emulated on the INT8 tensor cores (geninv_set_emulation): slices of X and of a chunk of G
  int emulate = -1;        // -1: not set (GENINV_EMULATE decides), 0 native DMMA, 1 emulated
  int8_t *emu_x = nullptr, *emu_g = nullptr;
  int *emu_ex = nullptr, *emu_eg = nullptr, *emu_flag = nullptr;
  double *emu_sc = nullptr;
  unsigned long long *emu_cm = nullptr;
  size_t emu_x_bytes = 0, emu_g_bytes = 0, emu_ex_n = 0, emu_eg_n = 0, emu_sc_n = 0, emu_cm_n = 0;
  // state of the last factorisation (for geninv_apply_d)
  int x_s = -1;
  int last_rank = 0;
  long long launches = 0;
};

namespace {

// NVTX range per step (SURVEY §5 tracing): visible in nsys / ncu --nvtx timelines; a no-op (one call into the
// NVTX stub) when no tool is attached.
struct Range {
  explicit Range(const char *name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
  Range(const Range &) = delete;
  Range &operator=(const Range &) = delete;
};

geninv_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return GENINV_OK;
  if (e == cudaErrorMemoryAllocation) return GENINV_ENOMEM;
  if (e == cudaErrorMisalignedAddress) return GENINV_EALIGN;
  fprintf(stderr, "[geninv] CUDA error: %s\n", cudaGetErrorString(e));
  return GENINV_ECUDA;
}

#define GI_TRY(expr)                                                             \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      fprintf(stderr, "[geninv] %s:%d: %s\n", __FILE__, __LINE__, #expr);        \
      return cuda_status(_e);                                                    \
    }                                                                            \
  } while (0)

// GENINV_DEBUG_SYNC: synchronise the device after a step and report the first failing one (diagnostics)
bool debug_sync_on() {
  static const bool on = getenv("GENINV_DEBUG_SYNC") != nullptr;
  return on;
}
#define GI_DBG_SYNC(tag)                                                                        \
  do {                                                                                          \
    if (debug_sync_on()) {                                                                      \
      cudaError_t _e = cudaDeviceSynchronize();                                                 \
      fprintf(stderr, "[geninv] sync after %s: %s\n", tag, cudaGetErrorString(_e));            \
    }                                                                                           \
  } while (0)

#define GI_TRYS(expr)                                 \
  do {                                                \
    geninv_status _s = (expr);                        \
    if (_s != GENINV_OK) return _s;                   \
  } while (0)

void free_ws(geninv_handle h) {
  double **bufs[] = {&h->A, &h->L, &h->Bm, &h->Cf, &h->Ci, &h->Mm, &h->Kb, &h->X, &h->T, &h->Wp};
  for (auto b : bufs) {
    if (*b) cudaFree(*b);
    *b = nullptr;
  }
  int **ibufs[] = {&h->rk, &h->piv, &h->rk2, &h->piv2};
  for (auto b : ibufs) {
    if (*b) cudaFree(*b);
    *b = nullptr;
  }
  if (h->fs) cudaFree(h->fs);
  if (h->fs2) cudaFree(h->fs2);
  h->fs = h->fs2 = nullptr;
  h->s_cap = 0;
  h->x_s = -1;
}

geninv_status ensure_ws(geninv_handle h, int s) {
  if (s <= h->s_cap) return GENINV_OK;
  cudaStreamSynchronize(h->st);
  free_ws(h);
  const long long ld = (s + 31) / 32 * 32;
  const size_t sq = (size_t)ld * ld * sizeof(double);
  double **bufs[] = {&h->A, &h->L, &h->Bm, &h->Cf, &h->Ci, &h->Mm, &h->Kb, &h->X, &h->T};
  for (auto b : bufs) GI_TRY(cudaMalloc(b, sq));
  h->wp_elems = 40LL * ld * PB;
  GI_TRY(cudaMalloc(&h->Wp, h->wp_elems * sizeof(double)));
  const int np = (int)(ld / PB) + 2;
  GI_TRY(cudaMalloc(&h->rk, np * sizeof(int)));
  GI_TRY(cudaMalloc(&h->rk2, np * sizeof(int)));
  GI_TRY(cudaMalloc(&h->piv, ld * sizeof(int)));
  GI_TRY(cudaMalloc(&h->piv2, ld * sizeof(int)));
  GI_TRY(cudaMalloc(&h->fs, sizeof(FactorStats)));
  GI_TRY(cudaMalloc(&h->fs2, sizeof(FactorStats)));
  h->s_cap = (int)ld;
  h->ld = ld;
  return GENINV_OK;
}

geninv_status ensure_part(geninv_handle h, size_t bytes) {
  if (bytes <= h->part_bytes) return GENINV_OK;
  cudaStreamSynchronize(h->st);
  if (h->part) cudaFree(h->part);
  h->part = nullptr;
  h->part_bytes = 0;
  GI_TRY(cudaMalloc(&h->part, bytes));
  h->part_bytes = bytes;
  return GENINV_OK;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Split-K count for `tiles` output tiles over `nslab` k-slabs: the smallest
// split whose wave efficiency (1 CTA / SM) is within 2 % of the best.
int pick_splits(long long tiles, long long nslab) {
  const int sms = num_sms();
  double eff[17];
  double best = 0;
  for (int S = 1; S <= 16; ++S) {
    eff[S] = 0;
    if (S > 1 && nslab / S < 16) break;
    const long long work = tiles * S;
    const long long waves = (work + sms - 1) / sms;
    eff[S] = (double)work / (double)(waves * sms);
    best = std::max(best, eff[S]);
  }
  for (int S = 1; S <= 16; ++S)
    if (eff[S] >= best - 0.02) return S;
  return 1;
}

bool emulation_on(geninv_handle h) {
  if (h->emulate >= 0) return h->emulate != 0;
  static const int env = [] {
    const char *e = getenv("GENINV_EMULATE");
    return e ? atoi(e) : 0;
  }();
  return env != 0;
}

template <typename T>
geninv_status grow(T *&p, size_t &have, size_t need) {
  if (need <= have) return GENINV_OK;
  if (p) cudaFree(p);
  p = nullptr;
  have = 0;
  GI_TRY(cudaMalloc(&p, need * sizeof(T)));
  have = need;
  return GENINV_OK;
}

// Digits per line (7: 7 + 6 x 8 = 55 bits) and the largest digit group t + u of the emulated products
// (9: 34 products, |error| <= 2.4e-17 sum |x g| measured -- FP64-level; 8: 28 products, 2.9e-15, too
// coarse for the 1e-9 gate on C4); GENINV_EMU_T (2 .. 14) trades accuracy for work in measurements.
constexpr int EMU_S = 7;
constexpr int EMU_K = 4096;   // K per exact int32 pass: 7 pairs x 4096 x 255^2 < 2^31
int emu_groups() {
  static const int T = [] {
    const char *e = getenv("GENINV_EMU_T");
    const int t = e ? atoi(e) : 9;
    return t >= 2 && t <= 14 ? t : 9;
  }();
  return T;
}

// a1 on the INT8 tensor cores (geninv_set_emulation): K-chunks of <= EMU_K lines of G (the int32
// group sums stay exact), each split into EMU_S int8 digits per column (N) / row (T) of the chunk, the
// lower tiles of A accumulated chunk after chunk in FP64 (fixed order: deterministic).  GENINV_ERANGE:
// a line outside the exact-scaling range (the caller then runs the DMMA Gram).
geninv_status gram_emulated(geninv_handle h, const double *G, long long m, long long n, long long ld, int trans,
                            double *A, long long lda, bool accumulate) {
  constexpr int S = EMU_S, KC = EMU_K;
  const int T = emu_groups();
  const long long s = trans ? m : n, ell = trans ? n : m;
  const int Kp = emu_kpad(KC);
  GI_TRYS(grow(h->emu_g, h->emu_g_bytes, (size_t)S * s * Kp));
  GI_TRYS(grow(h->emu_eg, h->emu_eg_n, (size_t)s));
  GI_TRYS(grow(h->emu_cm, h->emu_cm_n, (size_t)s));
  GI_TRYS(grow(h->emu_sc, h->emu_sc_n, (size_t)emu_scratch_elems((int)s, (int)s)));
  if (!h->emu_flag) GI_TRY(cudaMalloc(&h->emu_flag, sizeof(int)));
  GI_TRY(cudaMemsetAsync(h->emu_flag, 0, sizeof(int), h->st));
  // two-level FP64 accumulation of the exact chunk sums: groups of GRP chunks are summed into the handle's
  // s x s scratch T, and the group sums into A (a sequential sum over 2^21 / 4096 = 512 chunks would be the
  // emulated Gram's only rounding; C4: ~sqrt(512) -> ~sqrt(16) + sqrt(32) chunk-sum roundings)
  constexpr int GRP = 16;
  const long long nchunks = (ell + KC - 1) / KC;
  const bool grouped = nchunks > GRP && !accumulate && s <= h->ld;
  for (long long c = 0; c < nchunks; ++c) {
    const long long k0 = c * KC;
    const int kc = (int)std::min<long long>(KC, ell - k0);
    if (!trans)
      GI_TRY(emu_split_cols(G + k0 * ld, ld, kc, (int)s, S, h->emu_g, h->emu_eg, h->emu_cm, h->emu_flag, h->st));
    else
      GI_TRY(emu_split(G + k0, ld, (int)s, kc, S, h->emu_g, h->emu_eg, h->emu_flag, h->st));
    h->launches += trans ? 2 : 3;
    if (!grouped) {
      GI_TRY(emu_gemm_nt(h->emu_g, h->emu_eg, (int)s, h->emu_g, h->emu_eg, (int)s, kc, S, T, A, lda, h->emu_sc, h->st,
                         1, (k0 > 0 || accumulate) ? 1 : 0));
      continue;
    }
    const bool first_of_group = c % GRP == 0, last_of_group = c % GRP == GRP - 1 || c == nchunks - 1;
    double *dst = c < GRP ? A : h->T;                      // the first group directly into A
    const long long ldd = c < GRP ? lda : h->ld;
    GI_TRY(emu_gemm_nt(h->emu_g, h->emu_eg, (int)s, h->emu_g, h->emu_eg, (int)s, kc, S, T, dst, ldd, h->emu_sc, h->st,
                       1, first_of_group ? 0 : 1));
    if (c >= GRP && last_of_group) {   // A += T (lower triangle, in place)
      GI_TRY(splitk_reduce(h->T, 0, 1, h->ld, A, lda, A, lda, 1.0, (int)s, (int)s, true, h->st));
      h->launches += 1;
    }
  }
  int flag = 0;
  GI_TRY(cudaMemcpyAsync(&flag, h->emu_flag, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  GI_TRY(cudaStreamSynchronize(h->st));
  return flag ? GENINV_ERANGE : GENINV_OK;
}

// Rows of G per register-accumulated partial sum of the DMMA Gram (GENINV_GRAM_CHUNK_ROWS; 0 = one
// sequential sum per CTA).  8192: C4's 2^21-row sums become 8k-row partials added in a fixed order.
int gram_chunk_rows() {
  static const int rows = [] {
    const char *e = getenv("GENINV_GRAM_CHUNK_ROWS");
    const int v = e ? atoi(e) : 8192;
    return v <= 0 ? 0 : std::max(16, v / 16 * 16);
  }();
  return rows;
}

// a1: A (s x s, lower) = G'G (trans == 0) or GG' (trans == 1).
geninv_status gram(geninv_handle h, const double *G, long long m, long long n, long long ld, int trans, double *A,
                   long long lda, const double *accumulate = nullptr) {
  Range rg("geninv a1 gram");
  const long long s = trans ? m : n, ell = trans ? n : m;
  // emulated Gram: only where its 128 x 256 lower tiles fill the machine (s >= 3072: >= 170 tiles);
  // an accumulating call could not fall back after a range flag
  if (emulation_on(h) && !accumulate && s >= 3072 && s <= 16384) {   // K-chunks of EMU_K lines
    const geninv_status es = gram_emulated(h, G, m, n, ld, trans, A, lda, false);
    if (es != GENINV_ERANGE) return es;   // out of the emulation's range: the DMMA Gram below
  }
  GemmOp op;
  op.A = Mat{G, ld, m, n};
  op.B = op.A;
  op.a_kmajor = op.b_kmajor = (trans != 0);  // T: A[i][j] = sum_k G[i][k] G[j][k]; N: sum_k G[k][i] G[k][j]
  op.M = op.N = (int)s;
  op.K = (int)ell;
  op.lower = true;
  const long long mt = (s + 127) / 128;
  const long long tiles = mt * (mt + 1) / 2;
  int S = pick_splits(tiles, (ell + 15) / 16);
  // accuracy: no partial sum runs over more than 2^17 rows of G (each DMMA tile accumulates its
  // k-range sequentially); the fixed-order reduction then adds the partials.  When that asks for
  // splits anyway, the count is rounded to the one (up to 48, partial slices within ~6 GB) with
  // the best last-wave fill of the tiles x splits CTAs (C4: 37 -> exactly 132 waves of 148).
  {
    const long long pbytes = (long long)h->ld * h->ld * 8;
    const int s_acc = (int)std::min<long long>(16, (ell + (1LL << 17) - 1) >> 17);
    const int s_cap = (int)std::max<long long>(1, (6144LL << 20) / pbytes);
    S = std::min(std::max(S, s_acc), std::max(S, s_cap));
    if (s_acc > 1 && ell / (16LL * 48) >= 16) {
      const int sms = num_sms();
      double best = -1.0;
      int bs = S;
      for (int c = S; c <= std::min(48, s_cap); ++c) {
        const long long work = tiles * c, waves = (work + sms - 1) / sms;
        const double eff = (double)work / (double)(waves * sms);
        if (eff > best + 1e-9) { best = eff; bs = c; }
      }
      S = bs;
    }
  }
  // two-level accumulation inside each CTA: register sums over chunks of <= gram_chunk_rows() rows of G,
  // added into the tile in memory (GemmOp::kchunk) -- the accuracy of the long Gram sums (C4: 2^21 rows)
  const long long per_cta = (ell + S - 1) / S;
  const int crow = gram_chunk_rows();
  if (crow > 0 && per_cta > crow) op.kchunk = crow / 16;
  if (S == 1 && !accumulate) {
    op.C = A;
    op.ldc = lda;
    GI_TRY(gemm(op, h->st));
    h->launches += 1;
    return GENINV_OK;
  }
  const long long pstride = (long long)h->ld * h->ld;
  GI_TRYS(ensure_part(h, (size_t)S * pstride * sizeof(double)));
  op.C = h->part;
  op.ldc = h->ld;
  op.splits = S;
  op.split_stride = pstride;
  GI_TRY(gemm(op, h->st));
  GI_TRY(splitk_reduce(h->part, pstride, S, h->ld, A, lda, accumulate, lda, 1.0, (int)s, (int)s, true, h->st));
  h->launches += 2;
  return GENINV_OK;
}

// One product C (M x N, ldc) = A B with split-K when the output has few tiles (skinny solves:
// K = m can be millions of rows); partial slices in the handle's Gram workspace, fixed-order sum.
geninv_status gemm_splitk(geninv_handle h, GemmOp op) {
  const long long tiles = (long long)((op.M + 127) / 128) * ((op.N + 127) / 128);
  int S = pick_splits(tiles, (op.K + 15) / 16);
  const long long pstride = (long long)op.M * op.N;
  S = (int)std::min<long long>(S, std::max<long long>(1, (1LL << 30) / (pstride * 8)));
  if (S <= 1) {
    GI_TRY(gemm(op, h->st));
    h->launches += 1;
    return GENINV_OK;
  }
  double *C = op.C;
  const long long ldc = op.ldc;
  GI_TRYS(ensure_part(h, (size_t)S * pstride * sizeof(double)));
  op.C = h->part;
  op.ldc = op.N;
  op.splits = S;
  op.split_stride = pstride;
  if (debug_sync_on())
    fprintf(stderr, "[geninv] gemm_splitk: part %p (%zu B) S %d pstride %lld -> C %p ldc %lld\n", (void *)h->part,
            h->part_bytes, S, pstride, (void *)C, ldc);
  GI_TRY(gemm(op, h->st));
  GI_DBG_SYNC("gemm_splitk: gemm");
  GI_TRY(splitk_reduce(h->part, pstride, S, op.N, C, ldc, nullptr, 0, 1.0, op.M, op.N, false, h->st));
  GI_DBG_SYNC("gemm_splitk: reduce");
  h->launches += 2;
  return GENINV_OK;
}

double tol_rel_of(const geninv_opts *o) { return o ? o->tol_rel : 1e-9; }
double tol_abs_of(const geninv_opts *o) { return o ? o->tol_abs : -1.0; }

// a2 + a3 on h->A-like input; L zeroed here.  Returns rank via host sync.
bool graphs_on() {
  static const bool on = [] {
    const char *e = getenv("GENINV_NO_GRAPH");
    return !(e && atoi(e) != 0);
  }();
  return on;
}

// Run `enqueue(stream)` as a CUDA graph on the handle's private stream, ordered after / before the
// work of h->st by events: captured on first use, replayed while `key` matches (same shapes and
// buffers).  The panel chain is ~4 launches per 32 columns; as a graph the host submits it once.
template <typename F>
geninv_status run_graph(geninv_handle h, geninv_handle_s::GraphSlot &slot, const long long (&key)[10], F enqueue) {
  if (!graphs_on()) return enqueue(h->st);
  cudaStream_t gs = h->gstream;
  GI_TRY(cudaEventRecord(h->ev_g[0], h->st));
  GI_TRY(cudaStreamWaitEvent(gs, h->ev_g[0], 0));
  bool hit = slot.exec != nullptr;
  for (int i = 0; i < 10 && hit; ++i) hit = slot.key[i] == key[i];
  if (!hit) {
    if (slot.exec) cudaGraphExecDestroy(slot.exec);
    slot.exec = nullptr;
    cudaGraph_t g = nullptr;
    GI_TRY(cudaStreamBeginCapture(gs, cudaStreamCaptureModeThreadLocal));
    const long long l0 = h->launches;
    geninv_status st = enqueue(gs);
    slot.nlaunch = h->launches - l0;
    h->launches = l0;
    cudaError_t e = cudaStreamEndCapture(gs, &g);
    if (st != GENINV_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    GI_TRY(e);
    e = cudaGraphInstantiate(&slot.exec, g, 0);
    cudaGraphDestroy(g);
    GI_TRY(e);
    for (int i = 0; i < 10; ++i) slot.key[i] = key[i];
  }
  GI_TRY(cudaGraphLaunch(slot.exec, gs));
  h->launches += slot.nlaunch;
  GI_TRY(cudaEventRecord(h->ev_g[1], gs));
  GI_TRY(cudaStreamWaitEvent(h->st, h->ev_g[1], 0));
  return GENINV_OK;
}

long long dbits(double x) {
  long long v;
  memcpy(&v, &x, sizeof(v));
  return v;
}

geninv_status factor(geninv_handle h, const double *A, long long lda, int s, double *L, long long ldl, int *piv,
                     const geninv_opts *opts, int *rank_out, FactorStats *hst) {
  Range rg("geninv a2-a3 tolerance + full-rank Cholesky");
  const long long key[10] = {(long long)(uintptr_t)A, lda, s, (long long)(uintptr_t)L, ldl, (long long)(uintptr_t)piv,
                             dbits(tol_rel_of(opts)), dbits(tol_abs_of(opts)), h->ld, 1};
  GI_TRYS(run_graph(h, h->g_factor, key, [&](cudaStream_t st) -> geninv_status {
    GI_TRY(tolerance(A, lda, s, tol_rel_of(opts), tol_abs_of(opts), h->fs, st));
    GI_TRY(cudaMemsetAsync(L, 0, (size_t)s * ldl * sizeof(double), st));
    GI_TRY(frchol(A, lda, s, L, ldl, piv, h->rk, h->fs, 0, h->Wp, h->wp_elems, st, h->upd, h->upd2, h->ev_fr));
    return GENINV_OK;
  }));
  const int np = (s + PB - 1) / PB;
  h->launches += 1 + frchol_launches(s);
  int r = 0;
  GI_TRY(cudaMemcpyAsync(&r, h->rk + np, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  GI_TRY(cudaMemcpyAsync(hst, h->fs, sizeof(FactorStats), cudaMemcpyDeviceToHost, h->st));
  GI_TRY(cudaStreamSynchronize(h->st));
  *rank_out = r;
  if (hst->flags & 1) return GENINV_ENONFINITE;
  if (hst->flags & 4) return GENINV_ERANGE;
  return GENINV_OK;
}

// ---- the chain GEMMs (a4-a6), built in one place so the split plan can be computed before capture
GemmOp op_ltl(geninv_handle h, int s, int r) {   // a4: B = L'L (r x r, lower): B[i][j] = sum_k L[k][i] L[k][j]
  const long long ld = h->ld;
  GemmOp b;
  b.A = Mat{h->L, ld, s, ld};
  b.B = b.A;
  b.a_kmajor = b.b_kmajor = false;
  b.M = b.N = r;
  b.K = s;
  b.lower = true;
  b.k_lo_mode = 3;                                     // L[k][i] = 0 above the pivot row piv[i] (Eq. 1)
  b.k_lo_dev = h->piv;
  b.C = h->Bm;
  b.ldc = ld;
  return b;
}
GemmOp op_lauum(geninv_handle h, int r, double *M, long long ldm) {   // M = C^-T C^-1 (full symmetric)
  const long long ld = h->ld;
  const int r_pad = (r + 31) / 32 * 32;
  GemmOp op;
  op.A = Mat{h->Ci, ld, r_pad, r_pad};
  op.B = op.A;
  op.a_kmajor = op.b_kmajor = false;
  op.M = op.N = r;
  op.K = r_pad;
  op.lower = true;
  op.mirror = true;
  op.k_lo_mode = 1;                                    // C^-1 lower: Ci[k][i] = 0 for k < i
  op.C = M;
  op.ldc = ldm;
  return op;
}
GemmOp op_k(geninv_handle h, int s, int r) {   // a6: K = L M (s x r):  K[i][c] = sum_j L[i][j] M[j][c]
  const long long ld = h->ld;
  GemmOp k;
  k.A = Mat{h->L, ld, s, r};
  k.a_kmajor = true;
  k.B = Mat{h->Mm, ld, r, r};
  k.b_kmajor = false;
  k.M = s;
  k.N = r;
  k.K = r;
  k.k_hi_mode = 2;                                     // L[i][j] = 0 for rows i < piv[j] (Eq. 1)
  k.k_lo_dev = h->piv;
  k.C = h->Kb;
  k.ldc = ld;
  return k;
}
GemmOp op_x(geninv_handle h, int s, int r) {   // X = K K' (s x s, full symmetric)
  const long long ld = h->ld;
  GemmOp x;
  x.A = Mat{h->Kb, ld, s, r};
  x.B = x.A;
  x.a_kmajor = x.b_kmajor = true;
  x.M = x.N = s;
  x.K = r;
  x.lower = true;
  x.mirror = true;
  x.C = h->X;
  x.ldc = ld;
  return x;
}

// Tile size (128 x 128 or 64 x 64) and split-K count of one chain GEMM (balanced_plan's simulation).
GemmPlan chain_plan(const GemmOp &op) {
  static const int on = [] {
    const char *e = getenv("GENINV_CHAIN_SPLIT");   // 0 disables (tuning / A-B runs)
    return e ? atoi(e) : 1;
  }();
  return on ? balanced_plan(op, 8, num_sms()) : GemmPlan();
}
int chain_splits(const GemmOp &op) { return chain_plan(op).splits; }

// One chain GEMM with the split-K count of its schedule simulation; partial slices in h->part
// (sized by prepare_chain beforehand: no allocation while a graph is being captured).
geninv_status gemm_chain(geninv_handle h, GemmOp op) {
  const GemmPlan pl = chain_plan(op);
  int S = pl.splits;
  op.tile = pl.tile;
  const long long pstride = (long long)op.M * op.N;
  while (S > 1 && (size_t)S * pstride * sizeof(double) > h->part_bytes) --S;
  if (getenv("GENINV_DEBUG_SPLITS"))
    fprintf(stderr, "chain gemm M=%d N=%d K=%d lower=%d lo=%d hi=%d -> splits %d\n", op.M, op.N, op.K, (int)op.lower,
            op.k_lo_mode, op.k_hi_mode, S);
  if (S <= 1) {
    GI_TRY(gemm(op, h->st));
    h->launches += 1;
    return GENINV_OK;
  }
  double *C = op.C;
  const long long ldc = op.ldc;
  const double alpha = op.alpha;
  const double *C0 = op.C0;
  const long long ldc0 = op.ldc0;
  const bool mirror = op.lower && op.mirror;   // partial slices lower only; the reduction stores both halves
  op.C = h->part;
  op.ldc = op.N;
  op.C0 = nullptr;
  op.mirror = false;
  op.splits = S;
  op.split_stride = pstride;
  GI_TRY(gemm(op, h->st));
  GI_TRY(splitk_reduce(h->part, pstride, S, op.N, C, ldc, C0, ldc0, alpha, op.M, op.N, op.lower, h->st, mirror));
  h->launches += 2;
  return GENINV_OK;
}

// Size h->part for the chain GEMMs of (s, r) before the chain is captured.
geninv_status prepare_chain(geninv_handle h, int s, int r, bool want_x) {
  if (r == 0) return GENINV_OK;
  size_t need = 0;
  GemmOp ops[4] = {op_ltl(h, s, r), op_lauum(h, r, h->Mm, h->ld), op_k(h, s, r), op_x(h, s, r)};
  for (int i = 0; i < (want_x ? 4 : 3); ++i) {
    const int S = chain_splits(ops[i]);
    if (S > 1) need = std::max(need, (size_t)S * ops[i].M * ops[i].N * sizeof(double));
  }
  need = std::max(need, (size_t)trtri_part_elems(r, h->ld, h->ld) * sizeof(double));
  return ensure_part(h, need);
}

// a5: M (r x r, ldm, full symmetric) = inv(B), B SPD (lower, ldb).  No sync.
geninv_status spd_inverse(geninv_handle h, const double *B, int r, long long ldb, double *M, long long ldm) {
  const long long ld = h->ld;
  const int r_pad = (r + 31) / 32 * 32;
  GI_TRY(cudaMemsetAsync(h->Cf, 0, (size_t)r_pad * ld * sizeof(double), h->st));
  GI_TRY(cudaMemsetAsync(h->Ci, 0, (size_t)r_pad * ld * sizeof(double), h->st));
  GI_TRY(tolerance(B, ldb, r, 0.0, 0.0, h->fs2, h->st));
  GI_TRY(frchol(B, ldb, r, h->Cf, ld, h->piv2, h->rk2, h->fs2, 1, h->Wp, h->wp_elems, h->st, h->upd, h->upd2, h->ev_fr));
  GI_TRY(trtri_lower(h->Cf, ld, r, h->Ci, ld, h->T, h->part, (long long)(h->part_bytes / sizeof(double)), h->st));
  // M = C^-T C^-1 : M[i][j] = sum_k Ci[k][i] Ci[k][j]
  GI_TRYS(gemm_chain(h, op_lauum(h, r, M, ldm)));
  h->launches += 1 + frchol_launches(r) + trtri_launches(r, ld, ld, (long long)(h->part_bytes / sizeof(double)));
  return GENINV_OK;
}

// ---- device-side rank (geninv_d_async): the chain runs at the full size s; past the detected rank
//      the pivot list is padded with s (empty k-ranges) and B = L'L gets an identity block, so
//      M = inv(diag(B_r, I)) = diag(M_r, I) and K = L M, X = K K' are exactly the rank-r results.
__global__ void async_pad_kernel(int *piv, const int *rk_final, int s) {
  const int r = *rk_final;
  for (int i = r + blockIdx.x * blockDim.x + threadIdx.x; i < s; i += gridDim.x * blockDim.x) piv[i] = s;
}
__global__ void identity_tail_kernel(double *B, long long ldb, const int *rk_final, int s) {
  const int r = *rk_final;
  for (int i = r + blockIdx.x * blockDim.x + threadIdx.x; i < s; i += gridDim.x * blockDim.x)
    B[(long long)i * ldb + i] = 1.0;
}
__global__ void async_rank_kernel(int64_t *out, const int *rk_final, const FactorStats *fs, const FactorStats *fs2) {
  const int r = *rk_final;
  *out = (fs->flags & 1)                   ? -(int64_t)GENINV_ENONFINITE
         : ((fs->flags | fs2->flags) & 4)   ? -(int64_t)GENINV_ERANGE
         : (r > 0 && (fs2->flags & 2))      ? -(int64_t)GENINV_ENOTSPD
                                            : r;
}

// Full rank (r = s) evaluated through L^-1 (reading R27); GENINV_FULLRANK_DIRECT=0 forces the general path.
bool fullrank_direct_on() {
  static const bool on = [] {
    const char *e = getenv("GENINV_FULLRANK_DIRECT");
    return !(e && atoi(e) == 0);
  }();
  return on;
}

// a4-a6 after the factorisation: K = L M (s x r) and, if want_x, X (s x s, full) = K K' = L M M L'.
// rk_pad (device, optional): r is the full size s and the detected rank is *rk_pad (see above).
geninv_status build_x(geninv_handle h, int s, int r, bool want_x = true, const int *rk_pad = nullptr) {
  const long long ld = h->ld;
  if (r == 0) {
    GI_TRY(cudaMemsetAsync(h->X, 0, (size_t)s * ld * sizeof(double), h->st));
    return GENINV_OK;
  }
  if (r == s && want_x && !rk_pad && fullrank_direct_on()) {
    // Every column kept: L is square lower triangular with a positive diagonal, so M = inv(L'L) = L^-1 L^-T
    // exactly, K = L M = L^-T and X = K K' = L^-T L^-1 (P:137-139 with the products collapsed, R27): one
    // TRTRI of L and one LAUUM instead of L'L, the SPD Cholesky of L'L, its TRTRI and LAUUM, K and X.
    const int r_pad = (r + 31) / 32 * 32;
    if (r_pad > s) GI_TRY(cudaMemsetAsync(h->L + (long long)s * ld, 0, (size_t)(r_pad - s) * ld * sizeof(double), h->st));
    GI_TRY(cudaMemsetAsync(h->Ci, 0, (size_t)r_pad * ld * sizeof(double), h->st));
    GI_TRY(cudaMemsetAsync(h->fs2, 0, sizeof(FactorStats), h->st));   // no SPD factorisation: no flags
    GI_TRY(trtri_lower(h->L, ld, r, h->Ci, ld, h->T, h->part, (long long)(h->part_bytes / sizeof(double)), h->st));
    GI_TRYS(gemm_chain(h, op_lauum(h, r, h->X, ld)));                  // X = Ci' Ci
    h->launches += 3 + trtri_launches(r, ld, ld, (long long)(h->part_bytes / sizeof(double)));
    return GENINV_OK;
  }
  GI_TRYS(gemm_chain(h, op_ltl(h, s, r)));
  if (rk_pad) {
    identity_tail_kernel<<<(s + 255) / 256, 256, 0, h->st>>>(h->Bm, ld, rk_pad, s);
    GI_TRY(cudaGetLastError());
    h->launches += 1;
  }
  // a5
  GI_TRYS(spd_inverse(h, h->Bm, r, ld, h->Mm, ld));
  GI_TRYS(gemm_chain(h, op_k(h, s, r)));
  if (!want_x) return GENINV_OK;
  GI_TRYS(gemm_chain(h, op_x(h, s, r)));
  return GENINV_OK;
}

// Order switch: G+ = K (K' G') / (G' K) K' costs 4 r s ell flops against
// s(s+1) r + 2 s^2 ell for X = K K' then X G'; the K order wins for low rank (roughly r < s/2).
bool k_order_cheaper(long long s, long long ell, long long r) {
  return r > 0 && 4.0 * r * s * ell < (double)s * (s + 1) * r + 2.0 * s * s * ell;
}

// a7 in the K order, in chunks of the long side through the handle's s x s scratch T:
//   N: T (r x c) = K' G[j0:j0+c]',  G+[:, j0:j0+c] = K T;   T: T (c x r) = G[:, i0:i0+c]' K,  G+[i0:i0+c, :] = T K'
geninv_status apply_k(geninv_handle h, const double *G, long long m, long long n, long long ld, int trans,
                      double *Gp, long long ldp, int r) {
  Range rg("geninv a7 output (K order)");
  const long long s = trans ? m : n, ell = trans ? n : m;
  const long long cap = (long long)h->ld * h->ld;   // doubles of the scratch T
  const int rp = (r + 1) / 2 * 2;
  // chunk width: T holds r x c (N) or c x rp (T) doubles, so c <= cap / rp; whole 128-wide tiles when that
  // allows, else even (the T view's leading dimension), at least 2 (cap >= 32 * 32 and rp <= s <= ld)
  long long c = std::min<long long>((ell + 1) / 2 * 2, cap / rp);
  c = c >= 128 ? c / 128 * 128 : std::max<long long>(2, c / 2 * 2);
  for (long long c0 = 0; c0 < ell; c0 += c) {
    const long long w = std::min(c, ell - c0);   // c even: the T view has an even leading dimension
    GemmOp a, b;
    if (!trans) {
      a.A = Mat{h->Kb, h->ld, s, r};       // A(q, i) = K[i][q]  (MN-major)
      a.a_kmajor = false;
      a.B = Mat{G + c0 * ld, ld, w, n};    // B(i, j) = G[c0 + j][i]  (K-major)
      a.b_kmajor = true;
      a.M = r; a.N = (int)w; a.K = (int)s;
      a.C = h->T; a.ldc = c;
      b.A = Mat{h->Kb, h->ld, s, r};       // A(i, q) = K[i][q]
      b.a_kmajor = true;
      b.B = Mat{h->T, c, r, c};            // B(q, j) = T[q][j]  (MN-major)
      b.b_kmajor = false;
      b.M = (int)s; b.N = (int)w; b.K = r;
      b.C = Gp + c0; b.ldc = ldp;
    } else {
      a.A = Mat{G, ld, m, n};              // A(i, j) = G[j][c0 + i]  (MN-major)
      a.a_kmajor = false;
      a.a_mn0 = (int)c0;
      a.B = Mat{h->Kb, h->ld, s, r};       // B(j, q) = K[j][q]  (MN-major)
      a.b_kmajor = false;
      a.M = (int)w; a.N = r; a.K = (int)s;
      a.C = h->T; a.ldc = rp;
      b.A = Mat{h->T, rp, w, r};           // A(i, q) = T[i][q]
      b.a_kmajor = true;
      b.B = Mat{h->Kb, h->ld, s, r};       // B(q, j) = K[j][q]  (K-major)
      b.b_kmajor = true;
      b.M = (int)w; b.N = (int)s; b.K = r;
      b.C = Gp + c0 * ldp; b.ldc = ldp;
    }
    GI_TRY(gemm(a, h->st));
    GI_TRY(gemm(b, h->st));
    h->launches += 2;
  }
  return GENINV_OK;
}

// a7: Gp = X G' (trans 0: Gp is n x m) or G' X (trans 1: Gp is n x m).
// a7 on the INT8 tensor cores: N branch Gp (s x m) = X G', T branch Gp (n x m) = G' X, over K = s in
// exact int32 passes of EMU_K (each pass has its own per-line exponents, the passes add up in FP64).
// The digit planes of X for every pass are made once; G is taken in chunks of its long side (rows
// for N, columns for T: those are the lines of G' X).  Returns GENINV_ERANGE (nothing usable written)
// for a line outside the exact-scaling range or with NaN / Inf; the caller then uses DMMA.
geninv_status apply_emulated(geninv_handle h, const double *G, long long m, long long n, long long ld, int trans,
                             double *Gp, long long ldp, cudaStream_t st) {
  const int T = emu_groups();
  constexpr int S = EMU_S;
  const int s = (int)(trans ? m : n);
  const long long ell = trans ? n : m;
  const int npass = (s + EMU_K - 1) / EMU_K;
  long long xplanes = 0;   // bytes of X's digit planes over all passes
  for (int p = 0; p < npass; ++p) xplanes += (long long)S * s * emu_kpad(std::min(EMU_K, s - p * EMU_K));
  const int Kp1 = emu_kpad(std::min(EMU_K, s));
  const long long chunk =
      std::max<long long>(256, std::min<long long>(ell, (2LL << 30) / ((long long)S * Kp1)) / 256 * 256);
  const long long cmax = std::min<long long>(chunk, ell);
  GI_TRYS(grow(h->emu_x, h->emu_x_bytes, (size_t)xplanes));
  GI_TRYS(grow(h->emu_ex, h->emu_ex_n, (size_t)s * npass));
  GI_TRYS(grow(h->emu_g, h->emu_g_bytes, (size_t)S * cmax * Kp1));
  GI_TRYS(grow(h->emu_eg, h->emu_eg_n, (size_t)cmax));
  GI_TRYS(grow(h->emu_cm, h->emu_cm_n, (size_t)cmax));
  GI_TRYS(grow(h->emu_sc, h->emu_sc_n,
               (size_t)std::max(emu_scratch_elems(s, (int)cmax), emu_scratch_elems((int)cmax, s))));
  if (!h->emu_flag) GI_TRY(cudaMalloc(&h->emu_flag, sizeof(int)));
  GI_TRY(cudaMemsetAsync(h->emu_flag, 0, sizeof(int), st));
  std::vector<long long> xoff(npass + 1, 0);
  for (int p = 0; p < npass; ++p) {
    const int k0 = p * EMU_K, kw = std::min(EMU_K, s - k0);
    xoff[p + 1] = xoff[p] + (long long)S * s * emu_kpad(kw);
    GI_TRY(emu_split(h->X + k0, h->ld, s, kw, S, h->emu_x + xoff[p], h->emu_ex + (long long)p * s, h->emu_flag, st));
    h->launches += 1;
  }
  for (long long j0 = 0; j0 < ell; j0 += chunk) {
    const int nc = (int)std::min<long long>(chunk, ell - j0);
    for (int p = 0; p < npass; ++p) {
      const int k0 = p * EMU_K, kw = std::min(EMU_K, s - k0);
      const int8_t *xs = h->emu_x + xoff[p];
      const int *xe = h->emu_ex + (long long)p * s;
      if (!trans) {   // lines of G = its rows j0 .., K columns k0 ..;  C[i][j] = sum_k X[i][k] G[j][k]
        GI_TRY(emu_split(G + j0 * ld + k0, ld, nc, kw, S, h->emu_g, h->emu_eg, h->emu_flag, st));
        GI_TRY(emu_gemm_nt(xs, xe, s, h->emu_g, h->emu_eg, nc, kw, S, T, Gp + j0, ldp, h->emu_sc, st, 0, p > 0));
        h->launches += 2;
      } else {        // lines of G' = columns j0 .. of G, K rows k0 ..;  C[i][j] = sum_k G[k][i] X[j][k]
        GI_TRY(emu_split_cols(G + (long long)k0 * ld + j0, ld, kw, nc, S, h->emu_g, h->emu_eg, h->emu_cm, h->emu_flag,
                              st));
        GI_TRY(emu_gemm_nt(h->emu_g, h->emu_eg, nc, xs, xe, s, kw, S, T, Gp + j0 * ldp, ldp, h->emu_sc, st, 0, p > 0));
        h->launches += 3;
      }
    }
  }
  int flag = 0;
  GI_TRY(cudaMemcpyAsync(&flag, h->emu_flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  GI_TRY(cudaStreamSynchronize(st));
  return flag ? GENINV_ERANGE : GENINV_OK;
}

geninv_status apply(geninv_handle h, const double *G, long long m, long long n, long long ld, int trans, double *Gp,
                    long long ldp, cudaStream_t st) {
  Range rg("geninv a7 output");
  const long long s = trans ? m : n;
  if (emulation_on(h) && s <= 16384) {
    const geninv_status es = apply_emulated(h, G, m, n, ld, trans, Gp, ldp, st);
    if (es != GENINV_ERANGE) return es;   // out of the emulation's range: the native product below
  }
  GemmOp op;
  if (!trans) {
    // Gp[i][j] = sum_k X[i][k] G[j][k],  i < n = s, j < m
    op.A = Mat{h->X, h->ld, s, s};
    op.a_kmajor = true;
    op.B = Mat{G, ld, m, n};
    op.b_kmajor = true;
    op.M = (int)s;
    op.N = (int)m;
  } else {
    // Gp[i][j] = sum_k G[k][i] X[k][j] = sum_k G[k][i] X[j][k],  i < n, j < m = s
    op.A = Mat{G, ld, m, n};
    op.a_kmajor = false;
    op.B = Mat{h->X, h->ld, s, s};
    op.b_kmajor = true;
    op.M = (int)n;
    op.N = (int)s;
  }
  op.K = (int)s;
  op.C = Gp;
  op.ldc = ldp;
  GI_TRY(gemm(op, st));
  h->launches += 1;
  return GENINV_OK;
}

// s: the factored size (0: unknown).  not_psd_hint: a tentative pivot below -s * tol (SPEC S:138's
// definiteness rule) -- the paper drops it like any other pivot <= tol (reading R3), so it is
// reported, not an error: a Gram matrix G'G never produces one beyond rounding, a user-supplied A that is
// not positive semidefinite does.
void fill_info(geninv_info *info, const FactorStats &fs, int r, int tr, geninv_status st, long long s = 0) {
  if (!info) return;
  info->tol = fs.tol;
  info->rank = r;
  info->transposed = tr;
  info->status = st;
  info->min_acc = fs.min_acc;
  info->max_drop = fs.max_drop;
  info->min_pivot = fs.min_pivot;
  info->order = 0;
  info->not_psd_hint = (s > 0 && fs.tol > 0 && fs.min_pivot < -(double)s * fs.tol) ? 1 : 0;
}

geninv_status check_g(const double *G, long long m, long long n, long long ld) {
  if (!G || m < 1 || n < 1 || ld < n) return GENINV_EINVAL;
  if (m > 0x7fffffffLL || n > 0x7fffffffLL) return GENINV_EINVAL;
  return GENINV_OK;
}

// An operand the TMA path cannot read in place (base not 16-byte aligned, or an odd leading dimension:
// tensor-map strides are multiples of 16 bytes) is copied once, on the handle's stream, into a handle-owned
// buffer with the leading dimension rounded up to even; X (rows x cols, ld) is redirected to the copy.
// slot 0: G, slot 1: the right-hand sides F of geninv_solve_d.  Costs rows x cols doubles of device memory
// and one device-to-device copy; aligned operands are used in place.
geninv_status stage_operand(geninv_handle h, int slot, const double *&X, long long rows, long long cols,
                            long long &ld) {
  if (aligned16(X) && !(ld & 1)) return GENINV_OK;
  const long long lds = (cols + 1) / 2 * 2;
  const size_t need = (size_t)rows * lds * sizeof(double);
  if (need > h->stage_bytes[slot]) {
    cudaStreamSynchronize(h->st);
    if (h->stage[slot]) cudaFree(h->stage[slot]);
    h->stage[slot] = nullptr;
    h->stage_bytes[slot] = 0;
    GI_TRY(cudaMalloc(&h->stage[slot], need));
    h->stage_bytes[slot] = need;
  }
  GI_TRY(cudaMemcpy2DAsync(h->stage[slot], lds * 8, X, ld * 8, cols * 8, rows, cudaMemcpyDeviceToDevice, h->st));
  X = h->stage[slot];
  ld = lds;
  return GENINV_OK;
}

// Steps a2-a6 on A (s x s lower, lda); leaves X in the handle -- or, when ell > 0 and the K order
// is cheaper for this rank (f4), only K (*k_order = true, X not formed).
geninv_status from_gram(geninv_handle h, const double *A, int s, long long lda, const geninv_opts *opts, int *r_out,
                        FactorStats *fs, long long ell = 0, bool *k_order = nullptr) {
  GI_TRYS(ensure_ws(h, s));
  int r = 0;
  geninv_status st = factor(h, A, lda, s, h->L, h->ld, h->piv, opts, &r, fs);
  if (st != GENINV_OK) return st;
  const bool ko = ell > 0 && k_order && k_order_cheaper(s, ell, r);
  if (k_order) *k_order = ko;
  // a4-a6 (L'L, the SPD inverse's panel chain, TRTRI, the products) as one CUDA graph per (s, r)
  GI_TRYS(prepare_chain(h, s, r, !ko));
  Range rg("geninv a4-a6 L'L, inverse, K, X");
  const long long key[10] = {s, r, ko ? 0 : 1, h->ld, (long long)(uintptr_t)h->L, 2, (long long)(uintptr_t)h->part,
                             0, 0, 0};
  GI_TRYS(run_graph(h, h->g_build, key, [&](cudaStream_t st) -> geninv_status {
    cudaStream_t saved = h->st;
    h->st = st;
    const geninv_status rs = build_x(h, s, r, !ko);
    h->st = saved;
    return rs;
  }));
  h->x_s = ko ? -1 : s;
  h->last_rank = r;
  *r_out = r;
  return GENINV_OK;
}

geninv_status finish_spd_check(geninv_handle h, int r) {
  if (r == 0) return GENINV_OK;
  int flags = 0;
  GI_TRY(cudaMemcpyAsync(&flags, &h->fs2->flags, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  GI_TRY(cudaStreamSynchronize(h->st));
  return (flags & 2) ? GENINV_ENOTSPD : (flags & 4) ? GENINV_ERANGE : GENINV_OK;
}

bool is_small(long long m, long long n) { return std::min(m, n) <= 64 && std::max(m, n) <= 128; }

// Small matrix (C1, the paper's n = 32 / 64): the whole path in one CTA -- the batched kernel with
// batch = 1, one launch instead of ~20 latency-bound ones.  Synchronises; X is not kept.
geninv_status small_path(geninv_handle h, const double *G, long long m, long long n, long long ld, double *Gp,
                         long long ldp, const geninv_opts *opts, int *r_out, FactorStats *fs) {
  GI_TRYS(ensure_ws(h, 64));
  // the rank goes to the stats record's spare int, so one copy returns both
  GI_TRY(batched_geninv(G, (int)m, (int)n, ld, 0, 1, Gp, ldp, 0, &h->fs->pad, tol_rel_of(opts), tol_abs_of(opts),
                        h->st, h->fs));
  h->launches += 1;
  GI_TRY(cudaMemcpyAsync(fs, h->fs, sizeof(FactorStats), cudaMemcpyDeviceToHost, h->st));
  GI_TRY(cudaStreamSynchronize(h->st));
  const int rr = fs->pad;
  h->x_s = -1;
  *r_out = rr < 0 ? 0 : rr;
  return rr == -2 ? GENINV_ENONFINITE : rr == -3 ? GENINV_ENOTSPD : rr == -9 ? GENINV_ERANGE : GENINV_OK;
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

geninv_status geninv_create(geninv_handle *out, int device) {
  if (!out) return GENINV_EINVAL;
  auto *h = new geninv_handle_s();
  h->device = device;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->st2, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->upd, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->upd2, cudaStreamNonBlocking);
  for (int i = 0; i < 4 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&h->ev[i], cudaEventDisableTiming);
  for (int i = 0; i < 8 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&h->ev_fr[i], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&h->ev_g[i], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete h;
    return cuda_status(e);
  }
  h->st = h->own;
  *out = h;
  return GENINV_OK;
}

geninv_status geninv_set_stream(geninv_handle h, void *stream) {
  if (!h) return GENINV_EINVAL;
  h->st = static_cast<cudaStream_t>(stream);  // NULL = the legacy default stream
  return GENINV_OK;
}

geninv_status geninv_set_emulation(geninv_handle h, int mode) {
  if (!h || mode < 0 || mode > 1) return GENINV_EINVAL;
  h->emulate = mode;
  return GENINV_OK;
}

geninv_status geninv_destroy(geninv_handle h) {
  if (!h) return GENINV_EINVAL;
  cudaSetDevice(h->device);
  cudaStreamSynchronize(h->st);
  free_ws(h);
  if (h->part) cudaFree(h->part);
  if (h->Gdev) cudaFree(h->Gdev);
  if (h->T1) cudaFree(h->T1);
  for (auto &b : h->stage)
    if (b) cudaFree(b);
  if (h->coll) cudaFree(h->coll);
  for (void *p : {(void *)h->emu_x, (void *)h->emu_g, (void *)h->emu_ex, (void *)h->emu_eg, (void *)h->emu_flag,
                  (void *)h->emu_sc, (void *)h->emu_cm})
    if (p) cudaFree(p);
  for (auto &c : h->Gpchunk)
    if (c) cudaFree(c);
  for (auto &ev : h->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto &ev : h->ev_fr)
    if (ev) cudaEventDestroy(ev);
  if (h->upd) cudaStreamDestroy(h->upd);
  if (h->upd2) cudaStreamDestroy(h->upd2);
  if (h->g_factor.exec) cudaGraphExecDestroy(h->g_factor.exec);
  if (h->g_build.exec) cudaGraphExecDestroy(h->g_build.exec);
  if (h->g_async.exec) cudaGraphExecDestroy(h->g_async.exec);
  for (auto &ev : h->ev_g)
    if (ev) cudaEventDestroy(ev);
  if (h->gstream) cudaStreamDestroy(h->gstream);
  if (h->st2) cudaStreamDestroy(h->st2);
  if (h->own) cudaStreamDestroy(h->own);
  delete h;
  return GENINV_OK;
}

const char *geninv_strerror(geninv_status st) {
  switch (st) {
    case GENINV_OK: return "ok";
    case GENINV_EINVAL: return "invalid argument";
    case GENINV_ENONFINITE: return "non-finite entry in G (non-finite Gram diagonal)";
    case GENINV_ENOTSPD: return "L'L is not numerically SPD (pivot <= 0 in its Cholesky)";
    case GENINV_ECUDA: return "CUDA error";
    case GENINV_ENOMEM: return "device out of memory";
    case GENINV_EALIGN: return "reserved (alignment is handled by staging; not returned)";
    case GENINV_ESTATE: return "no factorisation of matching size in the handle";
    case GENINV_ENCCL: return "NCCL unavailable or the all-reduce failed";
    case GENINV_ERANGE: return "an accepted pivot is subnormal (|G| too small): scale G by a power of two";
  }
  return "unknown status";
}

geninv_status geninv_d(geninv_handle h, const double *G, int64_t m, int64_t n, int64_t ld, double *Gp, int64_t ldp,
                       int64_t *rank, const geninv_opts *opts, geninv_info *info) {
  Range rg_call("geninv_d");
  if (!h || !Gp || ldp < m) return GENINV_EINVAL;
  GI_TRYS(check_g(G, m, n, ld));
  cudaSetDevice(h->device);
  const int tr = m < n;  // P:109 (strict; m == n takes the N branch, R6)
  const int s = (int)(tr ? m : n);
  GI_TRYS(ensure_ws(h, s));
  if (is_small(m, n)) {   // the one-CTA path reads G with 8-byte loads when needed: any alignment / ld
    int r = 0;
    FactorStats fs{};
    geninv_status st = small_path(h, G, m, n, ld, Gp, ldp, opts, &r, &fs);
    if (rank) *rank = r;
    fill_info(info, fs, r, tr, st, s);
    return st;
  }
  long long ldg = ld;
  GI_TRYS(stage_operand(h, 0, G, m, n, ldg));
  ld = ldg;
  GI_TRYS(gram(h, G, m, n, ld, tr, h->A, h->ld));
  int r = 0;
  FactorStats fs{};
  bool ko = false;
  geninv_status st = from_gram(h, h->A, s, h->ld, opts, &r, &fs, tr ? n : m, &ko);
  if (st == GENINV_OK) st = ko ? apply_k(h, G, m, n, ld, tr, Gp, ldp, r) : apply(h, G, m, n, ld, tr, Gp, ldp, h->st);
  if (st == GENINV_OK) st = finish_spd_check(h, r);
  if (st == GENINV_OK) {
    cudaError_t e = cudaStreamSynchronize(h->st);
    if (e != cudaSuccess) st = cuda_status(e);
  }
  if (rank) *rank = r;
  fill_info(info, fs, r, tr, st, s);
  if (info) info->order = ko ? 1 : 0;
  return st;
}

geninv_status geninv_d_async(geninv_handle h, const double *G, int64_t m, int64_t n, int64_t ld, double *Gp,
                             int64_t ldp, int64_t *rank_dev, const geninv_opts *opts) {
  Range rg_call("geninv_d_async");
  if (!h || !Gp || !rank_dev || ldp < m) return GENINV_EINVAL;
  GI_TRYS(check_g(G, m, n, ld));
  cudaSetDevice(h->device);
  const int tr = m < n;
  const int s = (int)(tr ? m : n);
  GI_TRYS(ensure_ws(h, s));
  {
    long long ldg = ld;
    GI_TRYS(stage_operand(h, 0, G, m, n, ldg));
    ld = ldg;
  }
  GI_TRYS(gram(h, G, m, n, ld, tr, h->A, h->ld));
  const int np = (s + PB - 1) / PB;
  const int *rk_final = h->rk + np;
  GI_TRYS(prepare_chain(h, s, s, true));
  const long long key[10] = {s, h->ld, (long long)(uintptr_t)h->A, dbits(tol_rel_of(opts)), dbits(tol_abs_of(opts)),
                             (long long)(uintptr_t)rank_dev, 3, (long long)(uintptr_t)h->part, 0, 0};
  GI_TRYS(run_graph(h, h->g_async, key, [&](cudaStream_t st) -> geninv_status {
    cudaStream_t saved = h->st;
    h->st = st;
    geninv_status rs = GENINV_OK;
    do {
      cudaError_t e = tolerance(h->A, h->ld, s, tol_rel_of(opts), tol_abs_of(opts), h->fs, st);
      if (e == cudaSuccess) e = cudaMemsetAsync(h->L, 0, (size_t)s * h->ld * sizeof(double), st);
      if (e == cudaSuccess)
        e = frchol(h->A, h->ld, s, h->L, h->ld, h->piv, h->rk, h->fs, 0, h->Wp, h->wp_elems, st, h->upd, h->upd2, h->ev_fr);
      if (e == cudaSuccess) {
        async_pad_kernel<<<(s + 255) / 256, 256, 0, st>>>(h->piv, rk_final, s);
        e = cudaGetLastError();
      }
      if (e != cudaSuccess) { rs = cuda_status(e); break; }
      h->launches += 2 + frchol_launches(s);
      rs = build_x(h, s, s, true, rk_final);
      if (rs != GENINV_OK) break;
      async_rank_kernel<<<1, 1, 0, st>>>(rank_dev, rk_final, h->fs, h->fs2);
      if ((e = cudaGetLastError()) != cudaSuccess) rs = cuda_status(e);
      h->launches += 1;
    } while (0);
    h->st = saved;
    return rs;
  }));
  h->x_s = s;
  return apply(h, G, m, n, ld, tr, Gp, ldp, h->st);
}

geninv_status geninv_host_d(geninv_handle h, const double *G_host, int64_t m, int64_t n, int64_t ld, double *Gp_host,
                            int64_t ldp, int64_t *rank, const geninv_opts *opts, geninv_info *info) {
  Range rg_call("geninv_host_d");
  if (!h || !G_host || !Gp_host || m < 1 || n < 1 || ld < n || ldp < m) return GENINV_EINVAL;
  cudaSetDevice(h->device);
  const int tr = m < n;
  const int s = (int)(tr ? m : n);
  if (is_small(m, n)) {   // one H2D, the one-CTA path, one D2H
    const size_t gb = (size_t)m * n * sizeof(double), pb = (size_t)n * m * sizeof(double);
    if (gb > h->gdev_bytes) {
      if (h->Gdev) cudaFree(h->Gdev);
      h->Gdev = nullptr;
      h->gdev_bytes = 0;
      GI_TRY(cudaMalloc(&h->Gdev, gb));
      h->gdev_bytes = gb;
    }
    if (pb > h->chunk_bytes) {
      for (auto &c : h->Gpchunk) {
        if (c) cudaFree(c);
        c = nullptr;
      }
      h->chunk_bytes = 0;
      for (auto &c : h->Gpchunk) GI_TRY(cudaMalloc(&c, pb));
      h->chunk_bytes = pb;
    }
    GI_TRY(cudaMemcpy2DAsync(h->Gdev, n * 8, G_host, ld * 8, n * 8, m, cudaMemcpyHostToDevice, h->st));
    int r = 0;
    FactorStats fs{};
    geninv_status st = small_path(h, h->Gdev, m, n, n, h->Gpchunk[0], m, opts, &r, &fs);
    if (st == GENINV_OK || st == GENINV_ENOTSPD || st == GENINV_ENONFINITE) {
      GI_TRY(cudaMemcpy2DAsync(Gp_host, ldp * 8, h->Gpchunk[0], m * 8, m * 8, n, cudaMemcpyDeviceToHost, h->st));
      GI_TRY(cudaStreamSynchronize(h->st));
    }
    if (rank) *rank = r;
    fill_info(info, fs, r, tr, st, s);
    return st;
  }
  const long long ldg = (n + 1) / 2 * 2;  // device copy: even leading dimension
  const size_t gbytes = (size_t)m * ldg * sizeof(double);
  if (gbytes > h->gdev_bytes) {
    if (h->Gdev) cudaFree(h->Gdev);
    h->Gdev = nullptr;
    h->gdev_bytes = 0;
    GI_TRY(cudaMalloc(&h->Gdev, gbytes));
    h->gdev_bytes = gbytes;
  }
  GI_TRYS(ensure_ws(h, s));
  // ---- H2D in chunks of ~1/8 of G (64 .. 256 MB; C3 / C3T e2e: 32 MB chunks 38.9 ms, 64 MB 36.5,
  //      128 MB 37.4), the Gram of each chunk accumulated as soon as it
  //      lands: N branch row chunks (A = sum_c G_c' G_c), T branch column chunks (A = sum_c G_c G_c'),
  //      summed in chunk order (deterministic)
  static const long long chunk_mb = [] {   // tuning override of the chunk size (MB)
    const char *e = getenv("GENINV_HOST_CHUNK_MB");
    return e ? atoll(e) : 0LL;
  }();
  const long long target = chunk_mb > 0 ? (chunk_mb << 20)
                                        : std::min<long long>(256LL << 20, std::max<long long>(64LL << 20, (long long)gbytes / 8));
  if (!tr) {
    const long long rows_per = std::max<long long>(1, target / (ldg * 8));
    for (long long r0 = 0; r0 < m; r0 += rows_per) {
      const long long rows = std::min(rows_per, m - r0);
      GI_TRY(cudaMemcpy2DAsync(h->Gdev + r0 * ldg, ldg * 8, G_host + r0 * ld, ld * 8, n * 8, rows,
                               cudaMemcpyHostToDevice, h->st2));
      GI_TRY(cudaEventRecord(h->ev[0], h->st2));
      GI_TRY(cudaStreamWaitEvent(h->st, h->ev[0], 0));
      GI_TRYS(gram(h, h->Gdev + r0 * ldg, rows, n, ldg, 0, h->A, h->ld, r0 == 0 ? nullptr : h->A));
    }
  } else {
    const long long cols_per = std::max<long long>(16, target / (m * 8) / 16 * 16);
    for (long long c0 = 0; c0 < n; c0 += cols_per) {
      const long long cols = std::min(cols_per, n - c0);
      GI_TRY(cudaMemcpy2DAsync(h->Gdev + c0, ldg * 8, G_host + c0, ld * 8, cols * 8, m, cudaMemcpyHostToDevice,
                               h->st2));
      GI_TRY(cudaEventRecord(h->ev[0], h->st2));
      GI_TRY(cudaStreamWaitEvent(h->st, h->ev[0], 0));
      GI_TRYS(gram(h, h->Gdev + c0, m, cols, ldg, 1, h->A, h->ld, c0 == 0 ? nullptr : h->A));
    }
  }
  int r = 0;
  FactorStats fs{};
  geninv_status st = from_gram(h, h->A, s, h->ld, opts, &r, &fs);
  if (st == GENINV_OK) st = finish_spd_check(h, r);
  if (st != GENINV_OK) {
    fill_info(info, fs, r, tr, st, s);
    return st;
  }
  // ---- output in chunks, D2H of chunk c overlapped with the product of chunk c + 1
  //      N: column block j0..j1 of G+ (n x m) = X G[j0:j1]';  T: row block of G+ = G[:, i0:i1]' X
  // chunk width: a multiple of 16 (even leading dimension of the G+ chunk; 16-aligned TMA strips)
  long long cw = std::max<long long>(16, (tr ? target / (m * 8) : target / (ldg * 8)) / 16 * 16);
  {
    // round the chunk to whole 128-wide tiles with the best last-wave fill of its (s / 128) x (cw / 128)
    // output tiles (C3: 1024 -> 1152 columns, 1.73 -> 1.95 waves), within [cw / 2, 2 cw]
    const long long mt = (s + 127) / 128, sms = num_sms(), nt0 = std::max<long long>(1, cw / 128);
    double best = -1.0;
    long long bnt = nt0;
    for (long long nt = std::max<long long>(1, nt0 / 2); nt <= 2 * nt0; ++nt) {
      const long long t = mt * nt, waves = (t + sms - 1) / sms;
      const double fill = (double)t / (double)(waves * sms) - 0.002 * std::llabs(nt - nt0) / nt0;
      if (fill > best) { best = fill; bnt = nt; }
    }
    if (cw >= 128) cw = bnt * 128;
  }
  const long long total = tr ? n : m;
  const size_t cbytes = (size_t)cw * (s + 1) * sizeof(double) + 256;
  if (cbytes > h->chunk_bytes) {
    for (auto &c : h->Gpchunk) {
      if (c) cudaFree(c);
      c = nullptr;
    }
    h->chunk_bytes = 0;
    for (auto &c : h->Gpchunk) GI_TRY(cudaMalloc(&c, cbytes));
    h->chunk_bytes = cbytes;
  }
  int buf = 0;
  bool pending[2] = {false, false};
  for (long long c0 = 0; c0 < total; c0 += cw, buf ^= 1) {
    const long long w = std::min(cw, total - c0);
    if (pending[buf]) GI_TRY(cudaStreamWaitEvent(h->st, h->ev[2 + buf], 0));  // chunk buffer free again
    double *dst = h->Gpchunk[buf];
    if (!tr) {
      // chunk (s x w, ld wpad) = X G[c0:c0+w]'
      const long long wpad = (w + 1) / 2 * 2;
      GI_TRYS(apply(h, h->Gdev + c0 * ldg, w, n, ldg, 0, dst, wpad, h->st));
      GI_TRY(cudaEventRecord(h->ev[0], h->st));
      GI_TRY(cudaStreamWaitEvent(h->st2, h->ev[0], 0));
      GI_TRY(cudaMemcpy2DAsync(Gp_host + c0, ldp * 8, dst, wpad * 8, w * 8, s, cudaMemcpyDeviceToHost, h->st2));
    } else {
      // chunk (w x s, ld s) = G[:, c0:c0+w]' X : A-op is the column block of G (m x w)
      GemmOp op;
      op.A = Mat{h->Gdev, ldg, m, n};
      op.a_kmajor = false;
      op.a_mn0 = (int)c0;
      op.B = Mat{h->X, h->ld, s, s};
      op.b_kmajor = true;
      op.M = (int)w;
      op.N = s;
      op.K = s;
      op.C = dst;
      op.ldc = s;
      GI_TRY(gemm(op, h->st));
      h->launches += 1;
      GI_TRY(cudaEventRecord(h->ev[0], h->st));
      GI_TRY(cudaStreamWaitEvent(h->st2, h->ev[0], 0));
      GI_TRY(cudaMemcpy2DAsync(Gp_host + c0 * ldp, ldp * 8, dst, (size_t)s * 8, (size_t)s * 8, w,
                               cudaMemcpyDeviceToHost, h->st2));
    }
    GI_TRY(cudaEventRecord(h->ev[2 + buf], h->st2));
    pending[buf] = true;
  }
  GI_TRY(cudaStreamSynchronize(h->st2));
  GI_TRY(cudaStreamSynchronize(h->st));
  if (rank) *rank = r;
  fill_info(info, fs, r, tr, GENINV_OK, s);
  return GENINV_OK;
}

geninv_status geninv_batched_d(geninv_handle h, const double *G, int64_t m, int64_t n, int64_t ld, int64_t strideG,
                               int64_t batch, double *Gp, int64_t ldp, int64_t strideGp, int32_t *rank_dev,
                               const geninv_opts *opts) {
  Range rg_call("geninv_batched_d");
  if (!h || batch < 0 || m < 1 || n < 1 || ld < n || ldp < m) return GENINV_EINVAL;
  if (batch == 0) return GENINV_OK;
  if (!G || !Gp || !rank_dev) return GENINV_EINVAL;
  if (std::min(m, n) > 64 || std::max(m, n) > 128) return GENINV_EINVAL;
  cudaSetDevice(h->device);
  GI_TRY(batched_geninv(G, (int)m, (int)n, ld, strideG, batch, Gp, ldp, strideGp, rank_dev, tol_rel_of(opts),
                        tol_abs_of(opts), h->st));
  h->launches += 1;
  return GENINV_OK;
}

// ---- NCCL, resolved at run time (the library itself does not link NCCL): the communicator comes
//      from the caller (e.g. torch's ProcessGroupNCCL), so the already-loaded libnccl is reused.
typedef int (*nccl_allreduce_fn)(const void *, void *, size_t, int, int, void *, cudaStream_t);
static nccl_allreduce_fn nccl_allreduce() {
  static nccl_allreduce_fn fn = [] {
    void *lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!lib) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    return lib ? reinterpret_cast<nccl_allreduce_fn>(dlsym(lib, "ncclAllReduce")) : nullptr;
  }();
  return fn;
}

geninv_status geninv_sharded_d(geninv_handle h, void *nccl_comm, const double *G_local, int64_t m_local, int64_t n,
                               int64_t ld, int32_t trans, double *Gp_local, int64_t ldp, int64_t *rank,
                               const geninv_opts *opts, geninv_info *info) {
  Range rg_call("geninv_sharded_d");
  if (!h || !nccl_comm) return GENINV_EINVAL;
  nccl_allreduce_fn ar = nccl_allreduce();
  if (!ar) return GENINV_ENCCL;   // no communication possible at all (the same library on every rank)
  cudaSetDevice(h->device);
  if (!h->coll) GI_TRY(cudaMalloc(&h->coll, 4 * sizeof(double)));
  // Local checks and the local Gram first; then every rank takes part in one small MAX all-reduce of
  // (status, s, -s) before the big one, so a rank that failed locally (bad arguments, ENOMEM, a CUDA
  // error) or a shape that differs between ranks makes ALL ranks return the error instead of leaving
  // the others blocked in the all-reduce of A.
  const long long s = trans ? m_local : n;
  geninv_status st = check_g(G_local, m_local, n, ld);
  if (st == GENINV_OK && (!Gp_local || ldp < (trans ? s : m_local) || s > 0x7fffffffLL)) st = GENINV_EINVAL;
  long long ldg = ld;
  if (st == GENINV_OK) st = ensure_ws(h, (int)s);
  if (st == GENINV_OK) st = stage_operand(h, 0, G_local, m_local, n, ldg);
  if (st == GENINV_OK) {
    // a1 on the local block, into a zeroed A (the all-reduced upper triangle stays exactly zero)
    const cudaError_t e = cudaMemsetAsync(h->A, 0, (size_t)s * h->ld * sizeof(double), h->st);
    st = e == cudaSuccess ? gram(h, G_local, m_local, n, ldg, trans, h->A, h->ld) : cuda_status(e);
  }
  {
    double pre[3] = {(double)st, st == GENINV_OK ? (double)s : 0.0, st == GENINV_OK ? -(double)s : 0.0};
    GI_TRY(cudaMemcpyAsync(h->coll, pre, sizeof(pre), cudaMemcpyHostToDevice, h->st));
    if (ar(h->coll, h->coll, 3, /*ncclFloat64*/ 8, /*ncclMax*/ 2, nccl_comm, h->st) != 0) return GENINV_ENCCL;
    GI_TRY(cudaMemcpyAsync(pre, h->coll, sizeof(pre), cudaMemcpyDeviceToHost, h->st));
    GI_TRY(cudaStreamSynchronize(h->st));
    if (st != GENINV_OK) return st;
    if (pre[0] != 0.0) return (geninv_status)(int)pre[0];   // another rank failed
    if (pre[1] != -pre[2]) return GENINV_EINVAL;             // s differs between ranks
  }
  // a8: A = sum_p A_p -- the one exchange step (NCCL over NVLink / NVSwitch), FP64 sum
  {
    Range rg("geninv a8 all-reduce of A");
    if (ar(h->A, h->A, (size_t)s * h->ld, /*ncclFloat64*/ 8, /*ncclSum*/ 0, nccl_comm, h->st) != 0) return GENINV_ENCCL;
  }
  int r = 0;
  FactorStats fs{};
  st = from_gram(h, h->A, (int)s, h->ld, opts, &r, &fs);   // a2-a6, replicated (deterministic: same r, X)
  if (st == GENINV_OK) st = finish_spd_check(h, r);
  if (st == GENINV_OK) st = apply(h, G_local, m_local, n, ldg, trans, Gp_local, ldp, h->st);   // a7, local block
  if (st == GENINV_OK) {
    cudaError_t e = cudaStreamSynchronize(h->st);
    if (e != cudaSuccess) st = cuda_status(e);
  }
  if (rank) *rank = r;
  fill_info(info, fs, r, trans, st, s);
  return st;
}

geninv_status geninv_solve_d(geninv_handle h, const double *G, int64_t m, int64_t n, int64_t ld, const double *F,
                             int64_t k, int64_t ldf, double *W, int64_t ldw, int64_t *rank, const geninv_opts *opts,
                             geninv_info *info) {
  Range rg_call("geninv_solve_d");
  if (!h || !F || !W || k < 1 || ldf < k || ldw < k) return GENINV_EINVAL;
  GI_TRYS(check_g(G, m, n, ld));
  if (k > 0x7fffffffLL) return GENINV_EINVAL;
  cudaSetDevice(h->device);
  const int tr = m < n;
  const int s = (int)(tr ? m : n);
  GI_TRYS(ensure_ws(h, s));
  {
    long long ldg = ld, ldff = ldf;
    GI_TRYS(stage_operand(h, 0, G, m, n, ldg));
    GI_TRYS(stage_operand(h, 1, F, m, k, ldff));
    ld = ldg;
    ldf = ldff;
  }
  GI_DBG_SYNC("solve: staging");
  GI_TRYS(gram(h, G, m, n, ld, tr, h->A, h->ld));
  GI_DBG_SYNC("solve: gram");
  int r = 0;
  FactorStats fs{};
  geninv_status st = from_gram(h, h->A, s, h->ld, opts, &r, &fs);
  GI_DBG_SYNC("solve: from_gram");
  if (st == GENINV_OK) st = finish_spd_check(h, r);
  if (st != GENINV_OK) {
    if (rank) *rank = r;
    fill_info(info, fs, r, tr, st, s);
    return st;
  }
  const long long ldt = (k + 1) / 2 * 2;
  const size_t tb = (size_t)s * ldt * sizeof(double);
  if (tb > h->t1_bytes) {
    if (h->T1) cudaFree(h->T1);
    h->T1 = nullptr;
    h->t1_bytes = 0;
    GI_TRY(cudaMalloc(&h->T1, tb));
    h->t1_bytes = tb;
  }
  GemmOp a, b;
  if (!tr) {
    // T1 (n x k) = G' F:  T1[i][c] = sum_j G[j][i] F[j][c];   W (n x k) = X T1
    a.A = Mat{G, ld, m, n};
    a.a_kmajor = false;
    a.B = Mat{F, ldf, m, k};
    a.b_kmajor = false;
    a.M = s; a.N = (int)k; a.K = (int)m;
    a.C = h->T1; a.ldc = ldt;
    b.A = Mat{h->X, h->ld, s, s};
    b.a_kmajor = true;
    b.B = Mat{h->T1, ldt, s, k};
    b.b_kmajor = false;
    b.M = s; b.N = (int)k; b.K = s;
    b.C = W; b.ldc = ldw;
  } else {
    // T1 (m x k) = X F;   W (n x k) = G' T1:  W[i][c] = sum_j G[j][i] T1[j][c]
    a.A = Mat{h->X, h->ld, s, s};
    a.a_kmajor = true;
    a.B = Mat{F, ldf, m, k};
    a.b_kmajor = false;
    a.M = s; a.N = (int)k; a.K = s;
    a.C = h->T1; a.ldc = ldt;
    b.A = Mat{G, ld, m, n};
    b.a_kmajor = false;
    b.B = Mat{h->T1, ldt, s, k};
    b.b_kmajor = false;
    b.M = (int)n; b.N = (int)k; b.K = s;
    b.C = W; b.ldc = ldw;
  }
  GI_DBG_SYNC("solve: T1");
  GI_TRYS(gemm_splitk(h, a));
  GI_DBG_SYNC("solve: first product");
  GI_TRYS(gemm_splitk(h, b));
  cudaError_t e = cudaStreamSynchronize(h->st);
  if (e != cudaSuccess) st = cuda_status(e);
  if (rank) *rank = r;
  fill_info(info, fs, r, tr, st, s);
  return st;
}

geninv_status geninv_gram_d(geninv_handle h, const double *G, int64_t m, int64_t n, int64_t ld, int32_t trans,
                            double *A, int64_t lda) {
  if (!h || !A) return GENINV_EINVAL;
  GI_TRYS(check_g(G, m, n, ld));
  const long long s = trans ? m : n;
  if (lda < s) return GENINV_EINVAL;
  cudaSetDevice(h->device);
  GI_TRYS(ensure_ws(h, (int)s));
  long long ldg = ld;
  GI_TRYS(stage_operand(h, 0, G, m, n, ldg));
  return gram(h, G, m, n, ldg, trans ? 1 : 0, A, lda);
}

geninv_status geninv_from_gram_d(geninv_handle h, const double *A, int64_t s, int64_t lda, int64_t *rank,
                                 const geninv_opts *opts, geninv_info *info) {
  if (!h || !A || s < 1 || lda < s) return GENINV_EINVAL;
  cudaSetDevice(h->device);
  int r = 0;
  FactorStats fs{};
  geninv_status st = from_gram(h, A, (int)s, lda, opts, &r, &fs);
  if (st == GENINV_OK) st = finish_spd_check(h, r);
  if (rank) *rank = r;
  fill_info(info, fs, r, 0, st, s);
  return st;
}

geninv_status geninv_apply_d(geninv_handle h, const double *G, int64_t m, int64_t n, int64_t ld, int32_t trans,
                             double *Gp, int64_t ldp) {
  if (!h || !Gp) return GENINV_EINVAL;
  GI_TRYS(check_g(G, m, n, ld));
  const long long s = trans ? m : n;
  if (h->x_s != s) return GENINV_ESTATE;
  if (ldp < (trans ? s : m)) return GENINV_EINVAL;
  cudaSetDevice(h->device);
  long long ldg = ld;
  GI_TRYS(stage_operand(h, 0, G, m, n, ldg));
  return apply(h, G, m, n, ldg, trans ? 1 : 0, Gp, ldp, h->st);
}

geninv_status geninv_frchol_d(geninv_handle h, const double *A, int64_t s, int64_t lda, double *L, int64_t ldl,
                              int32_t *piv_dev, int64_t *rank, const geninv_opts *opts, geninv_info *info) {
  if (!h || !A || !L || !piv_dev || s < 1 || lda < s || ldl < s) return GENINV_EINVAL;
  cudaSetDevice(h->device);
  GI_TRYS(ensure_ws(h, (int)s));
  int r = 0;
  FactorStats fs{};
  // L is a TMA operand of the lookahead updates: an unaligned / odd-ld L is factored in the handle's
  // L workspace and copied out
  const bool direct = aligned16(L) && !(ldl & 1);
  geninv_status st = factor(h, A, lda, (int)s, direct ? L : h->L, direct ? ldl : h->ld, piv_dev, opts, &r, &fs);
  if (!direct && (st == GENINV_OK || st == GENINV_ENONFINITE || st == GENINV_ERANGE)) {
    GI_TRY(cudaMemcpy2DAsync(L, ldl * 8, h->L, h->ld * 8, (size_t)s * 8, s, cudaMemcpyDeviceToDevice, h->st));
    GI_TRY(cudaStreamSynchronize(h->st));
  }
  if (rank) *rank = r;
  fill_info(info, fs, r, 0, st, s);
  return st;
}

geninv_status geninv_spd_inverse_d(geninv_handle h, const double *B, int64_t r, int64_t ldb, double *M, int64_t ldm) {
  if (!h || !B || !M || r < 1 || ldb < r || ldm < r) return GENINV_EINVAL;
  cudaSetDevice(h->device);
  GI_TRYS(ensure_ws(h, (int)r));
  {
    const GemmOp o = op_lauum(h, (int)r, M, ldm);
    const int S = chain_splits(o);
    size_t need = S > 1 ? (size_t)S * o.M * o.N * sizeof(double) : 0;
    need = std::max(need, (size_t)trtri_part_elems((int)r, h->ld, h->ld) * sizeof(double));
    GI_TRYS(ensure_part(h, need));
  }
  GI_TRYS(spd_inverse(h, B, (int)r, ldb, M, ldm));
  return finish_spd_check(h, (int)r);
}

geninv_status geninv_copy_x(geninv_handle h, double *X, int64_t ldx, int64_t *s) {
  if (!h) return GENINV_EINVAL;
  if (h->x_s < 0) return GENINV_ESTATE;
  if (s) *s = h->x_s;
  if (!X) return GENINV_OK;
  if (ldx < h->x_s) return GENINV_EINVAL;
  cudaSetDevice(h->device);
  GI_TRY(cudaMemcpy2DAsync(X, ldx * 8, h->X, h->ld * 8, (size_t)h->x_s * 8, h->x_s, cudaMemcpyDeviceToDevice, h->st));
  GI_TRY(cudaStreamSynchronize(h->st));
  return GENINV_OK;
}

int64_t geninv_launch_count(geninv_handle h) { return h ? h->launches : 0; }

}  // extern "C"
