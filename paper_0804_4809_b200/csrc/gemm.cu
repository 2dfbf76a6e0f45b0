// Host launcher + instantiations of the FP64 DMMA GEMM core (gemm.cuh).
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <array>
#include <map>
#include <queue>
#include <vector>
#include <mutex>
#include <set>
#include <utility>

#include "gemm.cuh"
#include "gemm_host.h"

namespace gi {

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static cudaError_t get_encode() {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (err == cudaSuccess && q != cudaDriverEntryPointSuccess) err = cudaErrorNotSupported;
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return err;
}

int num_sms() {
  constexpr int MAXDEV = 64;
  static int sms[MAXDEV] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= MAXDEV) dev = 0;
  if (!sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = v > 0 ? v : 148;
  }
  return sms[dev];
}

cudaError_t smem_optin(const void *fn, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void *, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (done.count({fn, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({fn, dev});
  return e;
}

// 3-D map {cols (contiguous), rows, batch}; box {16, box_rows, 1}; 128B swizzle;
// out-of-bounds elements are filled with zeros.
static cudaError_t make_map(CUtensorMap *map, const Mat &m, int box_rows) {
  cudaError_t e = get_encode();
  if (e != cudaSuccess) return e;
  if ((reinterpret_cast<uintptr_t>(m.ptr) & 15) || (m.ld & 1) || (m.batch > 1 && (m.bstride & 1)))
    return cudaErrorMisalignedAddress;
  cuuint64_t dims[3] = {(cuuint64_t)m.cols, (cuuint64_t)m.rows, (cuuint64_t)m.batch};
  long long bstride = m.batch > 1 ? m.bstride : m.ld * m.rows;
  if (bstride < 2) bstride = 2;
  cuuint64_t strides[2] = {(cuuint64_t)m.ld * 8, (cuuint64_t)bstride * 8};
  cuuint32_t box[3] = {16, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double *>(m.ptr), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// MN-major operand as a 4-D view {16 (mn inner), rows (k), cols/16 (mn outer), batch}; box
// {16, 16, strips, 1} -> the whole [strip][k][16] tile in one TMA op, same smem layout and
// swizzle as the per-strip 3-D boxes.  Needs cols % 16 == 0.
static cudaError_t make_map_mn4d(CUtensorMap *map, const Mat &m, int strips) {
  cudaError_t e = get_encode();
  if (e != cudaSuccess) return e;
  if ((reinterpret_cast<uintptr_t>(m.ptr) & 15) || (m.ld & 1) || (m.cols % 16) || (m.batch > 1 && (m.bstride & 1)))
    return cudaErrorMisalignedAddress;
  cuuint64_t dims[4] = {16, (cuuint64_t)m.rows, (cuuint64_t)(m.cols / 16), (cuuint64_t)m.batch};
  long long bstride = m.batch > 1 ? m.bstride : m.ld * m.rows;
  if (bstride < 2) bstride = 2;
  cuuint64_t strides[3] = {(cuuint64_t)m.ld * 8, 128, (cuuint64_t)bstride * 8};
  cuuint32_t box[4] = {16, 16, (cuuint32_t)strips, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double *>(m.ptr), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// Bytes of A rows one raster band keeps L2-resident while N sweeps (GENINV_BAND_MB; default 48 MB of the
// 126 MB L2).
static long long band_bytes() {
  static const long long b = [] {
    const char *e = getenv("GENINV_BAND_MB");
    const long long mb = e ? atoll(e) : 48;
    return (mb > 0 ? mb : 48) << 20;
  }();
  return b;
}

// TMA ring depth of the 128 x 128 tiles (Gram, chain products, a7)
#ifndef GI_BIG_STAGES
#define GI_BIG_STAGES 7   // 7 x 32 KiB + 1 KiB align + barriers = 225.1 KiB of the 227 KiB opt-in (C4 Gram -0.2 %, a7 -0.13 % vs 6, A/B)
#endif

template <int BM, int BN, int WM, int WN, int ST, bool AK, bool BK_, bool CHUNK = false>
static cudaError_t launch(const GemmOp &op, GemmArgs &a, cudaStream_t st) {
  using Cfg = GemmCfg<BM, BN, WM, WN, ST, AK, BK_>;
  auto kern = dgemm_tc<BM, BN, WM, WN, ST, AK, BK_, CHUNK>;
  cudaError_t e = smem_optin((const void *)kern, Cfg::SMEM);
  if (e != cudaSuccess) return e;
  a.a_mn4d = !AK && (op.A.cols % 16 == 0) && (op.a_mn0 % 16 == 0);
  a.b_mn4d = !BK_ && (op.B.cols % 16 == 0) && (op.b_mn0 % 16 == 0);
  e = a.a_mn4d ? make_map_mn4d(&a.tmA, op.A, BM / 16) : make_map(&a.tmA, op.A, AK ? BM : 16);
  if (e != cudaSuccess) return e;
  e = a.b_mn4d ? make_map_mn4d(&a.tmB, op.B, BN / 16) : make_map(&a.tmB, op.B, BK_ ? BN : 16);
  if (e != cudaSuccess) return e;
  a.mtiles = (op.M + BM - 1) / BM;
  a.ntiles = (op.N + BN - 1) / BN;
  {
    // raster band: at most ~band_bytes() of A rows (BM x K doubles per M-tile) per band, bands balanced
    const long long per_tile = (long long)BM * (op.K > 0 ? op.K : 1) * 8;
    long long mb = std::max<long long>(1, band_bytes() / per_tile);
    const long long nb = (a.mtiles + mb - 1) / mb;
    a.mband = (int)((a.mtiles + nb - 1) / nb);
  }
  long long tiles = op.lower ? (long long)a.mtiles * (a.mtiles + 1) / 2 : (long long)a.mtiles * a.ntiles;
  if (tiles == 0) return cudaSuccess;
  dim3 grid((unsigned)tiles, op.splits, op.batch);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(a);
  return cudaGetLastError();
}

// Tile size (128 x 128, or 64 x 64 for small products) and split count (1..max_splits) of one chain GEMM that
// minimise its simulated duration: the tiles x splits CTAs in launch order, each placed on the SM slot that
// frees first, cost = per-CTA overhead + its k-slabs (a 64 x 64 slab is a quarter of a 128 x 128 one; two
// 64 x 64 CTAs share an SM), plus the fixed-order reduction's traffic.  Per-tile k-ranges follow GemmArgs
// (device-side pivots assumed evenly spread, rows ~ j * rows / K).
static double plan_sim(const GemmOp &op, int S, int tb, int sms);

static bool small_tiles_allowed() {
  static const bool on = [] {
    const char *e = getenv("GENINV_SMALL_TILES");   // 0: 128 x 128 tiles only (A/B measurements)
    return !(e && atoi(e) == 0);
  }();
  return on;
}

GemmPlan balanced_plan(const GemmOp &op, int max_splits, int sms) {
  GemmPlan pl;
  if (op.M <= 0 || op.N <= 0 || op.batch < 1 || op.K_dev) return pl;
  // memoised per shape (the simulation is ~1e4 heap operations; it must not sit on the host path)
  static std::mutex mu;
  static std::map<std::array<long long, 11>, GemmPlan> cache;
  const std::array<long long, 11> key = {op.M, op.N, op.K, op.lower, op.mirror, op.k_lo_mode, op.k_hi_mode, max_splits,
                                         sms, op.batch, small_tiles_allowed()};
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  double best = 1e300;
  for (int tb : {128, 64}) {
    if (tb == 64 && !small_tiles_allowed()) continue;
    for (int S = 1; S <= max_splits; ++S) {
      const double t = plan_sim(op, S, tb, sms);
      if (t < best * 0.97) {   // a split (or the smaller tile) must win by 3 %
        best = t;
        pl.splits = S;
        pl.tile = tb == 64 ? TILE_64x64 : TILE_128x128;
      }
    }
  }
  cache[key] = pl;
  return pl;
}

int balanced_splits(const GemmOp &op, int max_splits, int sms) { return balanced_plan(op, max_splits, sms).splits; }

static double plan_sim(const GemmOp &op, int S, int tb, int sms) {
  const int mt = (op.M + tb - 1) / tb, nt = (op.N + tb - 1) / tb;
  const long long nsl = (op.K + BK - 1) / BK;
  std::vector<int> len;
  // tile order of the kernel (lower: row-major over the lower triangle; else the banded raster)
  const long long per_tile = (long long)tb * (op.K > 0 ? op.K : 1) * 8;
  const long long mbw = std::max<long long>(1, band_bytes() / per_tile);
  const long long nbands = (mt + mbw - 1) / mbw;
  const int mband = (int)((mt + nbands - 1) / nbands);
  const double kpm = (double)op.K / op.M;   // pivots evenly spread: piv[j] ~ j K / M (L'L), #{piv < m} ~ m K / M (L M)
  auto tile_len = [&](int tm, int tn) {
    const long long m0 = (long long)tb * tm, n0 = (long long)tb * tn;
    long long klo = 0, khi = nsl;
    if (op.k_lo_mode == 1) klo = m0 / BK;
    else if (op.k_lo_mode == 2) klo = n0 / BK;
    else if (op.k_lo_mode == 3) klo = (long long)(m0 * kpm) / BK;
    if (op.k_hi_mode == 1) khi = std::min(khi, (m0 + tb + BK - 1) / BK);
    if (op.k_hi_mode == 2) khi = std::min(khi, ((long long)((m0 + tb) * kpm) + BK - 1) / BK);
    return (int)std::max(0LL, khi - std::min(klo, khi));
  };
  if (op.lower) {
    for (int bi = 0; bi < mt; ++bi)
      for (int bj = 0; bj <= bi; ++bj) len.push_back(tile_len(bi, bj));
  } else if (op.k_hi_mode) {   // the kernel's LPT order (M-tiles descending, N fastest)
    for (int tm = mt - 1; tm >= 0; --tm)
      for (int tn = 0; tn < nt; ++tn) len.push_back(tile_len(tm, tn));
  } else {
    for (int band = 0; band * mband < mt; ++band) {
      const int mb = std::min(mband, mt - band * mband);
      for (int t = 0; t < mb * nt; ++t) len.push_back(tile_len(band * mband + t % mb, t / mb));
    }
  }
  // in 128 x 128 k-slab units (~2.1 us): a 64 x 64 slab is 1/4 of the DMMA work, two such CTAs per SM
  // each at half the SM's rate -> 1/2 per slab on one of 2 x sms slots; the per-CTA overhead is the same
  const double over = 1.0, slab = tb == 64 ? 0.5 : 1.0;
  const int slots = tb == 64 ? 2 * sms : sms;
  static const double red_bw = [] {                      // bytes/s the reduction streams at (tuning override)
    const char *v = getenv("GENINV_RED_GBS");
    return (v ? atof(v) : 3000.0) * 1e9;
  }();
  const double red_per_elem = 8.0 / red_bw / 2.1e-6;     // slab units per element of the reduction
  const double out_elems = op.lower ? 0.5 * op.M * (op.M + 1.0) : (double)op.M * op.N;   // lower: partials lower only
  std::priority_queue<double, std::vector<double>, std::greater<double>> q;
  for (int i = 0; i < slots; ++i) q.push(0.0);
  double span = 0.0;
  for (int b = 0; b < op.batch; ++b)
    for (int z = 0; z < S; ++z)
      for (int l : len) {
        const int per = (l + S - 1) / S;
        const int mine = std::max(0, std::min(l, per * (z + 1)) - std::min(l, per * z));
        const double t0 = q.top();
        q.pop();
        const double t1 = t0 + over + slab * mine;
        q.push(t1);
        span = std::max(span, t1);
      }
  return span + (S > 1 ? (S + 1.0) * out_elems * op.batch * red_per_elem + 2.0 : 0.0);
}

int upd_tile_bm() {
  static const int bm = [] {
    const char *e = getenv("GENINV_UPD_TILE_BM");   // measurements: 128 = the earlier 128 x 32 tile
    return (e && atoi(e) == 128) ? 128 : 256;
  }();
  return bm;
}

cudaError_t gemm(const GemmOp &op, cudaStream_t st) {
  if (op.M <= 0 || op.N <= 0) return cudaSuccess;
  static const bool dbg = getenv("GENINV_DEBUG_GEMM") != nullptr;   // diagnostics: one line per launch
  if (dbg)
    fprintf(stderr,
            "gemm M=%d N=%d K=%d A=%p ld=%lld %lldx%lld %s mn0=%d k0=%d | B=%p ld=%lld %lldx%lld %s mn0=%d k0=%d | "
            "C=%p ldc=%lld splits=%d lower=%d kchunk=%d\n",
            op.M, op.N, op.K, (const void *)op.A.ptr, op.A.ld, op.A.rows, op.A.cols, op.a_kmajor ? "K" : "MN", op.a_mn0,
            op.a_k0, (const void *)op.B.ptr, op.B.ld, op.B.rows, op.B.cols, op.b_kmajor ? "K" : "MN", op.b_mn0, op.b_k0,
            (void *)op.C, op.ldc, op.splits, (int)op.lower, op.kchunk);
  if (op.lower && op.M != op.N) return cudaErrorInvalidValue;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.a_mn0 = op.a_mn0; a.a_k0 = op.a_k0; a.b_mn0 = op.b_mn0; a.b_k0 = op.b_k0;
  a.C = op.C; a.ldc = op.ldc; a.c_bstride = op.c_bstride; a.split_stride = op.split_stride;
  a.C0 = op.C0; a.ldc0 = op.ldc0; a.c0_bstride = op.c0_bstride;
  a.alpha = op.alpha; a.M = op.M; a.N = op.N; a.K = op.K; a.K_dev = op.K_dev;
  a.k_lo_mode = op.k_lo_mode; a.k_hi_mode = op.k_hi_mode; a.k_lo_dev = op.k_lo_dev;
  a.lower = op.lower; a.mirror = op.mirror; a.splits = op.splits < 1 ? 1 : op.splits;
  a.kchunk = op.kchunk;
  if (op.kchunk > 0) {   // the Gram (a1): both operands K-major (T branch) or both MN-major (N branch)
    if (op.alpha != 1.0 || op.C0 || op.mirror || op.tile != TILE_128x128) return cudaErrorInvalidValue;
    if (op.a_kmajor && op.b_kmajor) return launch<128, 128, 64, 32, GI_BIG_STAGES, true, true, true>(op, a, st);
    if (!op.a_kmajor && !op.b_kmajor) return launch<128, 128, 64, 32, GI_BIG_STAGES, false, false, true>(op, a, st);
    return cudaErrorInvalidValue;
  }
  if (op.tile == TILE_128x32) {
    // the panel update (K-major L both sides): 256 x 32 tiles, 8 warps = two per SM sub-partition
    // (the 128 x 32 tile keeps one warp per sub-partition with the DMMA pipe ~47 % busy)
    if (op.a_kmajor && op.b_kmajor && upd_tile_bm() == 256) return launch<256, 32, 32, 32, 6, true, true>(op, a, st);
    if (op.a_kmajor && op.b_kmajor) return launch<128, 32, 32, 32, 6, true, true>(op, a, st);
    if (op.a_kmajor && !op.b_kmajor) return launch<128, 32, 32, 32, 6, true, false>(op, a, st);
    if (!op.a_kmajor && op.b_kmajor) return launch<128, 32, 32, 32, 6, false, true>(op, a, st);
    return launch<128, 32, 32, 32, 6, false, false>(op, a, st);
  }
  if (op.tile == TILE_64x64) {   // small chain products (balanced_plan): 4 warps of 32 x 32, 4 stages
    if (op.a_kmajor && op.b_kmajor) return launch<64, 64, 32, 32, 4, true, true>(op, a, st);
    if (op.a_kmajor && !op.b_kmajor) return launch<64, 64, 32, 32, 4, true, false>(op, a, st);
    if (!op.a_kmajor && op.b_kmajor) return launch<64, 64, 32, 32, 4, false, true>(op, a, st);
    return launch<64, 64, 32, 32, 4, false, false>(op, a, st);
  }
  if (op.a_kmajor && op.b_kmajor) return launch<128, 128, 64, 32, GI_BIG_STAGES, true, true>(op, a, st);
  if (op.a_kmajor && !op.b_kmajor) return launch<128, 128, 64, 32, GI_BIG_STAGES, true, false>(op, a, st);
  if (!op.a_kmajor && op.b_kmajor) return launch<128, 128, 64, 32, GI_BIG_STAGES, false, true>(op, a, st);
  return launch<128, 128, 64, 32, GI_BIG_STAGES, false, false>(op, a, st);
}

// ---------------------------------------------------------------- split-K reduction
__global__ void splitk_reduce_kernel(const double *__restrict__ P, long long sstride, int splits, long long ldp,
                                     double *__restrict__ out, long long ldo, const double *__restrict__ C0,
                                     long long ldc0, double alpha, int M, int N, int lower, int mirror) {
  const long long total = (long long)M * N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / N), j = (int)(idx % N);
    if (lower && j > i) continue;
    // slices summed pairwise (a fixed tree: deterministic, and the rounding error grows like log2 of the
    // slice count instead of its square root): groups of 16 in flight at once, then the group sums
    double gs[4] = {0.0, 0.0, 0.0, 0.0};
    for (int z0 = 0, gi = 0; z0 < splits; z0 += 16, ++gi) {
      double v[16];
#pragma unroll
      for (int z = 0; z < 16; ++z) v[z] = z0 + z < splits ? P[(z0 + z) * sstride + (long long)i * ldp + j] : 0.0;
#pragma unroll
      for (int w = 1; w < 16; w <<= 1)
#pragma unroll
        for (int z = 0; z < 16; z += 2 * w) v[z] += v[z + w];
      if (gi < 4) gs[gi] = v[0];
      else gs[3] += v[0];   // beyond 64 slices (not used by the library's split counts)
    }
    const double s = (gs[0] + gs[1]) + (gs[2] + gs[3]);
    double o = alpha * s;
    if (C0) o += C0[(long long)i * ldc0 + j];
    out[(long long)i * ldo + j] = o;
    if (mirror && j != i) out[(long long)j * ldo + i] = o;
  }
}

cudaError_t splitk_reduce(const double *P, long long split_stride, int splits, long long ldp, double *out,
                          long long ldo, const double *C0, long long ldc0, double alpha, int M, int N, bool lower,
                          cudaStream_t st, bool mirror) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  long long total = (long long)M * N;
  int blocks = (int)std::min<long long>((total + 255) / 256, (long long)num_sms() * 16);
  splitk_reduce_kernel<<<blocks, 256, 0, st>>>(P, split_stride, splits, ldp, out, ldo, C0, ldc0, alpha, M, N,
                                               lower ? 1 : 0, (lower && mirror) ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace gi
