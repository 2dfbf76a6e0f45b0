// FP64 tensor-core GEMM core for sm_100a: TMA (128B-swizzled) -> shared
// memory ring (mbarrier full/empty) -> warp-level DMMA.8x8x4 with register
// accumulators.  Thread 0 issues TMA; all NW warps compute (no
// producer warp: 8 warps keep the 255-register budget per thread).
//
// Used for every dense contraction of the geninv hot path:
//   a1 Gram A = G'G / GG'      -> lower-triangle tiles, split-K
//   a3 panel update  A - L L'         -> BN = 32 tiles, split-K, device-side K
//   a4 B = L'L, a5 TRTRI / LAUUM, a6 K = L M, X = K K', a7 X G' / G' X
//
// C(m, n) = sum_k A(m, k) B(k, n), operands row-major in HBM:
//   A "K-major":  A(m, k) = A[m*ld + k]      A "MN-major": A(m, k) = A[k*ld + m]
//   B "K-major":  B(k, n) = B[n*ld + k]      B "MN-major": B(k, n) = B[k*ld + n]
// There is no FP64 tcgen05 kind on sm_100a (ptxas rejects .kind::f64), so
// the FP64 tensor pipe is reached through mma.sync.m8n8k4 (SASS DMMA.8x8x4).
#pragma once
#include "common.cuh"

namespace gi {

constexpr int BK = 16;  // doubles per k-slab: one 128-byte swizzle row

struct GemmArgs {
  CUtensorMap tmA, tmB;     // 3-D maps {inner, outer, batch}; see make_operand_map()
  int a_mn0, a_k0;          // tile-origin offsets inside the A map (m, k)
  int b_mn0, b_k0;          // (n, k) for B
  double *C;                // output (split > 1: partial slices)
  long long ldc, c_bstride, split_stride;
  const double *C0;         // optional addend: C = C0 + alpha * AB   (ignored for split > 1)
  long long ldc0, c0_bstride;
  double alpha;
  int M, N, K;              // K ignored if K_dev
  const int *K_dev;         // device-resident K (panel update: the running rank r0)
  int k_lo_mode, k_hi_mode;  // structured zeros of a triangular operand: the k-range of a tile is
                             //   lo: 1 -> k >= m0, 2 -> k >= n0, 3 -> k >= k_lo_dev[m0];
                             //   hi: 1 -> k < m0 + BM, 2 -> k < #{j : k_lo_dev[j] < m0 + BM}
  const int *k_lo_dev;       // mode 3: first nonzero k of each operand column (L'L: pivot rows)
  int mtiles, ntiles;
  int mband;                // M-tiles per raster band (non-lower): a band of A stays L2-resident while N sweeps
  int lower;                // 1: enumerate lower-triangle tiles of a square output (M == N)
  int mirror;               // 1 (with lower): also store C[n][m]; diagonal tiles store m >= n mirrored
  int splits;               // split-K count
  int a_mn4d, b_mn4d;       // MN-major operand mapped as a 4-D {16, k, mn/16, batch} view: one TMA op per tile
  int kchunk;               // CHUNK instances: k-slabs per register accumulation; each chunk's sum is added
                            //   into the CTA's output tile in memory (two-level accumulation, see below)
};

// row permutation inside an 8-row fragment: makes the LDS.128 fragment loads
// bank-conflict-free on 128B-swizzled tiles (rows of the same quarter-warp
// differ in bit 2).
GI_DEV int frag_perm(int g) { return (g >> 1) | ((g & 1) << 2); }

template <int BM, int BN, int WM, int WN, int STAGES, bool A_K, bool B_K>
struct GemmCfg {
  static constexpr int NWM = BM / WM, NWN = BN / WN, NW = NWM * NWN;
  static constexpr int THREADS = NW * 32;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int A_BYTES = BM * BK * 8, B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 2 * STAGES * 8;
  static_assert(WM % 16 == 0 && WN % 16 == 0, "warp tile must be a multiple of 16");
};

// Output tile (tm, tn) of CTA t: lower-triangle enumeration, LPT order for growing k-ranges, or the
// banded raster of the general case.
GI_DEV void tile_of(const GemmArgs &p, int t, int &tm, int &tn) {
  if (p.lower) {
    // t -> (bi, bj), bj <= bi, row-major over the lower triangle
    int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
    while (bi * (bi + 1) / 2 > t) --bi;
    tm = bi;
    tn = t - bi * (bi + 1) / 2;
  } else if (p.k_hi_mode) {
    // the k-range grows with the M-tile (A trapezoidal: K = L M, TRTRI's C22 products): longest
    // tiles first (LPT order, N fastest), so the last partial wave holds the short ones
    tm = p.mtiles - 1 - t / p.ntiles;
    tn = t - (t / p.ntiles) * p.ntiles;
  } else {
    // banded raster: M fastest inside a band of mband M-tiles, then N, then the next band, so the
    // A rows of one band (sized on the host to fit the L2) are re-read from L2, not HBM.
    const int band_tiles = p.mband * p.ntiles;
    const int band = t / band_tiles;
    const int rem = t - band * band_tiles;
    const int mb = min(p.mband, p.mtiles - band * p.mband);
    tm = band * p.mband + rem % mb;
    tn = rem / mb;
  }
}

// Special registers read without CSE (the CHUNK flush re-derives its coordinates instead of keeping
// them live across the main loop).
GI_DEV int fresh_ctaid_x() { int v; asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(v)); return v; }
GI_DEV int fresh_ctaid_y() { int v; asm volatile("mov.u32 %0, %%ctaid.y;" : "=r"(v)); return v; }
GI_DEV int fresh_tid_x() { int v; asm volatile("mov.u32 %0, %%tid.x;" : "=r"(v)); return v; }

// CHUNK (the Gram, a1): the k-range of a CTA is accumulated in register chunks of p.kchunk slabs; after
// each chunk the warp adds its fragment sums into the output tile in memory (the first chunk stores) and
// restarts from zero.  A 2^21-row Gram then sums ~8k-row partials instead of ~57k-row sequential chains
// (rounding error of a sequential sum grows like sqrt(length)); every element is owned by one thread, so
// the read-back needs no synchronisation, and the order is fixed (deterministic).
template <int BM, int BN, int WM, int WN, int STAGES, bool A_K, bool B_K, bool CHUNK = false>
__global__ void __launch_bounds__(GemmCfg<BM, BN, WM, WN, STAGES, A_K, B_K>::THREADS, 1)
    dgemm_tc(const __grid_constant__ GemmArgs p) {
  using Cfg = GemmCfg<BM, BN, WM, WN, STAGES, A_K, B_K>;
  constexpr int NW = Cfg::NW, FM = Cfg::FM, FN = Cfg::FN;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t *empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // ---- tile coordinates
  int tm, tn;
  tile_of(p, blockIdx.x, tm, tn);
  const int split = blockIdx.y, bz = blockIdx.z;
  const int m0 = tm * BM, n0 = tn * BN;
  const int K = p.K_dev ? *p.K_dev : p.K;
  const int nslab_all = (K + BK - 1) / BK;
  // k-range of this tile: [klo, khi) in slabs (triangular operands skip their zero blocks)
  int klo = 0, khi = nslab_all;
  if (p.k_lo_mode == 1) klo = m0 / BK;
  else if (p.k_lo_mode == 2) klo = n0 / BK;
  else if (p.k_lo_mode == 3) klo = (m0 < p.M ? p.k_lo_dev[m0] : K) / BK;
  if (p.k_hi_mode == 1) khi = min(khi, (m0 + BM + BK - 1) / BK);
  if (p.k_hi_mode == 2) {   // k < #{j : k_lo_dev[j] < m0 + BM}  (k_lo_dev increasing, length K)
    int lo = 0, hi = K;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (p.k_lo_dev[mid] < m0 + BM) lo = mid + 1;
      else hi = mid;
    }
    khi = min(khi, (lo + BK - 1) / BK);
  }
  klo = min(klo, khi);
  const int nrange = khi - klo;
  const int per = (nrange + p.splits - 1) / p.splits;
  const int s_begin = klo + min(nrange, split * per);
  const int s_end = min(khi, s_begin + per);
  const int nslab = max(0, s_end - s_begin);

  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], NW);
    }
    fence_barrier_init();
  }
  __syncthreads();

  // TMA issue (thread 0): slab `it` goes to stage it % STAGES.  The first
  // STAGES slabs are issued up front; at the top of iteration it, slab
  // it + STAGES - 1 is issued once every warp has released stage
  // (it - 1) % STAGES (empty barrier).
  // Issued by all 32 lanes of warp 0: lane 0 arms the barrier, then each TMA box
  // (one for a K-major tile, 16-column strips for an MN-major tile) is issued by
  // its own lane -- one warp instruction instead of up to 16 serial issues.
  auto issue = [&](int it) {
    const int st = it % STAGES;
    unsigned char *sA = smem + st * Cfg::STAGE_BYTES;
    unsigned char *sB = sA + Cfg::A_BYTES;
    if (lane == 0) mbar_arrive_expect_tx(&full[st], Cfg::STAGE_BYTES);
    __syncwarp();
    const int k = (s_begin + it) * BK;
    constexpr int NA = A_K ? 1 : BM / 16, NB = B_K ? 1 : BN / 16;
    static_assert(NA + NB <= 32, "one lane per TMA box");
    if (lane < NA) {
      if (A_K) tma_load_3d(sA, &p.tmA, &full[st], p.a_k0 + k, p.a_mn0 + m0, bz);
      else if (p.a_mn4d) { if (lane == 0) tma_load_4d(sA, &p.tmA, &full[st], 0, p.a_k0 + k, (p.a_mn0 + m0) / 16, bz); }
      else tma_load_3d(sA + lane * 2048, &p.tmA, &full[st], p.a_mn0 + m0 + 16 * lane, p.a_k0 + k, bz);
    } else if (lane < NA + NB) {
      const int q = lane - NA;
      if (B_K) tma_load_3d(sB, &p.tmB, &full[st], p.b_k0 + k, p.b_mn0 + n0, bz);
      else if (p.b_mn4d) { if (q == 0) tma_load_4d(sB, &p.tmB, &full[st], 0, p.b_k0 + k, (p.b_mn0 + n0) / 16, bz); }
      else tma_load_3d(sB + q * 2048, &p.tmB, &full[st], p.b_mn0 + n0 + 16 * q, p.b_k0 + k, bz);
    }
  };
  if (warp == 0 && nslab > 0) {
    if (lane == 0) {
      tma_prefetch(&p.tmA);
      tma_prefetch(&p.tmB);
    }
    for (int it = 0; it < STAGES && it < nslab; ++it) issue(it);
  }

  // ================= DMMA consumers =================
  const int wm = warp % Cfg::NWM, wn = warp / Cfg::NWM;
  const int g = lane >> 2, t = lane & 3;
  const int pg = frag_perm(g);

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // registers -> the output tile; add = 1: add to what this thread stored before (CHUNK only)
  auto chunk_out = [&](bool add, int tm, int tn, int split, int wm, int wn, int g, int t, int pg) {
    const int m0 = tm * BM, n0 = tn * BN;
    const bool diag_tile = p.lower && (tm == tn);
    double *Cb = p.C + (long long)bz * p.c_bstride + (p.splits > 1 ? (long long)split * p.split_stride : 0);
    const double *C0b = (p.C0 && p.splits == 1) ? p.C0 + (long long)bz * p.c0_bstride : nullptr;
    const double alpha = (p.splits > 1) ? 1.0 : p.alpha;
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      int m;
      if (A_K) m = m0 + wm * WM + i * 8 + pg;
      else m = m0 + wm * WM + 16 * (i >> 1) + 2 * g + (i & 1);
      if (m >= p.M) continue;
#pragma unroll
      for (int j = 0; j < FN; ++j) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          int n;
          if (B_K) n = n0 + wn * WN + j * 8 + t + 4 * v;
          else n = n0 + wn * WN + 16 * (j >> 1) + 4 * t + 2 * v + (j & 1);
          if (n >= p.N) continue;
          if (p.lower && diag_tile && n > m) continue;  // diagonal tiles: keep m >= n
          double *cp = Cb + (long long)m * p.ldc + n;
          if (CHUNK) {   // Gram: alpha = 1, no addend, no mirror
            *cp = add ? *cp + acc[i][j][v] : acc[i][j][v];
          } else {
            double val = alpha * acc[i][j][v];
            if (C0b) val += C0b[(long long)m * p.ldc0 + n];
            *cp = val;
            if (p.mirror && n != m) Cb[(long long)n * p.ldc + m] = val;
          }
        }
      }
    }
  };

  // CHUNK: coordinates re-derived from fresh special-register reads (nothing of the epilogue stays live
  // across the main loop: the two-operand K-major instance would otherwise spill)
  auto flush = [&](bool add) {
    int ftm, ftn;
    tile_of(p, fresh_ctaid_x(), ftm, ftn);
    const int tid = fresh_tid_x();
    const int fg = (tid & 31) >> 2;
    chunk_out(add, ftm, ftn, fresh_ctaid_y(), (tid >> 5) % Cfg::NWM, (tid >> 5) / Cfg::NWM, fg, tid & 3,
              frag_perm(fg));
  };

  const uint32_t sbase = smem_u32(smem);
  // CHUNK: an outer loop over chunks of p.kchunk slabs with the flush between them, so the inner loop is
  // the plain one (a flush test inside it cost ~8 % of the Gram's DMMA rate)
  const int chunk = CHUNK ? p.kchunk : nslab;
  for (int c0 = 0; c0 < nslab; c0 += chunk) {
  const int c1 = min(nslab, c0 + chunk);
  for (int it = c0; it < c1; ++it) {
    // refill the stage released by slab it - 1 with slab it + STAGES - 1 before computing slab it
    if (warp == 0 && it >= 1 && it + STAGES - 1 < nslab) {
      const int prev = it - 1;
      mbar_wait(&empty[prev % STAGES], (prev / STAGES) & 1);
      issue(it + STAGES - 1);
    }
    const int st = it % STAGES;
    const uint32_t ph = (it / STAGES) & 1;
    const bool kmask_slab = p.K_dev && (s_begin + it + 1) * BK > K;
    mbar_wait(&full[st], ph);
    const uint32_t sA = sbase + st * Cfg::STAGE_BYTES;
    const uint32_t sB = sA + Cfg::A_BYTES;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      // fragments for DMMA k-steps d = 2h (e = 0) and d = 2h + 1 (e = 1);
      // lane t of step d covers k = 8h + 2t + e.
      double2 av[2][FM], bv[2][FN];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int kap = 8 * h + 2 * t + e;  // MN-major k-row
        if (A_K) {
          if (e == 0) {
#pragma unroll
            for (int f = 0; f < FM; ++f) {
              const int row = wm * WM + f * 8 + pg;
              double2 v = lds128(sA + row * 128 + (((4 * h + t) ^ pg) << 4));
              av[0][f] = v;
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < FM / 2; ++q) {
            const int strip = (wm * WM) / 16 + q;
            double2 v = lds128(sA + strip * 2048 + kap * 128 + ((g ^ (kap & 7)) << 4));
            av[e][2 * q] = v;
          }
        }
        if (B_K) {
          if (e == 0) {
#pragma unroll
            for (int f = 0; f < FN; ++f) {
              const int row = wn * WN + f * 8 + pg;
              bv[0][f] = lds128(sB + row * 128 + (((4 * h + t) ^ pg) << 4));
            }
          }
        } else {
#pragma unroll
          for (int q = 0; q < FN / 2; ++q) {
            const int strip = (wn * WN) / 16 + q;
            bv[e][2 * q] = lds128(sB + strip * 2048 + kap * 128 + ((g ^ (kap & 7)) << 4));
          }
        }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double a[FM], b[FN];
#pragma unroll
        for (int f = 0; f < FM; ++f) {
          if (A_K) a[f] = e ? av[0][f].y : av[0][f].x;
          else a[f] = (f & 1) ? av[e][f & ~1].y : av[e][f & ~1].x;
        }
#pragma unroll
        for (int f = 0; f < FN; ++f) {
          if (B_K) b[f] = e ? bv[0][f].y : bv[0][f].x;
          else b[f] = (f & 1) ? bv[e][f & ~1].y : bv[e][f & ~1].x;
        }
        // device-side K (K_dev) that ends inside this slab: columns k >= K may hold live data
        // (the panel update reads L while later columns are being written) -> zero them.
        if (kmask_slab && (s_begin + it) * BK + 8 * h + 2 * t + e >= K) {
#pragma unroll
          for (int f = 0; f < FM; ++f) a[f] = 0.0;
        }
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j) dmma(acc[i][j], a[i], b[j]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  if (CHUNK && c1 < nslab) {
    flush(c0 > 0);
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  }
  }

  // ================= epilogue (registers -> global) =================
  if (CHUNK) flush(nslab > p.kchunk);
  else chunk_out(false, tm, tn, split, wm, wn, g, t, pg);
}

}  // namespace gi
