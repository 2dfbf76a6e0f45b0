// The two big FP64 contractions (a1 Gram, a7 output product) on the INT8 tensor cores (SURVEY §8(f)
// f4, opt-in: geninv_set_emulation; DESIGN.md §6 "FP64 emulation"), by Ozaki splitting.
//
// Every line (row or column, whichever runs along K) of both operands is scaled by a power of two 2^e
// (|x| < 2^e) and split error-free into S digits with weights w_t = 2^(1-8t):
//   v = x 2^-e in (-1, 1):  d_1 = floor(128 v) in [-128, 127] (signed int8),  v <- 128 v - d_1 in [0, 1);
//   t >= 2:                 d_t = floor(256 v) in [0, 255]   (unsigned int8), v <- 256 v - d_t,
// every step exact in FP64, so x = 2^e sum_t d_t w_t + r with 0 <= r 2^-e < 2^(1-8S).  Then
//   C[i][j] = 2^(e_i + f_j) sum_g 2^(2-8g) P_g[i][j],  P_g = sum_{t+u=g} sum_k d_t[i][k] d'_u[j][k],
// every P_g an exact int32 sum (at most 7 pairs x K x 255^2 < 2^31 for K <= 4096 per pass) computed by
// tcgen05.mma.kind::i8 with each operand's signedness set per digit (d_1 signed, the rest unsigned).
// Groups g = T .. 2 (smallest terms first) are converted exactly to FP64, scaled exactly (powers of
// two) and accumulated in FP64.  S = 7, T = 9 (34 int8 products) leaves |C - C_exact| <= 2.4e-17
// sum_k |x_ik g_jk| (tools/emu_gemm.cu against a long-double reference): below an FP64 GEMM's own
// rounding bound.  (T = 8, 28 products: 2.9e-15 -- the unsigned digits' errors do not cancel.)
//
// emu_gemm_kernel (persistent, 192 threads, one 128 x 256 tile of C at a time): warp 0 lane 0 issues
// the TMA loads (128-byte K slabs of the digit planes, SWIZZLE_128B, 4-stage ring), warp 1 lane 0
// issues the MMAs (M = 128, N = 256, K = 32) into one of two TMEM accumulators (2 x 256 columns,
// ping-pong by group), warps 2-5 (one TMEM lane quarter each) drain a finished group into the
// running sum while the next one runs.  The digit splits: emu_split_kernel (rows, K-major already),
// emu_colmax_kernel + emu_split_cols_kernel (columns: a shared-memory transpose).
#include <cudaTypedefs.h>
#include <stdio.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "emu.h"
#include "gemm_host.h"

namespace gi {

namespace {

constexpr int EBM = 128, EBN = 256, EBK = 128, ESTAGES = 4;
constexpr int EA_BYTES = EBM * EBK, EB_BYTES = EBN * EBK, ESTAGE_BYTES = EA_BYTES + EB_BYTES;
constexpr int ESMEM = ESTAGES * ESTAGE_BYTES + 1024 + 512 + EBN * 4;
constexpr int ENT = 192;
// kind::i8 instruction descriptor: D s32, K-major A and B, N = 256, M = 128; A / B signed (1) or not (0)
GI_DEV uint32_t idesc_i8(int a_signed, int b_signed) {
  return (2u << 4) | ((uint32_t)a_signed << 7) | ((uint32_t)b_signed << 10) | ((uint32_t)(EBN >> 3) << 17) |
         ((uint32_t)(EBM >> 4) << 24);
}

GI_DEV void tma_load_3d_u8(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2) {
  tma_load_3d(dst, m, bar, c0, c1, c2);
}
// K-major operand tile: 128-byte rows, 8-row swizzle atoms of 1024 bytes (SBO), SWIZZLE_128B, sm_100 version
GI_DEV uint64_t umma_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
GI_DEV void mma_i8(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
GI_DEV void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
#define GI_DEV_HOST_INLINE __host__ __device__ __forceinline__
GI_DEV double pow2i(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }   // 2^e, |e| <= 1022

// Tiles of a square output's lower triangle (128 x 256 tiles: column block nj holds row blocks
// 2 nj .. mt - 1; the upper halves inside them are computed too, never read).
GI_DEV_HOST_INLINE int lower_tiles(int mt, int ntn) {
  int n = 0;
  for (int nj = 0; nj < ntn; ++nj) n += mt - 2 * nj > 0 ? mt - 2 * nj : 0;
  return n;
}
GI_DEV void tile_origin(int tile, int mt, int lower, int &m0, int &n0) {
  if (!lower) {
    m0 = (tile % mt) * EBM;
    n0 = (tile / mt) * EBN;
    return;
  }
  int nj = 0;
  while (tile >= mt - 2 * nj) {
    tile -= mt - 2 * nj;
    ++nj;
  }
  m0 = (2 * nj + tile) * EBM;
  n0 = nj * EBN;
}

// Persistent: CTA c takes tiles c, c + gridDim.x, ... (tile = m-tile fastest, so CTAs working at the
// same time share the B slices of one n-tile); the stage ring, the TMEM ping-pong and the scratch tile
// carry over from one tile to the next, so a tile's last epilogue overlaps the next tile's MMAs.
__global__ void __launch_bounds__(ENT, 1) emu_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                          const __grid_constant__ CUtensorMap tmB,
                                                          const int *__restrict__ ea, const int *__restrict__ eb,
                                                          double *__restrict__ C, long long ldc, int M, int N,
                                                          int Kp, int S, int T, double *__restrict__ scratch,
                                                          int lower, int accumulate) {
  extern __shared__ uint8_t emu_smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)emu_smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(smem + ESTAGES * ESTAGE_BYTES);
  uint64_t *empty = full + ESTAGES;
  uint64_t *accfull = empty + ESTAGES;
  uint64_t *accempty = accfull + 2;
  uint32_t *tslot = (uint32_t *)(accempty + 2);
  int *s_eb = (int *)(smem + ESTAGES * ESTAGE_BYTES + 512);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nk = (Kp + EBK - 1) / EBK;
  const int mt = (M + EBM - 1) / EBM, ntn = (N + EBN - 1) / EBN;
  const int ntiles = lower ? lower_tiles(mt, ntn) : mt * ntn;
  if (tid == 0) {
    for (int i = 0; i < ESTAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accfull[i], 1);
      mbar_init(&accempty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {   // TMA producer over (tile, group, pair, k-slab)
      tma_prefetch(&tmA);
      tma_prefetch(&tmB);
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int m0, n0;
        tile_origin(tile, mt, lower, m0, n0);
        for (int g = T; g >= 2; --g)
          for (int t = max(1, g - S); t <= min(S, g - 1); ++t)
            for (int kb = 0; kb < nk; ++kb, ++it) {
              const int st = it % ESTAGES;
              if (it >= ESTAGES) mbar_wait(&empty[st], ((it / ESTAGES) & 1) ^ 1);
              uint8_t *sA = smem + st * ESTAGE_BYTES, *sB = sA + EA_BYTES;
              mbar_arrive_expect_tx(&full[st], ESTAGE_BYTES);
              tma_load_3d_u8(sA, &tmA, &full[st], kb * EBK, m0, t - 1);
              tma_load_3d_u8(sB, &tmB, &full[st], kb * EBK, n0, g - t - 1);
            }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // MMA issuer: the q-th group (over all tiles) into TMEM buffer q & 1
      int it = 0, q = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
        for (int g = T; g >= 2; --g, ++q) {
          const int buf = q & 1;
          if (q >= 2) mbar_wait(&accempty[buf], ((q >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t acc = tmem + buf * EBN;
          uint32_t accumulate = 0;
          for (int t = max(1, g - S); t <= min(S, g - 1); ++t) {
            const uint32_t idesc = idesc_i8(t == 1, g - t == 1);   // d_1 signed, later digits unsigned
            for (int kb = 0; kb < nk; ++kb, ++it) {
              const int st = it % ESTAGES;
              mbar_wait(&full[st], (it / ESTAGES) & 1);
              asm volatile("tcgen05.fence::after_thread_sync;");
              const uint32_t a0 = smem_u32(smem + st * ESTAGE_BYTES), b0 = a0 + EA_BYTES;
#pragma unroll
              for (int kk = 0; kk < EBK / 32; ++kk) {
                mma_i8(acc, umma_desc(a0 + 32 * kk), umma_desc(b0 + 32 * kk), idesc, accumulate);
                accumulate = 1;
              }
              mma_commit(&empty[st]);   // the stage is free once these MMAs have read it
            }
          }
          mma_commit(&accfull[buf]);
        }
    }
  } else {
    // epilogue warps 2..5: TMEM lane quarter warp & 3 = tile rows 32 (warp & 3) + lane.  The running sum
    // lives in this CTA's scratch tile, column-major ([c][row]: a warp's 32 rows are 256 contiguous
    // bytes, every access coalesced); the last group (g = 2) adds it into C.
    const int quarter = warp & 3;
    double *sc0 = scratch + (long long)blockIdx.x * EBN * EBM + 32 * quarter + lane;
    int q = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int m0, n0;
      tile_origin(tile, mt, lower, m0, n0);
      const int row = m0 + 32 * quarter + lane;
      const int ea_r = row < M ? ea[row] : 0;
      double *crow = C + (long long)row * ldc;
      asm volatile("bar.sync 1, 128;" ::: "memory");   // the previous tile's s_eb is no longer read
      for (int j = tid - 64; j < EBN; j += 128) s_eb[j] = n0 + j < N ? eb[n0 + j] : 0;
      asm volatile("bar.sync 1, 128;" ::: "memory");
      for (int g = T; g >= 2; --g, ++q) {
        const int buf = q & 1;
        const bool first = g == T, last = g == 2;
        mbar_wait(&accfull[buf], (q >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const double sr = pow2i(ea_r + 2 - 8 * g);   // the group's digit weight 2^(2-8g)
        for (int c0 = 0; c0 < EBN; c0 += 32) {
          uint32_t r[32];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
              "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
              : "r"(tmem + buf * EBN + ((uint32_t)(32 * quarter) << 16) + c0));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          double *sc = sc0 + (long long)c0 * EBM;
          double o[32];
          if (!first) {
#pragma unroll
            for (int j = 0; j < 32; ++j) o[j] = __ldcg(sc + j * EBM);
          }
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const double v = (double)(int)r[j] * sr * pow2i(s_eb[c0 + j]);
            o[j] = first ? v : o[j] + v;
          }
          if (!last) {
#pragma unroll
            for (int j = 0; j < 32; ++j) __stcg(sc + j * EBM, o[j]);
          } else if (row < M) {
            const int nb = n0 + c0;
            if (nb + 32 <= N && !(ldc & 1)) {
              double2 *d2 = reinterpret_cast<double2 *>(crow + nb);
              if (accumulate) {   // C += this pass (the Gram over K-chunks), old values loaded first
                double2 c[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) c[j] = d2[j];
#pragma unroll
                for (int j = 0; j < 16; ++j) d2[j] = make_double2(c[j].x + o[2 * j], c[j].y + o[2 * j + 1]);
              } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) d2[j] = make_double2(o[2 * j], o[2 * j + 1]);
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (nb + j < N) crow[nb + j] = accumulate ? crow[nb + j] + o[j] : o[j];
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive(&accempty[buf]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// One warp per row: e = the exponent with max|x| 2^-e < 127/128, then S int8 digits per element
// (slices [S][rows][Kp], columns [K, Kp) zero).  Rows whose exponent leaves the range the exact
// power-of-two scaling needs set *flag.
__global__ void emu_split_kernel(const double *__restrict__ X, long long ldx, int rows, int K, int Kp, int S,
                                 int8_t *__restrict__ sl, int *__restrict__ ex, int *flag) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const double *x = X + (long long)warp * ldx;
  double mx = 0.0;
  for (int k = lane; k < K; k += 32) mx = fmax(mx, fabs(x[k]));
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);                      // mx < 2^e
  if (!isfinite(mx) || e < -900 || e > 900) {
    if (lane == 0) atomicOr(flag, 1);
    e = 0;
  }
  if (lane == 0) ex[warp] = e;
  const double inv = ldexp(1.0, -e);
  const long long plane = (long long)rows * Kp;
  int8_t *out = sl + (long long)warp * Kp;
  bool bad = false;   // NaN / Inf: fmax above ignores NaN, so every element is checked here
  for (int k0 = 4 * lane; k0 < Kp; k0 += 128) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double xv = (k0 + q < K) ? x[k0 + q] : 0.0;
      bad |= !isfinite(xv);
      v[q] = xv * inv;
    }
    for (int t = 0; t < S; ++t) {
      char4 c;
      signed char d[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double y = v[q] * (t == 0 ? 128.0 : 256.0);
        const double r = floor(y);                   // t = 0: [-128, 127]; later: [0, 255] (v >= 0)
        d[q] = (signed char)(unsigned char)(int)r;
        v[q] = y - r;
      }
      c.x = d[0]; c.y = d[1]; c.z = d[2]; c.w = d[3];
      if (k0 + 3 < Kp) *reinterpret_cast<char4 *>(out + t * plane + k0) = c;
      else
        for (int q = 0; q < 4 && k0 + q < Kp; ++q) out[t * plane + k0 + q] = d[q];
    }
  }
  if (bad) atomicOr(flag, 1);
}

// Column maxima of |G| over rows [0, rows) of a row-major block (the N-branch Gram's K-chunk):
// bit patterns of non-negative doubles order like the doubles, so atomicMax on them is exact.
__global__ void emu_colmax_kernel(const double *__restrict__ G, long long ld, int rows, int cols,
                                  unsigned long long *__restrict__ mx) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const int r0 = blockIdx.y * 256, r1 = min(rows, r0 + 256);
  double m = 0.0;
  for (int r = r0; r < r1; ++r) m = fmax(m, fabs(G[(long long)r * ld + c]));
  atomicMax(mx + c, (unsigned long long)__double_as_longlong(m));
}

GI_DEV int emu_exponent(double mx, int *flag) {
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);                      // mx < 2^e
  if (!isfinite(mx) || e < -900 || e > 900) {
    atomicOr(flag, 1);
    e = 0;
  }
  return e;
}

// Digits of the COLUMNS of a row-major block (rows x cols): planes [S][cols][Kp] with Kp = padded rows,
// i.e. the K-major operand of G'G for this K-chunk.  Block: 128 rows x 32 columns through shared
// memory; warp w writes columns w, w + 8, .. as 128 contiguous bytes per plane.
__global__ void __launch_bounds__(256) emu_split_cols_kernel(const double *__restrict__ G, long long ld, int rows,
                                                            int cols, int Kp, int S,
                                                            const unsigned long long *__restrict__ mx,
                                                            int8_t *__restrict__ sl, int *__restrict__ ex,
                                                            int *flag) {
  __shared__ double t[32][129];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 128;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = warp; i < 128; i += 8) {
    const int r = r0 + i, c = c0 + lane;
    t[lane][i] = (r < rows && c < cols) ? G[(long long)r * ld + c] : 0.0;
  }
  __syncthreads();
  const long long plane = (long long)cols * Kp;
  for (int cc = warp; cc < 32; cc += 8) {
    const int c = c0 + cc;
    if (c >= cols) break;
    const int e = emu_exponent(__longlong_as_double((long long)mx[c]), flag);
    if (blockIdx.y == 0 && lane == 0) ex[c] = e;
    const double inv = ldexp(1.0, -e);
    const int k = r0 + 4 * lane;
    double v[4];
    bool bad = false;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      bad |= !isfinite(t[cc][4 * lane + q]);
      v[q] = t[cc][4 * lane + q] * inv;
    }
    if (bad) atomicOr(flag, 1);
    int8_t *out = sl + (long long)c * Kp;
    for (int tt = 0; tt < S; ++tt) {
      signed char d[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double y = v[q] * (tt == 0 ? 128.0 : 256.0);
        const double rr = floor(y);
        d[q] = (signed char)(unsigned char)(int)rr;
        v[q] = y - rr;
      }
      if (k + 3 < Kp) {
        char4 c4;
        c4.x = d[0]; c4.y = d[1]; c4.z = d[2]; c4.w = d[3];
        *reinterpret_cast<char4 *>(out + tt * plane + k) = c4;
      } else {
        for (int q = 0; q < 4 && k + q < Kp; ++q) out[tt * plane + k + q] = d[q];
      }
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 g_enc8 = nullptr;

cudaError_t get_enc8() {
  static std::once_flag once;
  static cudaError_t err = cudaSuccess;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void *fn = nullptr;
    err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (err == cudaSuccess && q != cudaDriverEntryPointSuccess) err = cudaErrorNotSupported;
    g_enc8 = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return err;
}

cudaError_t slice_map(CUtensorMap *m, const int8_t *p, int rows, int Kp, int S, int box_rows) {
  cudaError_t e = get_enc8();
  if (e != cudaSuccess) return e;
  cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)S};
  cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)Kp * rows};
  cuuint32_t box[3] = {EBK, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_enc8(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void *)p, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

int num_sms_emu() { return num_sms(); }   // per device (gemm.cu)

}  // namespace

int emu_kpad(int K) { return (K + 15) / 16 * 16; }

cudaError_t emu_split(const double *X, long long ldx, int rows, int K, int S, int8_t *slices, int *exps, int *flag,
                      cudaStream_t st) {
  if (rows <= 0) return cudaSuccess;
  const int Kp = emu_kpad(K);
  const int wpb = 8;
  emu_split_kernel<<<(rows + wpb - 1) / wpb, 32 * wpb, 0, st>>>(X, ldx, rows, K, Kp, S, slices, exps, flag);
  return cudaGetLastError();
}

static int emu_ctas(int M, int N, int lower) {
  const int mt = (M + EBM - 1) / EBM, ntn = (N + EBN - 1) / EBN;
  const long long tiles = lower ? lower_tiles(mt, ntn) : (long long)mt * ntn;
  return (int)std::min<long long>(tiles, num_sms_emu());
}

long long emu_scratch_elems(int M, int N) { return (long long)emu_ctas(M, N, 0) * EBM * EBN; }

cudaError_t emu_gemm_nt(const int8_t *As, const int *ea, int M, const int8_t *Bs, const int *eb, int N, int K, int S,
                        int T, double *C, long long ldc, double *scratch, cudaStream_t st, int lower,
                        int accumulate) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const int Kp = emu_kpad(K);
  CUtensorMap ta, tb;
  cudaError_t e = slice_map(&ta, As, M, Kp, S, EBM);
  if (e != cudaSuccess) return e;
  if ((e = slice_map(&tb, Bs, N, Kp, S, EBN)) != cudaSuccess) return e;
  if ((e = smem_optin((const void *)emu_gemm_kernel, ESMEM)) != cudaSuccess) return e;
  emu_gemm_kernel<<<emu_ctas(M, N, lower), ENT, ESMEM, st>>>(ta, tb, ea, eb, C, ldc, M, N, Kp, S, T, scratch,
                                                              lower, accumulate);
  return cudaGetLastError();
}

cudaError_t emu_split_cols(const double *G, long long ld, int rows, int cols, int S, int8_t *slices, int *exps,
                           unsigned long long *colmax, int *flag, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const int Kp = emu_kpad(rows);
  cudaError_t e = cudaMemsetAsync(colmax, 0, (size_t)cols * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  emu_colmax_kernel<<<dim3((cols + 127) / 128, (rows + 255) / 256), 128, 0, st>>>(G, ld, rows, cols, colmax);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  emu_split_cols_kernel<<<dim3((cols + 31) / 32, (Kp + 127) / 128), 256, 0, st>>>(G, ld, rows, cols, Kp, S, colmax,
                                                                                 slices, exps, flag);
  return cudaGetLastError();
}

}  // namespace gi
