// a7 on the INT8 tensor cores (opt-in: geninv_set_emulation): the FP64 product
// C = X G' emulated by Ozaki splitting (DESIGN.md §6 "FP64 emulation").
//
// Every row of X (and of G) is scaled by a power of two 2^e (|x| 2^-e <= 127/128) and split into S
// int8 digits, x = 2^e sum_{t=1..S} d_t 2^-7t + r with |r| <= 2^(e - 7S - 1) (error-free: each step
// y = 128 v, d = rint(y), v = y - d is exact in FP64).  Then
//   C[i][j] = 2^(e_i + f_j) sum_g 2^-7g P_g[i][j],  P_g = sum_{t+u=g} sum_k d_t[i][k] d'_u[j][k]
// with every P_g an exact int32 sum (|P_g| <= S K 127^2 < 2^31 for K < 16384) computed by
// tcgen05.mma.kind::i8 into TMEM.  Groups g = T .. 2 (smallest terms first) are converted exactly to
// FP64, scaled exactly (powers of two) and accumulated into C in FP64.  S = 8, T = 9 (36 int8
// products) leaves |C - C_exact| <~ 4e-17 sum_k |x_ik g_jk| (tools/emu_gemm.cu), i.e. below an FP64
// GEMM's own rounding bound.
//
// Kernel layout (one 128 x 256 tile of C per CTA, 192 threads): warp 0 lane 0 issues the TMA loads
// (128-byte K slabs of the slice arrays, SWIZZLE_128B, 4-stage ring), warp 1 lane 0 issues the MMAs
// (M = 128, N = 256, K = 32) into one of two TMEM accumulators (2 x 256 columns, ping-pong by group),
// warps 2-5 (one TMEM lane quarter each) drain a finished group into C while the next one runs.
#include <cudaTypedefs.h>
#include <stdio.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "emu.h"

namespace gi {

namespace {

constexpr int EBM = 128, EBN = 256, EBK = 128, ESTAGES = 4;
constexpr int EA_BYTES = EBM * EBK, EB_BYTES = EBN * EBK, ESTAGE_BYTES = EA_BYTES + EB_BYTES;
constexpr int ESMEM = ESTAGES * ESTAGE_BYTES + 1024 + 512 + EBN * 4;
constexpr int ENT = 192;
constexpr uint32_t IDESC_I8 =
    (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(EBN >> 3) << 17) | ((uint32_t)(EBM >> 4) << 24);

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
GI_DEV void mma_i8(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(IDESC_I8), "r"(acc));
}
GI_DEV void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
GI_DEV double pow2i(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }   // 2^e, |e| <= 1022

// Persistent: CTA c takes tiles c, c + gridDim.x, ... (tile = m-tile fastest, so CTAs working at the
// same time share the B slices of one n-tile); the stage ring, the TMEM ping-pong and the scratch tile
// carry over from one tile to the next, so a tile's last epilogue overlaps the next tile's MMAs.
__global__ void __launch_bounds__(ENT, 1) emu_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                          const __grid_constant__ CUtensorMap tmB,
                                                          const int *__restrict__ ea, const int *__restrict__ eb,
                                                          double *__restrict__ C, long long ldc, int M, int N,
                                                          int Kp, int S, int T, double *__restrict__ scratch) {
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
  const int mt = (M + EBM - 1) / EBM, ntiles = mt * ((N + EBN - 1) / EBN);
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
        const int m0 = (tile % mt) * EBM, n0 = (tile / mt) * EBN;
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
          for (int t = max(1, g - S); t <= min(S, g - 1); ++t)
            for (int kb = 0; kb < nk; ++kb, ++it) {
              const int st = it % ESTAGES;
              mbar_wait(&full[st], (it / ESTAGES) & 1);
              asm volatile("tcgen05.fence::after_thread_sync;");
              const uint32_t a0 = smem_u32(smem + st * ESTAGE_BYTES), b0 = a0 + EA_BYTES;
#pragma unroll
              for (int kk = 0; kk < EBK / 32; ++kk) {
                mma_i8(acc, umma_desc(a0 + 32 * kk), umma_desc(b0 + 32 * kk), accumulate);
                accumulate = 1;
              }
              mma_commit(&empty[st]);   // the stage is free once these MMAs have read it
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
      const int m0 = (tile % mt) * EBM, n0 = (tile / mt) * EBN;
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
        const double sr = pow2i(ea_r - 7 * g);
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
#pragma unroll
              for (int j = 0; j < 16; ++j) d2[j] = make_double2(o[2 * j], o[2 * j + 1]);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (nb + j < N) crow[nb + j] = o[j];
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
  if (mx > 0.0) {
    frexp(mx * (128.0 / 127.0), &e);                // mx 128/127 < 2^e
    if (!(mx * (128.0 / 127.0) < ldexp(1.0, e))) ++e;
  }
  if (!isfinite(mx) || e < -900 || e > 900) {
    if (lane == 0) atomicOr(flag, 1);
    e = 0;
  }
  if (lane == 0) ex[warp] = e;
  const double inv = ldexp(1.0, -e);
  const long long plane = (long long)rows * Kp;
  int8_t *out = sl + (long long)warp * Kp;
  for (int k0 = 4 * lane; k0 < Kp; k0 += 128) {
    double v[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) v[q] = (k0 + q < K) ? x[k0 + q] * inv : 0.0;
    for (int t = 0; t < S; ++t) {
      char4 c;
      signed char d[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double y = v[q] * 128.0;
        const double r = rint(y);
        d[q] = (signed char)(int)r;
        v[q] = y - r;
      }
      c.x = d[0]; c.y = d[1]; c.z = d[2]; c.w = d[3];
      if (k0 + 3 < Kp) *reinterpret_cast<char4 *>(out + t * plane + k0) = c;
      else
        for (int q = 0; q < 4 && k0 + q < Kp; ++q) out[t * plane + k0 + q] = d[q];
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

int num_sms_emu() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

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

static int emu_ctas(int M, int N) {
  const long long tiles = (long long)((M + EBM - 1) / EBM) * ((N + EBN - 1) / EBN);
  return (int)std::min<long long>(tiles, num_sms_emu());
}

long long emu_scratch_elems(int M, int N) { return (long long)emu_ctas(M, N) * EBM * EBN; }

cudaError_t emu_gemm_nt(const int8_t *As, const int *ea, int M, const int8_t *Bs, const int *eb, int N, int K, int S,
                        int T, double *C, long long ldc, double *scratch, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  const int Kp = emu_kpad(K);
  CUtensorMap ta, tb;
  cudaError_t e = slice_map(&ta, As, M, Kp, S, EBM);
  if (e != cudaSuccess) return e;
  if ((e = slice_map(&tb, Bs, N, Kp, S, EBN)) != cudaSuccess) return e;
  static bool attr = false;
  if (!attr) {
    if ((e = cudaFuncSetAttribute(emu_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ESMEM)) != cudaSuccess)
      return e;
    attr = true;
  }
  emu_gemm_kernel<<<emu_ctas(M, N), ENT, ESMEM, st>>>(ta, tb, ea, eb, C, ldc, M, N, Kp, S, T, scratch);
  return cudaGetLastError();
}

}  // namespace gi
