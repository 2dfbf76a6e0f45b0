// Host launcher + instantiations of the FP64 DMMA GEMM core (gemm.cuh).
#include <cudaTypedefs.h>
#include <stdio.h>

#include <algorithm>
#include <mutex>

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
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
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

template <int BM, int BN, int WM, int WN, int ST, bool AK, bool BK_>
static cudaError_t launch(const GemmOp &op, GemmArgs &a, cudaStream_t st) {
  using Cfg = GemmCfg<BM, BN, WM, WN, ST, AK, BK_>;
  auto kern = dgemm_tc<BM, BN, WM, WN, ST, AK, BK_>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  cudaError_t e;
  a.a_mn4d = !AK && (op.A.cols % 16 == 0) && (op.a_mn0 % 16 == 0);
  a.b_mn4d = !BK_ && (op.B.cols % 16 == 0) && (op.b_mn0 % 16 == 0);
  e = a.a_mn4d ? make_map_mn4d(&a.tmA, op.A, BM / 16) : make_map(&a.tmA, op.A, AK ? BM : 16);
  if (e != cudaSuccess) return e;
  e = a.b_mn4d ? make_map_mn4d(&a.tmB, op.B, BN / 16) : make_map(&a.tmB, op.B, BK_ ? BN : 16);
  if (e != cudaSuccess) return e;
  a.mtiles = (op.M + BM - 1) / BM;
  a.ntiles = (op.N + BN - 1) / BN;
  {
    // raster band: at most ~48 MB of A rows (BM x K doubles per M-tile) per band, bands balanced
    const long long per_tile = (long long)BM * (op.K > 0 ? op.K : 1) * 8;
    long long mb = std::max<long long>(1, (48LL << 20) / per_tile);
    const long long nb = (a.mtiles + mb - 1) / mb;
    a.mband = (int)((a.mtiles + nb - 1) / nb);
  }
  long long tiles = op.lower ? (long long)a.mtiles * (a.mtiles + 1) / 2 : (long long)a.mtiles * a.ntiles;
  if (tiles == 0) return cudaSuccess;
  dim3 grid((unsigned)tiles, op.splits, op.batch);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>(a);
  return cudaGetLastError();
}

cudaError_t gemm(const GemmOp &op, cudaStream_t st) {
  if (op.M <= 0 || op.N <= 0) return cudaSuccess;
  if (op.lower && op.M != op.N) return cudaErrorInvalidValue;
  GemmArgs a;
  memset(&a, 0, sizeof(a));
  a.a_mn0 = op.a_mn0; a.a_k0 = op.a_k0; a.b_mn0 = op.b_mn0; a.b_k0 = op.b_k0;
  a.C = op.C; a.ldc = op.ldc; a.c_bstride = op.c_bstride; a.split_stride = op.split_stride;
  a.C0 = op.C0; a.ldc0 = op.ldc0; a.c0_bstride = op.c0_bstride;
  a.alpha = op.alpha; a.M = op.M; a.N = op.N; a.K = op.K; a.K_dev = op.K_dev;
  a.k_lo_mode = op.k_lo_mode; a.k_hi_mode = op.k_hi_mode; a.k_lo_dev = op.k_lo_dev;
  a.lower = op.lower; a.mirror = op.mirror; a.splits = op.splits < 1 ? 1 : op.splits;
  if (op.tile == TILE_128x32) {
    if (op.a_kmajor && op.b_kmajor) return launch<128, 32, 32, 32, 6, true, true>(op, a, st);
    if (op.a_kmajor && !op.b_kmajor) return launch<128, 32, 32, 32, 6, true, false>(op, a, st);
    if (!op.a_kmajor && op.b_kmajor) return launch<128, 32, 32, 32, 6, false, true>(op, a, st);
    return launch<128, 32, 32, 32, 6, false, false>(op, a, st);
  }
  if (op.a_kmajor && op.b_kmajor) return launch<128, 128, 64, 32, 6, true, true>(op, a, st);
  if (op.a_kmajor && !op.b_kmajor) return launch<128, 128, 64, 32, 6, true, false>(op, a, st);
  if (!op.a_kmajor && op.b_kmajor) return launch<128, 128, 64, 32, 6, false, true>(op, a, st);
  return launch<128, 128, 64, 32, 6, false, false>(op, a, st);
}

// ---------------------------------------------------------------- split-K reduction
__global__ void splitk_reduce_kernel(const double *__restrict__ P, long long sstride, int splits, long long ldp,
                                     double *__restrict__ out, long long ldo, const double *__restrict__ C0,
                                     long long ldc0, double alpha, int M, int N, int lower) {
  const long long total = (long long)M * N;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(idx / N), j = (int)(idx % N);
    if (lower && j > i) continue;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += P[z * sstride + (long long)i * ldp + j];
    double v = alpha * s;
    if (C0) v += C0[(long long)i * ldc0 + j];
    out[(long long)i * ldo + j] = v;
  }
}

cudaError_t splitk_reduce(const double *P, long long split_stride, int splits, long long ldp, double *out,
                          long long ldo, const double *C0, long long ldc0, double alpha, int M, int N, bool lower,
                          cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  long long total = (long long)M * N;
  int blocks = (int)std::min<long long>((total + 255) / 256, (long long)num_sms() * 16);
  splitk_reduce_kernel<<<blocks, 256, 0, st>>>(P, split_stride, splits, ldp, out, ldo, C0, ldc0, alpha, M, N,
                                               lower ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace gi
