// FP64 GEMM emulated on the INT8 tensor cores (Ozaki splitting; measurement / development tool for
// SURVEY f4, not product code):  C (fp64, M x N) = A (fp64, M x K) * B (fp64, N x K)'.
// Each row of A and of B is scaled by a power of two and split into S digits with weights 2^(1-8t)
// (the first signed, base 128; the others unsigned, base 256 -- the scheme of csrc/emu.cu), so
// C[i][j] = 2^(ea_i + eb_j) sum_g 2^(2-8g) P_g[i][j] with the exact int32 group sums
// P_g = sum_{t+u=g} a_t b_u' (tcgen05.mma.kind::i8, TMEM accumulators), groups g <= T.
// The epilogue warps turn each group's int32 tile into fp64 (exact), scale it (exact power of two)
// and accumulate it into C in global memory, largest g (smallest terms) first.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/emu_gemm tools/emu_gemm.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int BM = 128, BN = 256, BK = 128, STAGES = 4;
constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 512 + BN * 4;
constexpr int NTHREADS = 192;   // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue (TMEM lane quarters 2,3,0,1)

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(sa(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_3d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(sa(dst)),
      "l"((uint64_t)m), "r"(sa(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t idesc_i8(int as, int bs) {
  return (2u << 4) | ((uint32_t)as << 7) | ((uint32_t)bs << 10) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)(BM >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(bar))
               : "memory");
}
__device__ __forceinline__ double pow2(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }

// group sequence: g = T, T-1, .., 2; pairs t = max(1, g - S) .. min(S, g - 1), u = g - t
__global__ void __launch_bounds__(NTHREADS, 1) emu_gemm(const __grid_constant__ CUtensorMap tmA,
                                                        const __grid_constant__ CUtensorMap tmB,
                                                        const int *__restrict__ ea, const int *__restrict__ eb,
                                                        double *__restrict__ C, long long ldc, int M, int N, int K,
                                                        int S, int T) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *accfull = empty + STAGES;
  uint64_t *accempty = accfull + 2;
  uint32_t *tslot = (uint32_t *)(accempty + 2);
  int *s_eb = (int *)(smem + STAGES * STAGE_BYTES + 512);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int nk = K / BK;
  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accfull[i], 1);
      mbar_init(&accempty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int j = tid; j < BN; j += NTHREADS) s_eb[j] = n0 + j < N ? eb[n0 + j] : 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {   // TMA producer over (group, pair, k-slab)
      int it = 0;
      for (int g = T; g >= 2; --g)
        for (int t = max(1, g - S); t <= min(S, g - 1); ++t)
          for (int kb = 0; kb < nk; ++kb, ++it) {
            const int st = it % STAGES;
            if (it >= STAGES) mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1);
            uint8_t *sA = smem + st * STAGE_BYTES, *sB = sA + A_BYTES;
            mbar_expect_tx(&full[st], STAGE_BYTES);
            tma_3d(sA, &tmA, &full[st], kb * BK, m0, t - 1);
            tma_3d(sB, &tmB, &full[st], kb * BK, n0, g - t - 1);
          }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // MMA issuer
      int it = 0, q = 0;
      for (int g = T; g >= 2; --g, ++q) {
        const int buf = q & 1;
        if (q >= 2) mbar_wait(&accempty[buf], ((q >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + buf * BN;
        bool first = true;
        for (int t = max(1, g - S); t <= min(S, g - 1); ++t) {
          const uint32_t idesc = idesc_i8(t == 1, g - t == 1);
          for (int kb = 0; kb < nk; ++kb, ++it) {
            const int st = it % STAGES;
            mbar_wait(&full[st], (it / STAGES) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t a0 = sa(smem + st * STAGE_BYTES), b0 = a0 + A_BYTES;
#pragma unroll
            for (int kk = 0; kk < BK / 32; ++kk) {
              mma_i8(acc, smem_desc(a0 + 32 * kk), smem_desc(b0 + 32 * kk), idesc, first ? 0u : 1u);
              first = false;
            }
            mma_commit(&empty[st]);
          }
        }
        mma_commit(&accfull[buf]);
      }
    }
  } else {
    // epilogue warps 2..5: TMEM lane quarter (warp & 3), i.e. rows m0 + 32 (warp & 3) + lane
    const int quarter = warp & 3;
    const int row = m0 + 32 * quarter + lane;
    const int ea_r = row < M ? ea[row] : 0;
    int q = 0;
    for (int g = T; g >= 2; --g, ++q) {
      const int buf = q & 1;
      mbar_wait(&accfull[buf], (q >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int c0 = 0; c0 < BN; c0 += 32) {
        uint32_t r[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
              "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
              "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
              "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(tmem + buf * BN + ((uint32_t)(32 * quarter) << 16) + c0));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        if (row < M) {
          double *dst = C + (long long)row * ldc + n0 + c0;
#pragma unroll
          for (int j = 0; j < 32; j += 2) {
            if (n0 + c0 + j + 1 < N + 1) {
              const double v0 = (double)(int)r[j] * pow2(ea_r + s_eb[c0 + j] + 2 - 8 * g);
              const double v1 = (double)(int)r[j + 1] * pow2(ea_r + s_eb[c0 + j + 1] + 2 - 8 * g);
              double2 *d2 = (double2 *)(dst + j);
              if (q == 0) {
                *d2 = make_double2(v0, v1);
              } else {
                double2 o = *d2;
                *d2 = make_double2(o.x + v0, o.y + v1);
              }
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&accempty[buf]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// ------------------------------------------------------------------------------------------- host
static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;

static CUtensorMap make_map(const int8_t *p, int rows, int K, int S, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)S};
  cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)K * rows};
  cuuint32_t box[3] = {BK, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void *)p, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

// row-wise split of X (rows x K) into S int8 slices [S][rows][K] and exponents
// row-wise split of X (rows x K) into S digit slices [S][rows][K] (digit 1 signed, base 128; later
// digits unsigned, base 256: weights 2^(1-8t)) and exponents (max |x| < 2^e)
static void split_host(const std::vector<double> &X, int rows, int K, int S, std::vector<int8_t> &sl,
                       std::vector<int> &e) {
  sl.assign((size_t)S * rows * K, 0);
  e.assign(rows, 0);
  for (int i = 0; i < rows; ++i) {
    double mx = 0;
    for (int k = 0; k < K; ++k) mx = std::max(mx, std::fabs(X[(size_t)i * K + k]));
    int ex = 0;
    if (mx > 0) std::frexp(mx, &ex);
    e[i] = ex;
    for (int k = 0; k < K; ++k) {
      double v = std::ldexp(X[(size_t)i * K + k], -ex);
      for (int t = 0; t < S; ++t) {
        const double y = v * (t == 0 ? 128.0 : 256.0);
        const double d = std::floor(y);
        sl[((size_t)t * rows + i) * K + k] = (int8_t)(uint8_t)(int)d;
        v = y - d;
      }
    }
  }
}

int main(int argc, char **argv) {
  cudaDriverEntryPointQueryResult qr;
  void *fn = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int S = 7, T = argc > 1 ? atoi(argv[1]) : 9;
  for (int pass = 0; pass < 2; ++pass) {
    const int M = pass ? 4096 : 256, N = pass ? (argc > 2 ? atoi(argv[2]) : 32768) : 512, K = pass ? 4096 : 4096;
    std::vector<double> A((size_t)M * K), B((size_t)N * K);
    unsigned s = 7;
    auto rnd = [&]() {
      s = s * 1664525u + 1013904223u;
      return ((s >> 8) / 16777216.0) * 2 - 1;
    };
    for (auto &v : A) v = rnd() * std::exp(3 * rnd());
    for (auto &v : B) v = rnd();
    std::vector<int8_t> As, Bs;
    std::vector<int> ea, eb;
    split_host(A, M, K, S, As, ea);
    split_host(B, N, K, S, Bs, eb);
    int8_t *dA, *dB;
    int *dea, *deb;
    double *dC;
    cudaMalloc(&dA, As.size());
    cudaMalloc(&dB, Bs.size());
    cudaMalloc(&dea, M * 4);
    cudaMalloc(&deb, N * 4);
    cudaMalloc(&dC, (size_t)M * N * 8);
    cudaMemcpy(dA, As.data(), As.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bs.data(), Bs.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dea, ea.data(), M * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(deb, eb.data(), N * 4, cudaMemcpyHostToDevice);
    CUtensorMap ta = make_map(dA, M, K, S, BM), tb = make_map(dB, N, K, S, BN);
    cudaFuncSetAttribute(emu_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    dim3 grid(M / BM, N / BN);
    emu_gemm<<<grid, NTHREADS, SMEM>>>(ta, tb, dea, deb, dC, N, M, N, K, S, T);
    cudaError_t err = cudaDeviceSynchronize();
    if (err != cudaSuccess) {
      printf("kernel error %s\n", cudaGetErrorString(err));
      return 1;
    }
    if (!pass) {
      std::vector<double> C((size_t)M * N);
      cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost);
      double worst = 0, worst_abs = 0;
      for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
          long double ref = 0, mag = 0;
          for (int k = 0; k < K; ++k) {
            ref += (long double)A[(size_t)i * K + k] * B[(size_t)j * K + k];
            mag += std::fabs((long double)A[(size_t)i * K + k] * B[(size_t)j * K + k]);
          }
          const double err_ = (double)std::fabs((long double)C[(size_t)i * N + j] - ref);
          worst = std::max(worst, err_ / (double)mag);
          worst_abs = std::max(worst_abs, err_);
        }
      printf("check %dx%dx%d S=%d T=%d: max |C - C_exact| / sum|a b| = %.3e\n", M, N, K, S, T, worst);
    } else {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      const int reps = 5;
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) emu_gemm<<<grid, NTHREADS, SMEM>>>(ta, tb, dea, deb, dC, N, M, N, K, S, T);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= reps;
      int pairs = 0;
      for (int g = T; g >= 2; --g)
        for (int t = std::max(1, g - S); t <= std::min(S, g - 1); ++t) ++pairs;
      printf("%d x %d x %d fp64-emulated (S=%d, T=%d, %d int8 products): %.3f ms, %.1f TFLOP/s fp64-equivalent, "
             "%.0f int8 TOPS\n",
             M, N, K, S, T, pairs, ms, 2.0 * M * N * K / (ms * 1e-3) / 1e12,
             2.0 * M * N * K * pairs / (ms * 1e-3) / 1e12);
    }
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dea);
    cudaFree(deb);
    cudaFree(dC);
  }
  return 0;
}
