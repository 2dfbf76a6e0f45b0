// tcgen05 INT8 GEMM probe (measurement tool for SURVEY f4's FP64-emulation question, not product
// code): C (int32, M x N) = A (int8, M x K, K contiguous) * B (int8, N x K, K contiguous)'.
// One 128 x 256 tile per CTA, K in 128-byte slabs through a 4-stage TMA ring (SWIZZLE_128B),
// one elected thread issues tcgen05.mma.kind::i8 (M = 128, N = 256, K = 32) into a TMEM accumulator,
// tcgen05.commit releases the stage; the 4 warps read the accumulator back with tcgen05.ld.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8gemm tools/i8gemm.cu
//   ./tools/i8gemm              (checks a small case against the host, then times 8192 x 8192 x 16384)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

constexpr int BM = 128, BN = 256, BK = 128, STAGES = 4;
constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int TMEM_COLS = 256;

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra W_%=;\n}\n" ::"r"(sa(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_2d(void *dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
      ::"r"(sa(dst)), "l"((uint64_t)m), "r"(sa(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// K-major operand tile, 128-byte rows, 8-row swizzle atoms of 1024 bytes (SBO), SWIZZLE_128B
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;             // LBO (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;   // SBO
  d |= (uint64_t)1 << 46;             // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;             // SWIZZLE_128B
  return d;
}
// kind::i8 instruction descriptor: D s32, A/B signed, K-major both, N = 256, M = 128
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(bar))
               : "memory");
}

__global__ void __launch_bounds__(128, 1) i8gemm(const __grid_constant__ CUtensorMap tmA,
                                                 const __grid_constant__ CUtensorMap tmB, int32_t *C, int M, int N,
                                                 int K) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t *full = (uint64_t *)(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *done = empty + STAGES;
  uint32_t *tslot = (uint32_t *)(done + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * BM;
  const int nk = K / BK;
  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa(tslot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;

  if (warp == 0 && lane == 0) {            // TMA producer
    for (int it = 0; it < nk; ++it) {
      const int st = it % STAGES;
      if (it >= STAGES) mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1);
      uint8_t *sA = smem + st * STAGE_BYTES, *sB = sA + A_BYTES;
      mbar_expect_tx(&full[st], STAGE_BYTES);
      tma_2d(sA, &tmA, &full[st], it * BK, m0);
      tma_2d(sB, &tmB, &full[st], it * BK, n0);
    }
  } else if (warp == 1 && lane == 0) {     // MMA issuer
    for (int it = 0; it < nk; ++it) {
      const int st = it % STAGES;
      mbar_wait(&full[st], (it / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = sa(smem + st * STAGE_BYTES), b0 = a0 + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < BK / 32; ++kk)
        mma_i8(tmem, smem_desc(a0 + 32 * kk), smem_desc(b0 + 32 * kk), (it | kk) != 0);
      mma_commit(&empty[st]);              // the stage is free once these MMAs have read it
    }
    mma_commit(done);
  }
  __syncwarp();
  // epilogue: warp w reads TMEM lanes 32w .. 32w+31 (rows m0 + 32w + lane)
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = m0 + 32 * warp + lane;
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem + ((uint32_t)(32 * warp) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (row < M) {
      int4 *dst = (int4 *)(C + (long long)row * N + n0 + c0);
#pragma unroll
      for (int q = 0; q < 8; ++q) dst[q] = make_int4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;

static CUtensorMap make_map(const int8_t *p, int rows, int K, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K};
  cuuint32_t box[2] = {BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, (void *)p, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    printf("encode failed %d\n", (int)r);
    exit(1);
  }
  return m;
}

static float run(int M, int N, int K, bool check, int reps) {
  std::vector<int8_t> hA((size_t)M * K), hB((size_t)N * K);
  unsigned s = 1;
  for (auto &v : hA) { s = s * 1664525u + 1013904223u; v = (int8_t)((s >> 24) & 0xff); }
  for (auto &v : hB) { s = s * 1664525u + 1013904223u; v = (int8_t)((s >> 24) & 0xff); }
  int8_t *A, *B;
  int32_t *C;
  cudaMalloc(&A, hA.size());
  cudaMalloc(&B, hB.size());
  cudaMalloc(&C, (size_t)M * N * 4);
  cudaMemcpy(A, hA.data(), hA.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB.data(), hB.size(), cudaMemcpyHostToDevice);
  CUtensorMap ta = make_map(A, M, K, BM), tb = make_map(B, N, K, BN);
  cudaFuncSetAttribute(i8gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  dim3 grid(N / BN, M / BM);
  i8gemm<<<grid, 128, SMEM>>>(ta, tb, C, M, N, K);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("kernel error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  if (check) {
    std::vector<int32_t> hC((size_t)M * N);
    cudaMemcpy(hC.data(), C, hC.size() * 4, cudaMemcpyDeviceToHost);
    long long bad = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        int32_t acc = 0;
        for (int k = 0; k < K; ++k) acc += (int32_t)hA[(size_t)i * K + k] * (int32_t)hB[(size_t)j * K + k];
        if (acc != hC[(size_t)i * N + j] && bad++ < 5)
          printf("mismatch (%d,%d): %d vs %d\n", i, j, hC[(size_t)i * N + j], acc);
      }
    printf("check %dx%dx%d: %lld mismatches\n", M, N, K, bad);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) i8gemm<<<grid, 128, SMEM>>>(ta, tb, C, M, N, K);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  cudaFree(A);
  cudaFree(B);
  cudaFree(C);
  return ms;
}

int main() {
  cudaDriverEntryPointQueryResult q;
  void *fn = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  run(256, 512, 512, true, 1);
  run(384, 768, 1024, true, 1);
  const int M = 8192, N = 8192, K = 16384;
  const float ms = run(M, N, K, false, 10);
  printf("%d x %d x %d int8: %.3f ms, %.1f TOPS\n", M, N, K, ms, 2.0 * M * N * K / (ms * 1e-3) / 1e12);
  return 0;
}
