// tcgen05 INT8 GEMM microbenchmark, CTA-pair variant (cta_group::2): one 2-CTA cluster per 256 x 256
// output tile, M = 256 per MMA instruction, each CTA stages its own 128 A rows and 128 B rows (the
// pair shares operands, halving per-SM shared-memory operand traffic). Compare with tc_i8_gemm.cu.
//   C[M][N] (int32) = A[M][K] (int8, K-major) . B[N][K]^T (int8, K-major)
// (1-SM version:) one CTA per 128 x 256 output tile: warp 0 issues 2D TMA loads (SWIZZLE_128B boxes of 128 bytes x
// rows) into a 4-stage mbarrier ring, warp 1 (one lane) issues tcgen05.mma.cta_group::1.kind::i8
// (M = 128, N = 256, K = 32 per instruction) into a TMEM accumulator and commits each stage back to
// the ring, warps 4-7 drain TMEM with tcgen05.ld.32x32b and store int32 rows.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc_i8_gemm2 tools/tc_i8_gemm2.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int BM = 128, BN = 256, BKB = 128;  // per CTA: 128 A rows, 128 B rows (BN / 2) per stage
constexpr int STAGES = 6;
constexpr int A_BYTES = BM * BKB, B_BYTES = (BN / 2) * BKB, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NT = 256;
constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + 256;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("{\n\t.reg .b64 s;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;\n\t}\n" ::"r"(smem_u32(b)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap *m, uint64_t *bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n"
               ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa0(uint32_t saddr) {  // the same smem offset in CTA 0 of the cluster
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(r) : "r"(saddr));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// TMA into this CTA's smem, completion (bytes) signalled on the leader CTA's barrier
__device__ __forceinline__ void tma_2d_pair(uint32_t dst, const CUtensorMap *m, uint32_t bar_cluster, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
               " [%0], [%1, {%3, %4}], [%2];\n"
               ::"r"(dst), "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1) : "memory");
}
// K-major, SWIZZLE_128B canonical layout: 8-row groups 1024 B apart (SBO), LBO unused (1), version 1
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(1024 >> 4) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
// s8 x s8 -> s32, K-major A and B, M = 256 (CTA pair), N = 256
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
                           (static_cast<uint32_t>(256 >> 4) << 24);

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NT, 1)
    i8_gemm2(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb, int M, int N,
             int K, int32_t *__restrict__ C) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *accf = empty + STAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accf + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const int tm = blockIdx.y, tn = blockIdx.x / 2;
  const int nk = K / BKB;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % STAGES;
      if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
      if (rank == 0) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
      const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
      const uint32_t bar = mapa0(smem_u32(&full[s]));
      tma_2d_pair(base, &ta, bar, kt * BKB, tm * 256 + rank * BM);
      tma_2d_pair(base + A_BYTES, &tb, bar, kt * BKB, tn * BN + rank * (BN / 2));
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % STAGES;
      mbar_wait(&full[s], (kt / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
      const uint64_t da = umma_desc(base), db = umma_desc(base + A_BYTES);
#pragma unroll
      for (int k = 0; k < BKB / 32; ++k) {
        const uint32_t acc = (kt > 0 || k > 0) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
                     ::"r"(tmem), "l"(da + 2 * k), "l"(db + 2 * k), "r"(IDESC), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                   ::"r"(smem_u32(&empty[s])), "h"(static_cast<uint16_t>(3)) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n"
                 ::"r"(smem_u32(accf)), "h"(static_cast<uint16_t>(3)) : "memory");
  } else if (warp >= 4) {
    mbar_wait(accf, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    const int q = warp - 4;  // TMEM lane quarter
    const int row = tm * 256 + rank * BM + q * 32 + lane;
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t v[32];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + c0;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                     "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                     "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                     "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
      if (row < M) {
        int32_t *cr = C + static_cast<int64_t>(row) * N + tn * BN + c0;
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<int4 *>(cr + j) = make_int4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  cluster_sync();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(BN));
}

typedef CUresult (*EncFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                          const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap make_map(EncFn enc, void *p, int rows, int K, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(K)};
  cuuint32_t box[2] = {BKB, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, p, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { fprintf(stderr, "encode failed %d\n", (int)r); exit(1); }
  return m;
}

static void run(EncFn enc, int M, int N, int K, bool check, int reps) {
  std::vector<int8_t> hA(static_cast<size_t>(M) * K), hB(static_cast<size_t>(N) * K);
  uint32_t x = 12345u;
  for (auto &v : hA) { x = x * 1664525u + 1013904223u; v = static_cast<int8_t>(x >> 24); }
  for (auto &v : hB) { x = x * 1664525u + 1013904223u; v = static_cast<int8_t>(x >> 24); }
  int8_t *dA, *dB; int32_t *dC;
  CK(cudaMalloc(&dA, hA.size())); CK(cudaMalloc(&dB, hB.size()));
  CK(cudaMalloc(&dC, sizeof(int32_t) * M * N));
  CK(cudaMemcpy(dA, hA.data(), hA.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, hB.data(), hB.size(), cudaMemcpyHostToDevice));
  CUtensorMap ta = make_map(enc, dA, M, K, BM), tb = make_map(enc, dB, N, K, BN / 2);
  dim3 grid(2 * (N / BN), M / 256);
  i8_gemm2<<<grid, NT, SMEM>>>(ta, tb, M, N, K, dC);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  if (check) {
    std::vector<int32_t> hC(static_cast<size_t>(M) * N);
    CK(cudaMemcpy(hC.data(), dC, sizeof(int32_t) * M * N, cudaMemcpyDeviceToHost));
    long bad = 0;
    for (int i = 0; i < M; i += (M > 512 ? 7 : 1))
      for (int j = 0; j < N; j += (N > 512 ? 5 : 1)) {
        int64_t s = 0;
        for (int k = 0; k < K; ++k) s += int64_t(hA[size_t(i) * K + k]) * hB[size_t(j) * K + k];
        if (s != hC[size_t(i) * N + j]) {
          if (bad < 5) fprintf(stderr, "mismatch (%d,%d): %lld vs %d\n", i, j, (long long)s, hC[size_t(i) * N + j]);
          ++bad;
        }
      }
    printf("{\"check\": \"M=%d N=%d K=%d\", \"mismatches\": %ld}\n", M, N, K, bad);
  }
  if (reps > 0) {
    cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    for (int r = 0; r < reps; ++r) i8_gemm2<<<grid, NT, SMEM>>>(ta, tb, M, N, K, dC);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    const double ops = 2.0 * M * N * double(K) * reps;
    printf("{\"gemm\": \"M=%d N=%d K=%d\", \"ms\": %.3f, \"tops\": %.1f}\n", M, N, K, ms / reps, ops / (ms / 1e3) / 1e12);
  }
  cudaFree(dA); cudaFree(dB); cudaFree(dC);
}

int main(int argc, char **argv) {
  CK(cudaSetDevice(0));
  const int sustain = argc > 1 ? atoi(argv[1]) : 0;  // > 0: only the darc-like GEMM, this many reps
  void *fn = nullptr; cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncFn enc = reinterpret_cast<EncFn>(fn);
  CK(cudaFuncSetAttribute(i8_gemm2, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  if (sustain > 0) {
    run(enc, 2048, 2048, 40960, false, sustain);
    return 0;
  }
  run(enc, 256, 256, 128, true, 0);
  run(enc, 256, 512, 1024, true, 0);
  run(enc, 2048, 2048, 40960, true, 3);
  run(enc, 4096, 4096, 8192, false, 5);
  return 0;
}
