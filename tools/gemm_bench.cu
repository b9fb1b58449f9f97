// gemm_bench.cu - microbenchmark of the per-CTA DMMA GEMM pipeline of cta_la.cuh in isolation:
// every CTA (one per SM) computes C -= A.B (or C = A.B) on its own matrices, shapes from argv.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gemm_bench tools/gemm_bench.cu
//   tools/gemm_bench M N K [a_kc b_kc read_c [mode]]   mode 2: the 8-warp 128x128 prototype
//   (gemm2_proto.cuh; C = A.B only), checked against la::gemm_set on the same random inputs
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1403_5524_b200/csrc/cta_la.cuh"
#include "gemm2_proto.cuh"

using namespace rmx;
using namespace rmx::la;

struct BenchSmem {
  double gemm[GEMM_SMEM_DOUBLES];
  GemmSync gs;
};

__global__ void __launch_bounds__(NT, 1) bench_kernel(double *ws, int64_t slot, int ld, int M, int N, int K,
                                                      const CUtensorMap *maps, bool akc, bool bkc,
                                                      bool readc, int reps) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  BenchSmem &sm = *reinterpret_cast<BenchSmem *>(smem_raw);
  double *base = ws + blockIdx.x * slot;
  const int64_t msz = static_cast<int64_t>(2048) * ld;
  const MatView A{maps + (blockIdx.x * 3 + 0) * NVIEW, base, ld};
  const MatView B{maps + (blockIdx.x * 3 + 1) * NVIEW, base + msz, ld};
  const MatView C{maps + (blockIdx.x * 3 + 2) * NVIEW, base + 2 * msz, ld};
  for (int r = 0; r < reps; ++r) {
    const Op a{A, 0, 0, akc}, b{B, 0, 0, bkc};
    if (readc)
      gemm_sub(M, N, K, a, b, C, 0, 0, false, sm.gemm, &sm.gs);
    else
      gemm_set(M, N, K, a, b, C, 0, 0, false, 0.0, sm.gemm, &sm.gs);
  }
}

template <bool AK, bool BK_>
__global__ void __launch_bounds__(proto::NT2, 1) bench2_kernel(double *ws, int64_t slot, int ld, int M, int N, int K,
                                                              const CUtensorMap *maps, int reps, int64_t cofs, bool readc_ = false) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t *al = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  proto::Sync2 *sy = reinterpret_cast<proto::Sync2 *>(al + proto::ST2 * proto::STAGE2);
  double *base = ws + blockIdx.x * slot;
  const int64_t msz = static_cast<int64_t>(2048) * ld;
  const MatView A{maps + (blockIdx.x * 3 + 0) * NVIEW, base, ld};
  const MatView B{maps + (blockIdx.x * 3 + 1) * NVIEW, base + msz, ld};
  for (int r = 0; r < reps; ++r) {
    if (cofs < 0) {  // mode 3: the full-featured variant behind a non-inlined call (C read when readc_)
      GemmArgs ga{Op{A, 0, 0, AK}, Op{B, 0, 0, BK_}, base - cofs, ld, M, N, K, false, readc_, false, 0.0};
      proto::gemm3_call<AK, BK_>(ga, al, sy);
    } else {
      proto::gemm2_set<AK, BK_>(M, N, K, Op{A, 0, 0, AK}, Op{B, 0, 0, BK_}, base + cofs, ld, al, sy);
    }
  }
}
__global__ void fill_kernel(double *p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull;
    x ^= x >> 29; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 32;
    p[i] = (double)(x >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
}

typedef CUresult (*PFN_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                          const cuuint64_t *, const cuuint32_t *, const cuuint32_t *,
                          CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                          CUtensorMapFloatOOBfill);

int main(int argc, char **argv) {
  int M = argc > 1 ? atoi(argv[1]) : 2000, N = argc > 2 ? atoi(argv[2]) : 2000,
      K = argc > 3 ? atoi(argv[3]) : 64;
  bool akc = argc > 4 ? atoi(argv[4]) : 1, bkc = argc > 5 ? atoi(argv[5]) : 0,
       readc = argc > 6 ? atoi(argv[6]) : 1;
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int ld = 2048 + 8;
  const int64_t msz = 2048LL * ld, slot = 3 * msz + 64;
  double *ws;
  cudaMalloc(&ws, slot * nsm * 8);
  cudaMemset(ws, 0, slot * nsm * 8);
  void *fp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  PFN_t enc = (PFN_t)fp;
  std::vector<CUtensorMap> h(nsm * 3 * NVIEW);
  const int boxr[3] = {128, 64, 32};
  for (int s = 0; s < nsm; ++s)
    for (int m = 0; m < 3; ++m)
      for (int v = 0; v < 3; ++v) {
        cuuint64_t dims[2] = {(cuuint64_t)ld, 2048}, str[1] = {(cuuint64_t)ld * 8};
        cuuint32_t box[2] = {16, (cuuint32_t)boxr[v]}, es[2] = {1, 1};
        enc(&h[(s * 3 + m) * 3 + v], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, ws + s * slot + m * msz, dims,
            str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      }
  CUtensorMap *dm;
  cudaMalloc(&dm, h.size() * sizeof(CUtensorMap));
  cudaMemcpy(dm, h.data(), h.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(bench_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, sizeof(BenchSmem));
  const int mode = argc > 7 ? atoi(argv[7]) : 0;
  if (mode == 2 || mode == 3) {
    // C_ref = A.B by la::gemm_set into rows 0.. of the C matrix, C_new by the prototype into rows
    // 1024.. of it (requires M <= 1024); same random A, B
    fill_kernel<<<1024, 256>>>(ws, slot * nsm);
    cudaDeviceSynchronize();
    auto launch2 = [&](int reps, int64_t cofs) {
      if (akc && bkc) {
        cudaFuncSetAttribute(bench2_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, proto::SMEM2);
        bench2_kernel<true, true><<<nsm, proto::NT2, proto::SMEM2>>>(ws, slot, ld, M, N, K, dm, reps, cofs, readc);
      } else if (akc) {
        cudaFuncSetAttribute(bench2_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, proto::SMEM2);
        bench2_kernel<true, false><<<nsm, proto::NT2, proto::SMEM2>>>(ws, slot, ld, M, N, K, dm, reps, cofs, readc);
      } else if (bkc) {
        cudaFuncSetAttribute(bench2_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, proto::SMEM2);
        bench2_kernel<false, true><<<nsm, proto::NT2, proto::SMEM2>>>(ws, slot, ld, M, N, K, dm, reps, cofs, readc);
      } else {
        cudaFuncSetAttribute(bench2_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, proto::SMEM2);
        bench2_kernel<false, false><<<nsm, proto::NT2, proto::SMEM2>>>(ws, slot, ld, M, N, K, dm, reps, cofs, readc);
      }
    };
    const int64_t c_ref = 2 * msz, c_new = (mode == 3 ? -1 : 1) * (2 * msz + 1024LL * ld);
    bench_kernel<<<nsm, NT, sizeof(BenchSmem)>>>(ws, slot, ld, M, N, K, dm, akc, bkc, false, 1);
    launch2(1, c_new);
    cudaDeviceSynchronize();
    std::vector<double> h1(static_cast<size_t>(M) * ld), h2(static_cast<size_t>(M) * ld);
    double maxd = 0.0, maxv = 0.0;
    for (int s = 0; s < nsm; s += 37) {
      cudaMemcpy(h1.data(), ws + s * slot + c_ref, sizeof(double) * M * ld, cudaMemcpyDeviceToHost);
      cudaMemcpy(h2.data(), ws + s * slot + (c_new < 0 ? -c_new : c_new), sizeof(double) * M * ld, cudaMemcpyDeviceToHost);
      for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
          maxd = fmax(maxd, fabs(h1[(size_t)i * ld + j] - h2[(size_t)i * ld + j]));
          maxv = fmax(maxv, fabs(h1[(size_t)i * ld + j]));
        }
    }
    const int reps2 = 4;
    cudaEvent_t f0, f1;
    cudaEventCreate(&f0);
    cudaEventCreate(&f1);
    float ms_old, ms_new;
    cudaEventRecord(f0);
    bench_kernel<<<nsm, NT, sizeof(BenchSmem)>>>(ws, slot, ld, M, N, K, dm, akc, bkc, readc, reps2);
    cudaEventRecord(f1);
    cudaEventSynchronize(f1);
    cudaEventElapsedTime(&ms_old, f0, f1);
    cudaEventRecord(f0);
    launch2(reps2, c_new);
    cudaEventRecord(f1);
    cudaEventSynchronize(f1);
    cudaEventElapsedTime(&ms_new, f0, f1);
    const double fl2 = 2.0 * M * N * K * reps2 * nsm;
    printf("{\"M\":%d,\"N\":%d,\"K\":%d,\"akc\":%d,\"bkc\":%d,\"tflops_9warp_128x64\":%.2f,"
           "\"tflops_8warp_128x128\":%.2f,\"max_abs_diff\":%.3e,\"max_abs\":%.3e,\"err\":\"%s\"}\n",
           M, N, K, akc, bkc, fl2 / ms_old / 1e9, fl2 / ms_new / 1e9, maxd, maxv,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
  }
  const int reps = 4;
  bench_kernel<<<nsm, NT, sizeof(BenchSmem)>>>(ws, slot, ld, M, N, K, dm, akc, bkc, readc, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench_kernel<<<nsm, NT, sizeof(BenchSmem)>>>(ws, slot, ld, M, N, K, dm, akc, bkc, readc, reps);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * M * N * K * reps * nsm;
  printf("{\"M\":%d,\"N\":%d,\"K\":%d,\"akc\":%d,\"bkc\":%d,\"readc\":%d,\"ms\":%.3f,\"tflops\":%.2f,\"err\":\"%s\"}\n",
         M, N, K, akc, bkc, readc, ms, fl / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
