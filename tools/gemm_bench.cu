// gemm_bench.cu - microbenchmark of the per-CTA DMMA GEMM pipeline of cta_la.cuh in isolation:
// every CTA (one per SM) computes C -= A.B (or C = A.B) on its own matrices, shapes from argv.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/gemm_bench tools/gemm_bench.cu
//   tools/gemm_bench M N K [a_kc b_kc read_c]
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_1403_5524_b200/csrc/cta_la.cuh"

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
