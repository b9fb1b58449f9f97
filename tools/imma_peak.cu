// Legacy (mma.sync) tensor-core peak microbenchmark on sm_100a: INT8 m16n8k32 and BF16 m16n8k16,
// independent accumulator chains per warp. Decides whether an Ozaki-style FP64 emulation of the
// R contraction on integer tensor cores could beat FP64 DMMA without tcgen05.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imma_peak tools/imma_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void imma(int (&d)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3,
                                     unsigned b0, unsigned b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void hmma(float (&d)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3,
                                     unsigned b0, unsigned b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__global__ void k_imma(int *out, int iters, unsigned x) {
  int c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = threadIdx.x + i;
  unsigned a0 = x ^ threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) imma(c[j], a0, a1, a2, a3, b0, b1);
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 123456789) out[0] = s;
}

__global__ void k_hmma(int *out, int iters, unsigned x) {
  float c[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = threadIdx.x + i;
  unsigned a0 = 0x3c003c00u, a1 = a0, a2 = a0, a3 = a0, b0 = a0, b1 = a0 ^ (x & 1);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) hmma(c[j], a0, a1, a2, a3, b0, b1);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 1234.5f) out[0] = 1;
}

int main(int argc, char **argv) {
  CK(cudaSetDevice(0));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int nsm = p.multiProcessorCount;
  int *out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int iters = argc > 1 ? atoi(argv[1]) : 20000;
  for (int kind = 0; kind < 2; ++kind)
    for (int bps = 1; bps <= 4; bps *= 2)
      for (int threads = 256; threads <= 512; threads *= 2) {
        dim3 grid(nsm * bps), block(threads);
        for (int w = 0; w < 2; ++w) {
          if (kind == 0) k_imma<<<grid, block>>>(out, iters / 10, 7); else k_hmma<<<grid, block>>>(out, iters / 10, 7);
        }
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        if (kind == 0) k_imma<<<grid, block>>>(out, iters, 7); else k_hmma<<<grid, block>>>(out, iters, 7);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
        const double macs_per = kind == 0 ? 16.0 * 8 * 32 : 16.0 * 8 * 16;
        double ops = 2.0 * macs_per * 8 * iters * (double)grid.x * (threads / 32);
        printf("{\"kind\": \"%s\", \"blocks_per_sm\": %d, \"threads\": %d, \"tops\": %.1f}\n",
               kind == 0 ? "imma_s8_m16n8k32" : "hmma_bf16_m16n8k16", bps, threads, ops / (ms / 1e3) / 1e12);
      }
  return 0;
}
