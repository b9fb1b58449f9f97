// FP64 peak microbenchmark for the roofline denominator (SURVEY.md §7 "Hard parts" 1, §8(d)).
// MEASURED_PEAKS.json carries no FP64 figure, so the R-formation kernel's "frac" is taken
// against the numbers this program prints on the bench box:
//   dfma   : independent DFMA chains, 8 per thread            -> FP64 pipe peak
//   dmma   : independent mma.sync.m8n8k4.f64 chains, 8/warp   -> FP64 tensor (DMMA) peak
//   mixed  : one DMMA + one DMUL per step                     -> do DMMA and DFMA share a pipe?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void k_dfma(double *out, int iters, double b, double c) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3,
         a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double *out, int iters, double a, double b) {
  double c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = threadIdx.x + i;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(c[2 * j], c[2 * j + 1], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_mixed(double *out, int iters, double a, double b) {
  double c[16];
  double m0 = threadIdx.x, m1 = m0 + 1, m2 = m0 + 2, m3 = m0 + 3;
#pragma unroll
  for (int i = 0; i < 16; ++i) c[i] = threadIdx.x + i;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) dmma(c[2 * j], c[2 * j + 1], a, b);
      m0 = fma(m0, a, b); m1 = fma(m1, a, b); m2 = fma(m2, a, b); m3 = fma(m3, a, b);
    }
  }
  double s = m0 + m1 + m2 + m3;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

int main(int argc, char **argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int nsm = p.multiProcessorCount;
  double *out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  int iters = argc > 1 ? atoi(argv[1]) : 4000;
  const int reps = 5;
  for (int blocks_per_sm = 1; blocks_per_sm <= 4; blocks_per_sm *= 2) {
    for (int threads = 256; threads <= 512; threads *= 2) {
      dim3 grid(nsm * blocks_per_sm), block(threads);
      // DFMA
      k_dfma<<<grid, block>>>(out, 10, 1.0000001, 1e-9); CK(cudaDeviceSynchronize());
      float best = 1e30f;
      for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(e0)); k_dfma<<<grid, block>>>(out, iters, 1.0000001, 1e-9);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
      }
      double fl = 2.0 * 64.0 * iters * (double)grid.x * threads;
      printf("{\"kernel\":\"dfma\",\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n",
             blocks_per_sm, threads, best, fl / best / 1e9);
      // DMMA
      k_dmma<<<grid, block>>>(out, 10, 1.0, 1e-9); CK(cudaDeviceSynchronize());
      best = 1e30f;
      int it2 = iters / 4;
      for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(e0)); k_dmma<<<grid, block>>>(out, it2, 1.0, 1e-9);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
      }
      double nwarps = (double)grid.x * threads / 32;
      fl = 2.0 * 256.0 * 64.0 * it2 * nwarps;
      printf("{\"kernel\":\"dmma\",\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.3f,\"tflops\":%.3f}\n",
             blocks_per_sm, threads, best, fl / best / 1e9);
      // mixed
      k_mixed<<<grid, block>>>(out, 10, 1.0, 1e-9); CK(cudaDeviceSynchronize());
      best = 1e30f;
      for (int r = 0; r < reps; ++r) {
        CK(cudaEventRecord(e0)); k_mixed<<<grid, block>>>(out, it2, 1.0, 1e-9);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
      }
      double fl_mma = 2.0 * 256.0 * 64.0 * it2 * nwarps;
      double fl_fma = 2.0 * 32.0 * 32.0 * it2 * nwarps;
      printf("{\"kernel\":\"mixed\",\"blocks_per_sm\":%d,\"threads\":%d,\"ms\":%.3f,\"tflops_mma\":%.3f,\"tflops_total\":%.3f}\n",
             blocks_per_sm, threads, best, fl_mma / best / 1e9, (fl_mma + fl_fma) / best / 1e9);
    }
  }
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  printf("{\"sms\":%d,\"clock_khz_attr\":%d}\n", nsm, clk);
  return 0;
}
