// rmx_common.cuh - sm_100a device helpers shared by the librmx kernels (not by the oracle).
// FP64 tensor-core MMA (DMMA), cp.async, mbarrier and TMA (cp.async.bulk.tensor) wrappers.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda.h>

#ifndef __CUDA_ARCH__
#define RMX_HOST_ONLY 1
#endif

namespace rmx {

constexpr double kPoleGuard = 1e-10;  // |E - E_k| < 1e-10 Ry -> RMX_E_POLE

// Device-side bounds checks of the bounds-checked build (python -m paper_1403_5524_b200.build
// --checked -> librmx_checked.so, -DRMX_CHECKS; tests/test_gpu_checked.py): a failed check prints its
// place and traps, which the host sees as a CUDA error. Compiled out of librmx.so.
#ifdef RMX_CHECKS
#define RMX_CHECK(cond)                                                                          \
  do {                                                                                           \
    if (!(cond)) {                                                                               \
      printf("RMX_CHECK(%s) failed at %s:%d block %d thread %d\n", #cond, __FILE__, __LINE__,   \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                       \
      __trap();                                                                                  \
    }                                                                                            \
  } while (0)
#else
#define RMX_CHECK(cond) \
  do {                  \
  } while (0)
#endif

// ---- nearest pole ----------------------------------------------------------------------------
// Index k* of the pole nearest to E (E_k ascending, the rmx.h precondition; ties -> lower index).
// Both R formations sum the term of k* apart from the others and add it last (reading N1):
// next to a pole that term is orders of magnitude larger than the rest, and accumulating the rest on
// top of it (or, for the INT8-CRT path, scaling the fixed point to it) would keep only the bits of
// the background that survive next to the pole term.
__device__ __forceinline__ int nearest_pole(const double *__restrict__ Ek, int nlev, double E) {
  int lo = 0, hi = nlev;  // first k with E_k >= E
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (Ek[mid] < E)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo >= nlev) return nlev - 1;
  if (lo == 0) return 0;
  return (E - Ek[lo - 1] <= Ek[lo] - E) ? lo - 1 : lo;
}

// ---- status helpers (first error wins) ---------------------------------------------------
__device__ __forceinline__ void set_status(int32_t *status, int64_t e, int32_t code) {
  if (status != nullptr && code != 0) atomicCAS(reinterpret_cast<int *>(status + e), 0, code);
}

// ---- FP64 tensor-core MMA: D(8x8) += A(8x4) * B(4x8) ----------------------------------------
// Fragment layout (PTX ISA, mma.m8n8k4 .f64): lane = 4*g + t
//   A: a = A[g][t]        B: b = B[t][g]        C/D: {c0, c1} = C[g][2t], C[g][2t+1]
__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---- shared-memory address helpers -----------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ double lds64(uint32_t addr) {
  double x;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(x) : "r"(addr));
  return x;
}
__device__ __forceinline__ void lds128(double &x, double &y, uint32_t addr) {
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];\n" : "=d"(x), "=d"(y) : "r"(addr));
}

__device__ __forceinline__ void stg128(double *p, double x, double y) {
  asm volatile("st.global.v2.f64 [%0], {%1,%2};\n" ::"l"(p), "d"(x), "d"(y) : "memory");
}

// ---- cp.async (LDGSTS) -------------------------------------------------------------------------
// 16-byte async copy with zero fill of the bytes beyond src_bytes (0, 8 or 16).
__device__ __forceinline__ void cp_async16(uint32_t dst, const void *src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void *src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src),
               "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- mbarrier ----------------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::);
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// ---- TMA: 2D tiled load global -> shared, completion on an mbarrier --------------------------
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, uint64_t *bar,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// 1D bulk async copy global -> shared (16-byte aligned, size % 16 == 0), completion on an mbarrier.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---- warp helpers ------------------------------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

}  // namespace rmx
