// photo.cu - NEXT-1 of SURVEY.md §8(f): the photoionisation variant of the sweep (PAPER.md:116-122,
// 148-156, the bound-free dipole outer region of Tables 1-2; readings P1-P4).
//
// Step (9), the outer-region dipole amplitude contraction, for a batch of energies:
//     g_i(E_e) = sum_k w_ik d_k / (E_k - E_e)
// i.e. G[ne][nch] = (W . C)^T with the Cauchy-like operand C_ke = d_k / (E_k - E_e) generated on chip
// (never stored). FP64 FMA register tiling: one CTA per 64 channels x 32 energies, 256 threads with
// 4 x 2 outputs each, W k-slabs (64 x 32) staged through shared memory with coalesced row loads;
// ascending k per output (deterministic). Pole guard as in R formation: |E - E_k| < 1e-10 gives
// status RMX_E_POLE and NaN amplitudes. 2 nch nlev flops per energy - 1/(nch+1) of R formation, so
// the kernel is a small fraction of the sweep; its bound is FP64 FMA issue.
//
// Steps (10)-(12) (v = (1/2) U'^T g, M = (I - iK_oo)^{-1} v via the SPD route, sigma) run inside the
// T epilogue (tepi.cu), which already holds the Cholesky factor of I + K_oo^2.
#include "rmx_common.cuh"
#include "rmx_internal.h"

namespace rmx {

constexpr int DG_BI = 64, DG_BE = 32, DG_BK = 32, DG_NT = 256;

__global__ void __launch_bounds__(DG_NT) dipole_g_kernel(const double *__restrict__ w, int64_t ldw,
                                                         const double *__restrict__ Ek,
                                                         const double *__restrict__ d,
                                                         const double *__restrict__ E, int nch,
                                                         int nlev, int64_t ne,
                                                         double *__restrict__ g,
                                                         int32_t *__restrict__ status) {
  __shared__ double Ws[DG_BI][DG_BK + 1];
  __shared__ double Cs[DG_BK][DG_BE];
  __shared__ int pole[DG_BE];
  const int i0 = blockIdx.x * DG_BI;
  const int64_t e0 = static_cast<int64_t>(blockIdx.y) * DG_BE;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // energies tx*2.., rows ty*4..
  if (threadIdx.x < DG_BE) pole[threadIdx.x] = 0;
  double acc[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int k0 = 0; k0 < nlev; k0 += DG_BK) {
    __syncthreads();
    // W slab: 64 rows x 32 k (each row a 256-byte coalesced segment)
    for (int q = threadIdx.x; q < DG_BI * DG_BK; q += DG_NT) {
      const int r = q / DG_BK, kk = q % DG_BK;
      const int i = i0 + r, k = k0 + kk;
      Ws[r][kk] = (i < nch && k < nlev) ? w[static_cast<int64_t>(i) * ldw + k] : 0.0;
    }
    // generated operand C_ke = d_k / (E_k - E_e)
    for (int q = threadIdx.x; q < DG_BK * DG_BE; q += DG_NT) {
      const int kk = q / DG_BE, c = q % DG_BE;
      const int k = k0 + kk;
      const int64_t e = e0 + c;
      double v = 0.0;
      if (k < nlev && e < ne) {
        const double diff = Ek[k] - E[e];
        if (fabs(diff) < kPoleGuard) pole[c] = 1;
        v = d[k] / diff;
      }
      Cs[kk][c] = v;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < DG_BK; ++kk) {
      const double c0 = Cs[kk][tx * 2], c1 = Cs[kk][tx * 2 + 1];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double wv = Ws[ty * 4 + r][kk];
        acc[r][0] = fma(wv, c0, acc[r][0]);
        acc[r][1] = fma(wv, c1, acc[r][1]);
      }
    }
  }
  __syncthreads();
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const int64_t e = e0 + tx * 2 + c;
    if (e >= ne) continue;
    const bool pl = pole[tx * 2 + c] != 0;
    if (pl && blockIdx.x == 0 && ty == 0) set_status(status, e, RMX_E_POLE);
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int i = i0 + ty * 4 + r;
      if (i < nch) g[e * nch + i] = pl ? nan : acc[r][c];
    }
  }
}

cudaError_t launch_dipole_g(const double *w, int64_t ldw, const double *Ek, const double *d,
                            int64_t nch, int64_t nlev, const double *E, int64_t ne, double *g,
                            int32_t *status, cudaStream_t st) {
  const int64_t max_e = static_cast<int64_t>(65535) * DG_BE;  // grid.y limit
  for (int64_t e0 = 0; e0 < ne; e0 += max_e) {
    const int64_t n = ne - e0 < max_e ? ne - e0 : max_e;
    dim3 grid(static_cast<unsigned>((nch + DG_BI - 1) / DG_BI), static_cast<unsigned>((n + DG_BE - 1) / DG_BE));
    dipole_g_kernel<<<grid, DG_NT, 0, st>>>(w, ldw, Ek, d, E + e0, static_cast<int>(nch),
                                            static_cast<int>(nlev), n, g + e0 * nch,
                                            status ? status + e0 : nullptr);
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) return ce;
  }
  return cudaSuccess;
}

}  // namespace rmx
