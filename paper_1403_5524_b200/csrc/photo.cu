// photo.cu - NEXT-1 of SURVEY.md §8(f): the photoionisation variant of the sweep (PAPER.md:116-122,
// 148-156, the bound-free dipole outer region of Tables 1-2; readings P1-P4).
//
// Step (9), the outer-region dipole amplitude contraction, for a batch of energies:
//     g_i(E_e) = sum_k w_ik d_k / (E_k - E_e)
// i.e. G[ne][nch] = (W . C)^T with the Cauchy-like operand C_ke = d_k / (E_k - E_e) generated on chip
// (never stored). FP64 FMA register tiling: one CTA per 128 channels x 64 energies, 256 threads with
// 8 x 4 outputs each (6 16-byte shared loads per 32 FMA), W k-slabs (128 x 32) staged transposed
// through shared memory from coalesced row loads;
// ascending k per output (deterministic). Pole guard as in R formation: |E - E_k| < 1e-10 gives
// status RMX_E_POLE and NaN amplitudes. 2 nch nlev flops per energy - 1/(nch+1) of R formation, so
// the kernel is a small fraction of the sweep; its bound is FP64 FMA issue. As in R formation
// (reading N1), the term of the pole nearest to E_e is left out of the contraction and added last
// (dipole_g_pole_kernel, after the split-K partial planes are summed).
//
// Steps (10)-(12) (v = (1/2) U'^T g, M = (I - iK_oo)^{-1} v, sigma) run inside the T epilogue
// (tepi.cu), which already holds (I - iK_oo)^{-1}.
#include "rmx_common.cuh"
#include "rmx_internal.h"
#include <algorithm>

namespace rmx {

constexpr int DG_BI = 128, DG_BE = 64, DG_BK = 32, DG_NT = 256;
constexpr int DG_RI = 8, DG_RE = 4;  // outputs per thread: 8 channels x 4 energies
constexpr int DG_LDW = DG_BI + 2;    // padded pitch of the transposed W slab (16-byte aligned rows)

__global__ void __launch_bounds__(DG_NT, 2) dipole_g_kernel(const double *__restrict__ w, int64_t ldw,
                                                         const double *__restrict__ Ek,
                                                         const double *__restrict__ d,
                                                         const double *__restrict__ E, int nch,
                                                         int nlev, int64_t ne, int kchunk,
                                                         double *__restrict__ g,
                                                         int32_t *__restrict__ status) {
  extern __shared__ __align__(16) double dg_smem[];
  double(*Wt)[DG_LDW] = reinterpret_cast<double(*)[DG_LDW]>(dg_smem);                  // [k][channel]
  double(*Cs)[DG_BE] = reinterpret_cast<double(*)[DG_BE]>(dg_smem + DG_BK * DG_LDW);  // d_k/(E_k - E_e)
  __shared__ int pole[DG_BE], kst[DG_BE];
  const int i0 = blockIdx.x * DG_BI;
  const int64_t e0 = static_cast<int64_t>(blockIdx.y) * DG_BE;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;  // energies tx*4.., channels ty*8..
  if (threadIdx.x < DG_BE) {
    pole[threadIdx.x] = 0;
    kst[threadIdx.x] = (e0 + threadIdx.x < ne) ? nearest_pole(Ek, nlev, E[e0 + threadIdx.x]) : -1;
  }
  double acc[DG_RI][DG_RE];
#pragma unroll
  for (int r = 0; r < DG_RI; ++r)
#pragma unroll
    for (int c = 0; c < DG_RE; ++c) acc[r][c] = 0.0;
  // split K: CTA z of gridDim.z sums k in [z kchunk, (z+1) kchunk) into its own partial plane
  const int kbeg = blockIdx.z * kchunk, kend = min(nlev, kbeg + kchunk);
  g += static_cast<int64_t>(blockIdx.z) * ne * nch;
  for (int k0 = kbeg; k0 < kend; k0 += DG_BK) {
    __syncthreads();
    // W slab: 128 channels x 32 k, coalesced 256-byte row segments, stored transposed
    for (int q = threadIdx.x; q < DG_BI * DG_BK; q += DG_NT) {
      const int r = q / DG_BK, kk = q % DG_BK;
      const int i = i0 + r, k = k0 + kk;
      Wt[kk][r] = (i < nch && k < kend) ? w[static_cast<int64_t>(i) * ldw + k] : 0.0;
    }
    for (int q = threadIdx.x; q < DG_BK * DG_BE; q += DG_NT) {
      const int kk = q / DG_BE, c = q % DG_BE;
      const int k = k0 + kk;
      const int64_t e = e0 + c;
      double v = 0.0;
      if (k < kend && e < ne) {
        const double diff = Ek[k] - E[e];
        if (fabs(diff) < kPoleGuard) pole[c] = 1;
        v = (k == kst[c]) ? 0.0 : d[k] / diff;  // nearest pole: added last (dipole_g_pole_kernel)
      }
      Cs[kk][c] = v;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < DG_BK; ++kk) {
      double wv[DG_RI], cv[DG_RE];
#pragma unroll
      for (int r = 0; r < DG_RI; r += 2) lds128(wv[r], wv[r + 1], smem_u32(&Wt[kk][ty * DG_RI + r]));
#pragma unroll
      for (int c = 0; c < DG_RE; c += 2) lds128(cv[c], cv[c + 1], smem_u32(&Cs[kk][tx * DG_RE + c]));
#pragma unroll
      for (int r = 0; r < DG_RI; ++r)
#pragma unroll
        for (int c = 0; c < DG_RE; ++c) acc[r][c] = fma(wv[r], cv[c], acc[r][c]);
    }
  }
  __syncthreads();
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
#pragma unroll
  for (int c = 0; c < DG_RE; ++c) {
    const int64_t e = e0 + tx * DG_RE + c;
    if (e >= ne) continue;
    const bool pl = pole[tx * DG_RE + c] != 0;  // (per k range; the reduction ORs via NaN)
    if (pl && blockIdx.x == 0 && ty == 0) set_status(status, e, RMX_E_POLE);
#pragma unroll
    for (int r = 0; r < DG_RI; ++r) {
      const int i = i0 + ty * DG_RI + r;
      if (i < nch) g[e * nch + i] = pl ? nan : acc[r][c];
    }
  }
}

// g += w_ik* d_k* / (E_k* - E_e), k* the pole nearest to E_e (reading N1: the large term last)
__global__ void dipole_g_pole_kernel(const double *__restrict__ w, int64_t ldw, const double *__restrict__ Ek,
                                     const double *__restrict__ d, const double *__restrict__ E, int nch,
                                     int nlev, int64_t ne, double *__restrict__ g) {
  const int64_t e = blockIdx.x;
  if (e >= ne) return;
  __shared__ int ks;
  if (threadIdx.x == 0) ks = nearest_pole(Ek, nlev, E[e]);
  __syncthreads();
  const double c = d[ks] / (Ek[ks] - E[e]);
  for (int i = threadIdx.x; i < nch; i += blockDim.x) g[e * nch + i] += w[static_cast<int64_t>(i) * ldw + ks] * c;
}

// g = sum of the nsplit partial planes, in plane order (deterministic)
__global__ void dipole_g_reduce_kernel(const double *__restrict__ part, int nsplit, int64_t n,
                                       double *__restrict__ g) {
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < nsplit; ++z) s += part[z * n + q];
    g[q] = s;
  }
}

// K splits so that the grid covers >= 2 CTAs per SM (the energies x channels tile count alone is
// small for a 296-energy batch: 16 x 5 = 80 CTAs at darc)
int dipole_g_splits(int64_t nch, int64_t nlev, int64_t ne) {
  const int64_t tiles = ((nch + DG_BI - 1) / DG_BI) * ((ne + DG_BE - 1) / DG_BE);
  int64_t s = (2 * 148 + tiles - 1) / tiles;
  s = std::min<int64_t>(s, std::max<int64_t>(1, nlev / (8 * DG_BK)));
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(s, 16)));
}

cudaError_t launch_dipole_g(const double *w, int64_t ldw, const double *Ek, const double *d,
                            int64_t nch, int64_t nlev, const double *E, int64_t ne, double *g,
                            int32_t *status, double *part, int64_t part_cap, cudaStream_t st) {
  constexpr int smem = sizeof(double) * (DG_BK * DG_LDW + DG_BK * DG_BE);
  cudaError_t ce = ensure_smem_attr(reinterpret_cast<const void *>(dipole_g_kernel), smem);
  if (ce != cudaSuccess) return ce;
  const int64_t max_e = static_cast<int64_t>(65535) * DG_BE;  // grid.y limit
  for (int64_t e0 = 0; e0 < ne; e0 += max_e) {
    const int64_t n = ne - e0 < max_e ? ne - e0 : max_e;
    int ns = part ? dipole_g_splits(nch, nlev, n) : 1;
    while (ns > 1 && ns * n * nch > part_cap) --ns;  // never beyond the caller's scratch
    const int kchunk = static_cast<int>(((nlev + ns - 1) / ns + DG_BK - 1) / DG_BK * DG_BK);
    dim3 grid(static_cast<unsigned>((nch + DG_BI - 1) / DG_BI), static_cast<unsigned>((n + DG_BE - 1) / DG_BE),
              static_cast<unsigned>(ns));
    dipole_g_kernel<<<grid, DG_NT, smem, st>>>(w, ldw, Ek, d, E + e0, static_cast<int>(nch),
                                            static_cast<int>(nlev), n, kchunk,
                                            ns > 1 ? part : g + e0 * nch,
                                            status ? status + e0 : nullptr);
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) return ce;
    if (ns > 1) {
      dipole_g_reduce_kernel<<<592, 256, 0, st>>>(part, ns, n * nch, g + e0 * nch);
      ce = cudaGetLastError();
      if (ce != cudaSuccess) return ce;
    }
    dipole_g_pole_kernel<<<static_cast<unsigned>(n), 256, 0, st>>>(w, ldw, Ek, d, E + e0, static_cast<int>(nch),
                                                                 static_cast<int>(nlev), n, g + e0 * nch);
    ce = cudaGetLastError();
    if (ce != cudaSuccess) return ce;
  }
  return cudaSuccess;
}

}  // namespace rmx
