// post.cu - NEXT-4 of SURVEY.md §8(f): post-processing of the sweep's spectra on the energy mesh.
//
//  (a) Gaussian convolution at a given FWHM with statistical admixture (Fig. 1
//      caption "convoluted with a 60 meV FWHM Gaussian"; Fig. 3 caption "the
//      appropriate Gaussian of FWHM and a statistical admixture of 2/3 ground and 1/3 metastable
//      states"; operational definition, reading C1):
//          x      = sum_m c_m x_m / sum_m c_m                       (admixture, optional)
//          y_i    = sum_{|j-i| <= M} g_{j-i} x_j / sum_{|j-i| <= M, 0 <= j < ne} g_{j-i}
//          g_d    = exp(-(d dE)^2 / (2 s^2)),  s = FWHM / (2 sqrt(2 ln 2)),  M = floor(5 s / dE)
//      on a uniform mesh of spacing dE (the kernel truncated at +-5s, renormalised at the edges).
//      One CTA per tile of 256 outputs stages x[i0 - M, i0 + 256 + M) in shared memory; one
//      thread per output runs the FP64 FMA loop over the window (bound: FP64 ALU, 2M+1 FMA per
//      output; the window weights g_d are a per-call table in shared memory).
//
//  (b) Maxwellian average (effective collision strength, reading U1):
//          Ups_p(T) = int_0^inf Omega_p(eps) exp(-eps/kT) d(eps/kT),  eps = E - E_th,p
//      by the trapezoid rule over the mesh points E_f..E_{ne-1} with E_i > E_th,p (no
//      extrapolation): with f_i = Omega_p(E_i) exp(-(E_i - E_th,p)/kT) / kT,
//          Ups_p(T) = sum_{i=f}^{ne-2} (E_{i+1} - E_i) (f_i + f_{i+1}) / 2
//      evaluated as sum_i tw_i f_i, tw_i = [(E_{i+1} - E_i)[i < ne-1] + (E_i - E_{i-1})[i > f]] / 2.
//      Omega [ne][npair] row-major
//      is read once (coalesced over pairs); the energy range is split into chunks whose partial
//      sums are added in chunk order by a second pass (deterministic, no atomics).
#include "rmx_common.cuh"
#include "rmx_internal.h"
#include <cmath>

namespace rmx {

constexpr int CONV_TILE = 256;

__global__ void conv_weights_kernel(double *g, int M, double dE, double s) {
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d <= M; d += gridDim.x * blockDim.x) {
    const double x = d * dE;
    g[d] = exp(-(x * x) / (2.0 * s * s));
  }
}

// x: [nspec][ne]; mix: nullptr (convolve each spectrum) or DEVICE [nspec] weights (one output)
__global__ void __launch_bounds__(CONV_TILE) conv_gauss_kernel(const double *__restrict__ x,
                                                               int nspec, const double *__restrict__ mix,
                                                               int64_t ne, int M,
                                                               const double *__restrict__ gtab,
                                                               double *__restrict__ y) {
  extern __shared__ double sm[];
  double *xs = sm;                        // [CONV_TILE + 2M]
  double *gs = sm + CONV_TILE + 2 * M;    // [M + 1]
  __shared__ double gfull;                // g_0 + 2 sum_d g_d: the interior normalisation
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * CONV_TILE;
  const int spec = blockIdx.y;  // output spectrum (0 when mixing)
  for (int d = threadIdx.x; d <= M; d += blockDim.x) gs[d] = gtab[d];
  double msum = 0.0;
  if (mix)
    for (int m = 0; m < nspec; ++m) msum += mix[m];
  const int span = CONV_TILE + 2 * M;
  for (int q = threadIdx.x; q < span; q += blockDim.x) {
    const int64_t j = i0 - M + q;
    double v = 0.0;
    if (j >= 0 && j < ne) {
      if (mix) {
        for (int m = 0; m < nspec; ++m) v += mix[m] * x[static_cast<int64_t>(m) * ne + j];
        v /= msum;
      } else {
        v = x[static_cast<int64_t>(spec) * ne + j];
      }
    }
    xs[q] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int d = M; d >= 1; --d) t += gs[d];
    gfull = gs[0] + 2.0 * t;
  }
  __syncthreads();
  const int64_t i = i0 + threadIdx.x;
  if (i >= ne) return;
  const double *xc = xs + threadIdx.x + M;  // x_i
  double num = gs[0] * xc[0], den = gs[0];
  const bool interior = (i - M >= 0) && (i + M < ne);
  if (interior) {  // symmetric window: one add + one FMA per pair (j = i -+ d)
    for (int d = 1; d <= M; ++d) num = fma(gs[d], xc[-d] + xc[d], num);
    den = gfull;
  } else {
    for (int d = 1; d <= M; ++d) {
      const double gd = gs[d];
      if (i - d >= 0) {
        num = fma(gd, xc[-d], num);
        den += gd;
      }
      if (i + d < ne) {
        num = fma(gd, xc[d], num);
        den += gd;
      }
    }
  }
  y[static_cast<int64_t>(spec) * ne + i] = num / den;
}

constexpr int MAXW_CHUNK = 1024;   // energies per partial sum
constexpr int MAXW_PAIRS = 128;    // pairs per CTA (one per thread)

struct MaxwT {
  double kT[RMX_MAX_TEMPS];
  int nT;
};

// part: [nchunk][npair][nT] partial trapezoid sums (without the dE/kT factor)
__global__ void __launch_bounds__(MAXW_PAIRS) maxwell_partial_kernel(
    const double *__restrict__ omega, int64_t ne, int64_t npair, const double *__restrict__ E,
    const double *__restrict__ Eth, const MaxwT T, double *__restrict__ part) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * MAXW_PAIRS + threadIdx.x;
  const int64_t c = blockIdx.y;
  if (p >= npair) return;
  const double eth = Eth[p];
  // first included mesh point: smallest i with E_i > eth (E ascending)
  int64_t lo = 0, hi = ne;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (E[mid] > eth) hi = mid; else lo = mid + 1;
  }
  const int64_t first = lo;
  double acc[RMX_MAX_TEMPS];
#pragma unroll
  for (int t = 0; t < RMX_MAX_TEMPS; ++t) acc[t] = 0.0;
  const int64_t ia = max(c * MAXW_CHUNK, first), ib = min((c + 1) * MAXW_CHUNK, ne);
  for (int64_t i = ia; i < ib; ++i) {
    const double Ei = E[i];
    const double tw = 0.5 * ((i < ne - 1 ? E[i + 1] - Ei : 0.0) + (i > first ? Ei - E[i - 1] : 0.0));
    const double om = tw * omega[i * npair + p];
    const double eps = Ei - eth;
#pragma unroll
    for (int t = 0; t < RMX_MAX_TEMPS; ++t)
      if (t < T.nT) acc[t] = fma(om, exp(-eps / T.kT[t]) / T.kT[t], acc[t]);
  }
  for (int t = 0; t < T.nT; ++t) part[(c * npair + p) * T.nT + t] = acc[t];
}

__global__ void maxwell_reduce_kernel(const double *__restrict__ part, int64_t nchunk, int64_t npair,
                                      int nT, double *__restrict__ ups) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (q >= npair * nT) return;
  double s = 0.0;
  for (int64_t c = 0; c < nchunk; ++c) s += part[c * npair * nT + q];
  ups[q] = s;
}

int conv_window(double dE, double fwhm, double *sigma) {
  const double s = fwhm / (2.0 * std::sqrt(2.0 * std::log(2.0)));
  if (sigma) *sigma = s;
  return static_cast<int>(std::floor(5.0 * s / dE));
}

cudaError_t launch_convolve(const double *x, int64_t nspec, const double *mix_dev, int64_t ne,
                            double dE, double fwhm, double *gtab, double *y, cudaStream_t st) {
  double s = 0.0;
  const int M = conv_window(dE, fwhm, &s);
  conv_weights_kernel<<<(M + 256) / 256, 256, 0, st>>>(gtab, M, dE, s);
  const size_t smem = sizeof(double) * (CONV_TILE + 2 * static_cast<size_t>(M) + M + 1);
  if (smem > 48 * 1024) {
    cudaError_t ce = cudaFuncSetAttribute(conv_gauss_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem));
    if (ce != cudaSuccess) return ce;
  }
  dim3 grid(static_cast<unsigned>((ne + CONV_TILE - 1) / CONV_TILE),
            static_cast<unsigned>(mix_dev ? 1 : nspec));
  conv_gauss_kernel<<<grid, CONV_TILE, smem, st>>>(x, static_cast<int>(nspec), mix_dev, ne, M, gtab, y);
  return cudaGetLastError();
}

int64_t maxwell_chunks(int64_t ne) { return (ne + MAXW_CHUNK - 1) / MAXW_CHUNK; }

cudaError_t launch_maxwell(const double *omega, int64_t ne, int64_t npair, const double *E,
                           const double *Eth, const double *kT, int nT, double *part, double *ups,
                           cudaStream_t st) {
  MaxwT T;
  for (int t = 0; t < RMX_MAX_TEMPS; ++t) T.kT[t] = t < nT ? kT[t] : 1.0;
  T.nT = nT;
  const int64_t nchunk = maxwell_chunks(ne);
  dim3 grid(static_cast<unsigned>((npair + MAXW_PAIRS - 1) / MAXW_PAIRS), static_cast<unsigned>(nchunk));
  maxwell_partial_kernel<<<grid, MAXW_PAIRS, 0, st>>>(omega, ne, npair, E, Eth, T, part);
  const int64_t nq = npair * nT;
  maxwell_reduce_kernel<<<static_cast<unsigned>((nq + 255) / 256), 256, 0, st>>>(part, nchunk, npair,
                                                                                nT, ups);
  return cudaGetLastError();
}

}  // namespace rmx
