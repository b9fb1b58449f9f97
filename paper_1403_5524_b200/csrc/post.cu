// post.cu - NEXT-4 of SURVEY.md §8(f): post-processing of the sweep's spectra on the energy mesh.
//
//  (a) Gaussian convolution at a given FWHM with statistical admixture (Fig. 1
//      caption "convoluted with a 60 meV FWHM Gaussian"; Fig. 3 caption "the
//      appropriate Gaussian of FWHM and a statistical admixture of 2/3 ground and 1/3 metastable
//      states"; operational definition, reading C1):
//          x      = sum_m (c_m / sum_m' c_m') x_m                   (admixture, optional)
//          y_i    = sum_{|j-i| <= M} g_{j-i} x_j / sum_{|j-i| <= M, 0 <= j < ne} g_{j-i}
//          g_d    = exp(-(d dE)^2 / (2 s^2)),  s = FWHM / (2 sqrt(2 ln 2)),  M = floor(5 s / dE)
//      on a uniform mesh of spacing dE (the kernel truncated at +-5s, renormalised at the edges).
//      One CTA per tile of 256 x 7 outputs stages x[i0 - M, i0 + tile + M) in shared memory; each
//      thread owns 7 consecutive outputs and slides two register windows over the symmetric pairs
//      (x_{i-d} + x_{i+d}), so one step costs 3 shared loads for 7 adds + 7 FMAs (bound: FP64 pipe;
//      the weights g_d are a per-call table in shared memory, the interior normalisation one sum).
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

constexpr int CONV_NT = 256;             // threads per CTA
constexpr int CONV_R = 7;                // consecutive outputs per thread (odd: conflict-free LDS)
constexpr int CONV_TILE = CONV_NT * CONV_R;

constexpr int CONV_MAX_MIX = 64;  // admixture components passed by value

struct ConvMix {
  double c[CONV_MAX_MIX];  // weights already divided by their sum
  int n;                   // 0: no admixture (each spectrum convolved alone)
};

// x: [nspec][ne]; mix: nullptr (convolve each spectrum) or DEVICE [nspec] weights (one output).
// Each thread owns CONV_R consecutive outputs and slides two register windows (x_{i+r-d}, x_{i+r+d})
// over d, so every step costs 2 shared loads + 1 broadcast weight load for CONV_R (add + FMA) pairs.
__global__ void __launch_bounds__(CONV_NT) conv_gauss_kernel(const double *__restrict__ x,
                                                             const ConvMix mix, int64_t ne, int M,
                                                             double dE, double sg,
                                                             double *__restrict__ y) {
  extern __shared__ double sm[];
  double *xs = sm;                        // [CONV_TILE + 2M]
  double *gs = sm + CONV_TILE + 2 * M;    // [M + 1]
  __shared__ double gfull;                // g_0 + 2 sum_d g_d: the interior normalisation
  const int64_t blk0 = static_cast<int64_t>(blockIdx.x) * CONV_TILE;
  const int spec = blockIdx.y;  // output spectrum (0 when mixing)
  for (int d = threadIdx.x; d <= M; d += blockDim.x) {
    const double u = d * dE;
    gs[d] = exp(-(u * u) / (2.0 * sg * sg));
  }
  const int span = CONV_TILE + 2 * M;
  for (int q = threadIdx.x; q < span; q += blockDim.x) {
    const int64_t j = blk0 - M + q;
    double v = 0.0;
    if (j >= 0 && j < ne) {
      if (mix.n) {
        for (int m = 0; m < mix.n; ++m) v = fma(mix.c[m], x[static_cast<int64_t>(m) * ne + j], v);
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
  const int64_t i0 = blk0 + static_cast<int64_t>(threadIdx.x) * CONV_R;
  if (i0 >= ne) return;
  const double *xc = xs + threadIdx.x * CONV_R + M;  // x_{i0}
  double *ye = y + static_cast<int64_t>(spec) * ne;
  const bool interior = (i0 - M >= 0) && (i0 + CONV_R - 1 + M < ne);
  if (interior) {
    double num[CONV_R], L[CONV_R], Rt[CONV_R];
#pragma unroll
    for (int r = 0; r < CONV_R; ++r) {
      num[r] = gs[0] * xc[r];
      L[r] = xc[r];   // x_{i0 + r - d} at d = 0
      Rt[r] = xc[r];  // x_{i0 + r + d} at d = 0
    }
    for (int d = 1; d <= M; ++d) {
#pragma unroll
      for (int r = CONV_R - 1; r > 0; --r) L[r] = L[r - 1];
      L[0] = xc[-d];
#pragma unroll
      for (int r = 0; r < CONV_R - 1; ++r) Rt[r] = Rt[r + 1];
      Rt[CONV_R - 1] = xc[CONV_R - 1 + d];
      const double gd = gs[d];
#pragma unroll
      for (int r = 0; r < CONV_R; ++r) num[r] = fma(gd, L[r] + Rt[r], num[r]);
    }
#pragma unroll
    for (int r = 0; r < CONV_R; ++r) ye[i0 + r] = num[r] / gfull;
    return;
  }
  for (int r = 0; r < CONV_R; ++r) {  // mesh edges: partial window, renormalised
    const int64_t i = i0 + r;
    if (i >= ne) break;
    double num = gs[0] * xc[r], den = gs[0];
    for (int d = 1; d <= M; ++d) {
      const double gd = gs[d];
      if (i - d >= 0) {
        num = fma(gd, xc[r - d], num);
        den += gd;
      }
      if (i + d < ne) {
        num = fma(gd, xc[r + d], num);
        den += gd;
      }
    }
    ye[i] = num / den;
  }
}

constexpr int MAXW_CHUNK = 128;    // energies per partial sum
constexpr int MAXW_PAIRS = 128;    // pairs per CTA (one per thread)

struct MaxwT {
  double kT[RMX_MAX_TEMPS];
  int nT;
};

// part: [nchunk][npair][nT] partial trapezoid sums. Within a chunk starting at mesh point c0 the
// Boltzmann factor splits as e^{-(E_i - Eth)/kT} = e^{-(E_i - E_c0)/kT} e^{-(E_c0 - Eth)/kT}: the first
// factor is shared by all pairs (one exp per (i, T) per CTA, staged in shared memory), the second is
// one exp per (pair, T, chunk). Where the second factor could overflow (threshold more than 600 kT
// above the chunk start) the pair falls back to one exp per term.
// NTT: temperatures of the compiled bucket (nT <= NTT, rows t >= nT of the table are zero, so the
// unrolled accumulation carries no per-temperature predicate; buckets 8 / 16 / 32 keep the
// accumulators in registers - one kernel for RMX_MAX_TEMPS = 32 spent half its FMAs on padding rows
// and its instruction fetch on predicated code). Points at or below threshold get the weight 0
// instead of a branch (E ascending: they form a prefix of the chunk).
template <int NTT>
__global__ void __launch_bounds__(MAXW_PAIRS, NTT <= 16 ? 4 : 2) maxwell_partial_kernel(
    const double *__restrict__ omega, int64_t ne, int64_t npair, const double *__restrict__ E,
    const double *__restrict__ Eth, const MaxwT T, double *__restrict__ part) {
  __shared__ __align__(16) double sE[MAXW_CHUNK][NTT];  // [point][T]: a point's factors read as double2
  __shared__ double sx[MAXW_CHUNK + 2];  // E_{c0-1} .. E_{c1}
  const int64_t p = static_cast<int64_t>(blockIdx.x) * MAXW_PAIRS + threadIdx.x;
  const int64_t c = blockIdx.y;
  const int64_t c0 = c * MAXW_CHUNK, c1 = min(c0 + MAXW_CHUNK, ne);
  const int n = static_cast<int>(c1 - c0);
  for (int q = threadIdx.x; q < n + 2; q += MAXW_PAIRS) {
    const int64_t i = c0 - 1 + q;
    sx[q] = (i >= 0 && i < ne) ? E[i] : 0.0;
  }
  __syncthreads();
  const double Ec0 = sx[1];
  for (int q = threadIdx.x; q < NTT * MAXW_CHUNK; q += MAXW_PAIRS) {
    const int ii = q / NTT, t = q % NTT;
    sE[ii][t] = (ii < n && t < T.nT) ? exp(-(sx[ii + 1] - Ec0) / T.kT[t]) : 0.0;
  }
  __syncthreads();
  if (p >= npair) return;
  const double eth = Eth[p];
  double acc[NTT];
#pragma unroll
  for (int t = 0; t < NTT; ++t) acc[t] = 0.0;
  bool direct = false;
  for (int t = 0; t < T.nT; ++t) direct |= (eth - Ec0) / T.kT[t] > 600.0;
  auto weight = [&](int ii) {  // trapezoid weight of point c0 + ii (0 if not above threshold)
    const int64_t i = c0 + ii;
    const double Ei = sx[ii + 1];
    if (ii >= n || !(Ei > eth)) return 0.0;
    // half the interval to the right (if any) plus half the interval to the left when the left
    // neighbour is also above threshold
    const double right = (i + 1 < ne) ? 0.5 * (sx[ii + 2] - Ei) : 0.0;
    const double left = (i > 0 && sx[ii] > eth) ? 0.5 * (Ei - sx[ii]) : 0.0;
    return right + left;
  };
  if (!direct) {
    // Omega loads issued in groups of PF (independent of the accumulation; latency-bound otherwise)
    constexpr int PF = NTT <= 8 ? 8 : 4;
    for (int g0 = 0; g0 < n; g0 += PF) {
      double ob[PF];
#pragma unroll
      for (int q = 0; q < PF; ++q) ob[q] = (g0 + q < n) ? omega[(c0 + g0 + q) * npair + p] : 0.0;
#pragma unroll
      for (int q = 0; q < PF; ++q) {
        const double wq = weight(g0 + q);
        const double om = wq != 0.0 ? wq * ob[q] : 0.0;  // Omega below threshold never read into the sum
        const double2 *ep = reinterpret_cast<const double2 *>(sE[g0 + q]);
#pragma unroll
        for (int t2 = 0; t2 < NTT / 2; ++t2) {
          const double2 f = ep[t2];
          acc[2 * t2] = fma(om, f.x, acc[2 * t2]);
          acc[2 * t2 + 1] = fma(om, f.y, acc[2 * t2 + 1]);
        }
      }
    }
  } else {  // threshold > 600 kT above the chunk start for some T: one exp per term (rare)
#pragma unroll 1
    for (int ii = 0; ii < n; ++ii) {
      const double om = weight(ii);
      if (om == 0.0) continue;
      const double ov = om * omega[(c0 + ii) * npair + p], Ei = sx[ii + 1];
#pragma unroll
      for (int t = 0; t < NTT; ++t)
        if (t < T.nT) acc[t] = fma(ov, exp(-(Ei - eth) / T.kT[t]), acc[t]);
    }
  }
#pragma unroll
  for (int t = 0; t < NTT; ++t) {
    if (t >= T.nT) break;
    const double f = direct ? 1.0 : exp(-(Ec0 - eth) / T.kT[t]);
    part[(c * npair + p) * T.nT + t] = acc[t] * f / T.kT[t];
  }
}
__global__ void maxwell_reduce_kernel(const double *__restrict__ part, int64_t nchunk, int64_t npair,
                                      int nT, double *__restrict__ ups) {
  const int64_t q = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (q >= npair * nT) return;
  double s = 0.0;
  for (int64_t c = lane; c < nchunk; c += 32) s += part[c * npair * nT + q];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) ups[q] = s;
}

int conv_window(double dE, double fwhm, double *sigma) {
  const double s = fwhm / (2.0 * std::sqrt(2.0 * std::log(2.0)));
  if (sigma) *sigma = s;
  return static_cast<int>(std::floor(5.0 * s / dE));
}

cudaError_t launch_convolve(const double *x, int64_t nspec, const double *mix, int64_t ne,
                            double dE, double fwhm, double *y, cudaStream_t st) {
  double s = 0.0;
  const int M = conv_window(dE, fwhm, &s);
  ConvMix cm;
  cm.n = mix ? static_cast<int>(nspec) : 0;
  double msum = 0.0;
  for (int m = 0; m < cm.n; ++m) msum += mix[m];
  for (int m = 0; m < CONV_MAX_MIX; ++m) cm.c[m] = m < cm.n ? mix[m] / msum : 0.0;
  const size_t smem = sizeof(double) * (CONV_TILE + 2 * static_cast<size_t>(M) + M + 1);
  if (smem > 48 * 1024) {
    cudaError_t ce = cudaFuncSetAttribute(conv_gauss_kernel,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem));
    if (ce != cudaSuccess) return ce;
  }
  dim3 grid(static_cast<unsigned>((ne + CONV_TILE - 1) / CONV_TILE),
            static_cast<unsigned>(mix ? 1 : nspec));
  conv_gauss_kernel<<<grid, CONV_NT, smem, st>>>(x, cm, ne, M, dE, s, y);
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
  if (nT <= 8)
    maxwell_partial_kernel<8><<<grid, MAXW_PAIRS, 0, st>>>(omega, ne, npair, E, Eth, T, part);
  else if (nT <= 16)
    maxwell_partial_kernel<16><<<grid, MAXW_PAIRS, 0, st>>>(omega, ne, npair, E, Eth, T, part);
  else
    maxwell_partial_kernel<32><<<grid, MAXW_PAIRS, 0, st>>>(omega, ne, npair, E, Eth, T, part);
  const int64_t nq = npair * nT;
  maxwell_reduce_kernel<<<static_cast<unsigned>((nq * 32 + 255) / 256), 256, 0, st>>>(part, nchunk, npair,
                                                                                     nT, ups);
  return cudaGetLastError();
}

}  // namespace rmx
