// match.cu - S3+S4 of the sweep: K = -(G - aRG')^{-1}(F - aRF')   (BASELINE.json:5).
// The paper is silent on this step (PAPER.md:459-514 stops at R); DESIGN.md §5.2 gives the design:
// one CTA per energy (persistent over energies, workspace slot = blockIdx.x), blocked right-looking
// LU with partial pivoting of A on the augmented matrix [A | B_open] (panel width 32, FP64 DMMA
// trailing updates), then blocked back substitution; only the n_open open columns of B are solved,
// closed columns of K are -e_j (precondition of rmx.h; SURVEY §8(c) reading 9).
#include "cta_la.cuh"
#include "rmx_internal.h"

namespace rmx {

using namespace la;

struct MatchSmem {
  double gemm[GEMM_SMEM_DOUBLES];
  double tri[TRI_SMEM_DOUBLES];
  double redv[NW];
  int redi[NW];
  int ipiv[PB];
};

// Workspace slot M [n][ldm] = [A | pad | B_open]; after elimination + back substitution the
// columns [npad, npad + o) hold Y = A^{-1} B_open and K[e] = -Y (open), -e_j (closed).
// K may alias R (the sweep reuses the R batch buffer): R[e] is fully consumed before K[e] is written.
__global__ void __launch_bounds__(NT, 1)
    match_kernel(const double *R, int64_t ldr, const double *__restrict__ F,
                 const double *__restrict__ G, const double *__restrict__ Fp,
                 const double *__restrict__ Gp, double a, int n, int64_t ne,
                 const int32_t *__restrict__ n_open, double *K, int64_t ldk, double *ws,
                 int64_t ws_slot, int ldm, int32_t *status) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  MatchSmem &sm = *reinterpret_cast<MatchSmem *>(smem_raw);
  double *Mw = ws + static_cast<int64_t>(blockIdx.x) * ws_slot;
  const int npad = (n + 1) & ~1;

  for (int64_t e = blockIdx.x; e < ne; e += gridDim.x) {
    int o = n_open ? n_open[e] : n;
    o = o < 0 ? 0 : (o > n ? n : o);
    const int ncols = npad + o;
    const double *Re = R + e * static_cast<int64_t>(n) * ldr;
    const double *Fe = F + e * n, *Ge = G + e * n, *Fpe = Fp + e * n, *Gpe = Gp + e * n;

    // ---- S3: A_ij = G_i d_ij - a R_ij G'_j ; B_ij = F_i d_ij - a R_ij F'_j ----
    for (int i = warp_id(); i < n; i += NW) {
      const double *Ri = Re + static_cast<int64_t>(i) * ldr;
      double *Mi = Mw + static_cast<int64_t>(i) * ldm;
      for (int j = lane_id(); j < ncols; j += 32) {
        double v = 0.0;
        if (j < n) {
          v = -(a * Ri[j]) * Gpe[j];
          if (j == i) v += Ge[i];
        } else if (j >= npad) {
          const int jb = j - npad;
          v = -(a * Ri[jb]) * Fpe[jb];
          if (jb == i) v += Fe[i];
        }
        Mi[j] = v;
      }
    }
    __syncthreads();

    // ---- S4a: blocked right-looking LU with partial pivoting on [A | B_open] ----
    int singular = 0;
    for (int p0 = 0; p0 < n; p0 += PB) {
      const int bw = min(PB, n - p0);
      singular |= panel_lu(Mw, ldm, n, p0, bw, sm.ipiv, sm.redv, sm.redi);
      swap_and_trsm_unit_lower(Mw, ldm, p0, bw, sm.ipiv, p0 + bw, ncols, sm.tri);
      const int m2 = n - p0 - bw, n2 = ncols - p0 - bw;
      if (m2 > 0 && n2 > 0) {
        double *C = Mw + static_cast<int64_t>(p0 + bw) * ldm + p0 + bw;
        const double *L21 = Mw + static_cast<int64_t>(p0 + bw) * ldm + p0;
        const double *U12 = Mw + static_cast<int64_t>(p0) * ldm + p0 + bw;
        gemm<true, false>(m2, n2, bw, L21, ldm, U12, ldm, false, sm.gemm, EpiSub{C, ldm});
      }
    }

    // ---- S4b: blocked back substitution U Y = L^{-1} P B_open (Y in columns [npad, npad+o)) ----
    if (o > 0) {
      double *Y = Mw + npad;
      for (int p0 = ((n - 1) / PB) * PB; p0 >= 0; p0 -= PB) {
        const int bw = min(PB, n - p0);
        trsm_upper_cols(Mw, ldm, p0, bw, Y, ldm, o, sm.tri);
        if (p0 > 0) {
          const double *U = Mw + p0;  // rows [0, p0), cols [p0, p0+bw): A[i][k] = U[i*ldm + k]
          const double *Yp = Y + static_cast<int64_t>(p0) * ldm;
          gemm<true, false>(p0, o, bw, U, ldm, Yp, ldm, false, sm.gemm, EpiSub{Y, ldm});
        }
      }
    }

    // ---- output: K = -Y (open columns), -e_j (closed columns); status ----
    int bad = 0;
    double *Ke = K + e * static_cast<int64_t>(n) * ldk;
    for (int i = warp_id(); i < n; i += NW) {
      const double *Yi = Mw + static_cast<int64_t>(i) * ldm + npad;
      double *Ki = Ke + static_cast<int64_t>(i) * ldk;
      for (int j = lane_id(); j < n; j += 32) {
        double v;
        if (j < o) {
          v = -Yi[j];
          if (i < o && !isfinite(v)) bad = 1;
        } else {
          v = (i == j) ? -1.0 : 0.0;
        }
        Ki[j] = v;
      }
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
      if (singular)
        set_status(status, e, RMX_E_SINGULAR);
      else if (bad)
        set_status(status, e, RMX_E_NONFINITE);
    }
  }
}

size_t match_smem_bytes() { return sizeof(MatchSmem); }

int64_t match_ws_doubles_per_slot(int64_t nch) {
  const int64_t npad = (nch + 1) & ~1LL;
  return nch * (2 * npad);
}

cudaError_t launch_match(const double *R, const double *F, const double *G, const double *Fp,
                         const double *Gp, double a, int64_t nch, int64_t ne, const int32_t *n_open,
                         double *K, double *ws, int64_t ws_slots, int32_t *status, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t ce = cudaFuncSetAttribute(match_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(sizeof(MatchSmem)));
    if (ce != cudaSuccess) return ce;
    attr = true;
  }
  const int64_t npad = (nch + 1) & ~1LL;
  const int ldm = static_cast<int>(2 * npad);
  const int grid = static_cast<int>(ne < ws_slots ? ne : ws_slots);
  match_kernel<<<grid, NT, sizeof(MatchSmem), st>>>(R, nch, F, G, Fp, Gp, a, static_cast<int>(nch),
                                                    ne, n_open, K, nch, ws,
                                                    match_ws_doubles_per_slot(nch), ldm, status);
  return cudaGetLastError();
}

}  // namespace rmx
