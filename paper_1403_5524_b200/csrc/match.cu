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
  int ipiv[NB];
  GemmSync gs;
};

// Workspace slot M [n][ldm] = [A | pad | B_open]; after elimination + back substitution the
// columns [npad, npad + o) hold Y = A^{-1} B_open and K[e] = -Y (open), -e_j (closed).
// K may alias R (the sweep reuses the R batch buffer): R[e] is fully consumed before K[e] is written.
//
// LU: outer blocks of NB = 64 columns, each factored as two inner panels of PB = 32 (the second
// after a K = 32 update of the block's right half), so that the big trailing updates run with
// K = 64 (half the C-tile traffic per flop of K = 32). Interchanges swap whole augmented rows right
// of the outer block's start (LAPACK getrf semantics restricted to what the solve needs).
__global__ void __launch_bounds__(NT, 1)
    match_kernel(const double *R, int64_t ldr, const double *__restrict__ F,
                 const double *__restrict__ G, const double *__restrict__ Fp,
                 const double *__restrict__ Gp, double a, int n, int64_t ne,
                 const int32_t *__restrict__ n_open, double *K, int64_t ldk, double *ws,
                 int64_t ws_slot, int ldm, int32_t *status) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  MatchSmem &sm = *reinterpret_cast<MatchSmem *>(smem_raw);
  gemm_sync_init(&sm.gs);
  double *Mw = ws + static_cast<int64_t>(blockIdx.x) * ws_slot;
  const int npad = (n + 1) & ~1;
  double *Tg = Mw + static_cast<int64_t>(n) * ldm + 32;  // PB x PB inverse of a diagonal block
  auto Mp = [&](int r, int c) { return Mw + static_cast<int64_t>(r) * ldm + c; };

  for (int64_t e = blockIdx.x; e < ne; e += gridDim.x) {
    int o = n_open ? n_open[e] : n;
    o = o < 0 ? 0 : (o > n ? n : o);
    const int ncols = npad + o;
    const double *Re = R + e * static_cast<int64_t>(n) * ldr;
    const double *Fe = F + e * n, *Ge = G + e * n, *Fpe = Fp + e * n, *Gpe = Gp + e * n;

    // ---- S3: A_ij = G_i d_ij - a R_ij G'_j ; B_ij = F_i d_ij - a R_ij F'_j (4 loads in flight) ----
    for (int i = warp_id(); i < n; i += NW) {
      const double *Ri = Re + static_cast<int64_t>(i) * ldr;
      double *Mi = Mw + static_cast<int64_t>(i) * ldm;
      constexpr int U = 4;
      for (int j0 = lane_id(); j0 < ncols; j0 += 32 * U) {
        double rv[U], sv[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int j = j0 + 32 * q;
          rv[q] = 0.0;
          sv[q] = 0.0;
          if (j < n) {
            rv[q] = Ri[j];
            sv[q] = Gpe[j];
          } else if (j >= npad && j < ncols) {
            rv[q] = Ri[j - npad];
            sv[q] = Fpe[j - npad];
          }
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int j = j0 + 32 * q;
          if (j < ncols) {
            double v = -(a * rv[q]) * sv[q];
            if (j == i) v += Ge[i];
            if (j - npad == i) v += Fe[i];
            Mi[j] = v;
          }
        }
      }
    }
    __syncthreads();

    // ---- S4a: blocked right-looking LU with partial pivoting on [A | B_open] ----
    // Triangular solves with the 32x32 diagonal blocks run as in-place DMMA GEMMs with their
    // explicit inverses (Tg); every operand stays in the slot workspace (aligned, even pitch).
    int singular = 0;
    for (int P0 = 0; P0 < n; P0 += NB) {
      const int W = min(NB, n - P0), w1 = min(PB, W), w2 = W - w1;
      singular |= panel_lu(Mw, ldm, n, P0, w1, P0, ncols, sm.ipiv, sm.redv, sm.redi);
      tri_inv(Mw, ldm, P0, w1, TRI_UNIT_LOWER, sm.tri, Tg);  // L_aa^{-1}
      if (w2 > 0) {
        // right half of the outer block: U_ab = L_aa^{-1} A_ab ; A_.b -= L_.a U_ab ; factor it
        gemm<true, false>(w1, w2, w1, Tg, PB, Mp(P0, P0 + w1), ldm, false, sm.gemm, &sm.gs,
                          EpiStore{Mp(P0, P0 + w1), ldm, 0.0});
        gemm<true, false>(n - P0 - w1, w2, w1, Mp(P0 + w1, P0), ldm, Mp(P0, P0 + w1), ldm, false,
                          sm.gemm, &sm.gs, EpiSub{Mp(P0 + w1, P0 + w1), ldm});
        singular |= panel_lu(Mw, ldm, n, P0 + w1, w2, P0, ncols, sm.ipiv + PB, sm.redv, sm.redi);
      }
      // trailing columns (A part and right-hand sides); when the last block ends on an odd n the
      // zero pad column n is skipped so that every tile row stays 16-byte aligned
      const int ct = min((P0 + W + 1) & ~1, ncols);
      const int nt = ncols - ct;
      if (nt > 0) {
        // U12 = L11^{-1} A12, L11 = [[L_aa, 0], [L_ba, L_bb]]
        gemm<true, false>(w1, nt, w1, Tg, PB, Mp(P0, ct), ldm, false, sm.gemm, &sm.gs,
                          EpiStore{Mp(P0, ct), ldm, 0.0});
        if (w2 > 0) {
          gemm<true, false>(w2, nt, w1, Mp(P0 + w1, P0), ldm, Mp(P0, ct), ldm, false, sm.gemm,
                            &sm.gs, EpiSub{Mp(P0 + w1, ct), ldm});
          tri_inv(Mw, ldm, P0 + w1, w2, TRI_UNIT_LOWER, sm.tri, Tg);  // L_bb^{-1}
          gemm<true, false>(w2, nt, w2, Tg, PB, Mp(P0 + w1, ct), ldm, false, sm.gemm, &sm.gs,
                            EpiStore{Mp(P0 + w1, ct), ldm, 0.0});
        }
        // trailing update with K = W
        if (P0 + W < n)
          gemm<true, false>(n - P0 - W, nt, W, Mp(P0 + W, P0), ldm, Mp(P0, ct), ldm, false,
                            sm.gemm, &sm.gs, EpiSub{Mp(P0 + W, ct), ldm});
      }
    }

    // ---- S4b: blocked back substitution U Y = L^{-1} P B_open (Y in columns [npad, npad+o)) ----
    if (o > 0) {
      double *Y = Mw + npad;
      auto Yr = [&](int r) { return Y + static_cast<int64_t>(r) * ldm; };
      for (int P0 = ((n - 1) / NB) * NB; P0 >= 0; P0 -= NB) {
        const int W = min(NB, n - P0), w1 = min(PB, W), w2 = W - w1;
        if (w2 > 0) {
          tri_inv(Mw, ldm, P0 + w1, w2, TRI_UPPER, sm.tri, Tg);  // U_bb^{-1}
          gemm<true, false>(w2, o, w2, Tg, PB, Yr(P0 + w1), ldm, false, sm.gemm, &sm.gs,
                            EpiStore{Yr(P0 + w1), ldm, 0.0});
          gemm<true, false>(w1, o, w2, Mp(P0, P0 + w1), ldm, Yr(P0 + w1), ldm, false, sm.gemm,
                            &sm.gs, EpiSub{Yr(P0), ldm});
        }
        tri_inv(Mw, ldm, P0, w1, TRI_UPPER, sm.tri, Tg);  // U_aa^{-1}
        gemm<true, false>(w1, o, w1, Tg, PB, Yr(P0), ldm, false, sm.gemm, &sm.gs,
                          EpiStore{Yr(P0), ldm, 0.0});
        if (P0 > 0)
          gemm<true, false>(P0, o, W, Mp(0, P0), ldm, Yr(P0), ldm, false, sm.gemm, &sm.gs,
                            EpiSub{Y, ldm});
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
  // M [n][2 npad] + tail padding for 16-byte bulk copies + the PB x PB diagonal-block inverse
  return nch * (2 * npad) + 32 + 32 * 32 + 32;
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
