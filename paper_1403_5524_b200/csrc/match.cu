// match.cu - S3+S4 of the sweep: K = -(G - aRG')^{-1}(F - aRF')   (BASELINE.json:5).
// The paper is silent on this step (PAPER.md:459-514 stops at R); DESIGN.md §5.2 gives the design:
// one CTA per energy (persistent over energies, workspace slot = blockIdx.x), blocked right-looking
// LU with partial pivoting of A on the augmented matrix [A | B_open] (outer blocks of 256 built from
// 32-wide panels, FP64 DMMA trailing updates through the TMA pipeline of cta_la.cuh), then
// blocked back substitution; only the n_open open columns of B are solved, closed columns of K
// are -e_j (precondition of rmx.h; SURVEY §8(c) reading 9).
#include "cta_la.cuh"
#include "rmx_internal.h"
#include <cstdlib>

namespace rmx {

using namespace la;

#ifdef RMX_PHASES
// per-phase clock64 totals of block 0 (diagnostic build only: python -m paper_1403_5524_b200.build
// --phases -> librmx_phases.so; tools/phases.py reads them)
__device__ unsigned long long g_match_phase[8];
#define PH_MARK(k)                                                          \
  do {                                                                      \
    __syncthreads();                                                        \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                              \
      const unsigned long long now_ = clock64();                            \
      g_match_phase[k] += now_ - ph_t0;                                     \
      ph_t0 = now_;                                                         \
    }                                                                       \
  } while (0)
#else
#define PH_MARK(k) \
  do {             \
  } while (0)
#endif

struct MatchSmem {
  union {  // the triangle scratch is only used between gemm calls
    double gemm[GEMM_SMEM_DOUBLES];
    double tri[TRI_SMEM_DOUBLES];
  };
  double redv[NW];
  int redi[NW];
  int ipiv[NB];
  double ubuf[SPW * PB];
  GemmSync gs;
};


// Workspace slot: M [n][ldm] = [A P | pad | B_open] with the unknowns permuted closed-first (P);
// Tg [32][32] (inverse of a diagonal block). After elimination + back substitution the columns
// [npad, npad + o) of M hold Y = (A P)^{-1} B_open, and K[e] = -P Y (open columns), -e_j (closed
// columns); with open_rows_only (the sweep: the T epilogue reads K_oo only) just K_oo is solved for
// and written.
// K may alias R (the sweep reuses the R batch buffer): R[e] is fully consumed before K[e] is written.
// Triangular solves with the 32x32 diagonal blocks run as in-place DMMA GEMMs with their explicit
// inverses (MAGMA-style); interchanges swap whole augmented rows right of the outer block start.
__global__ void __launch_bounds__(NT, 1)
    match_kernel(const double *R, int64_t ldr, const double *__restrict__ F,
                 const double *__restrict__ G, const double *__restrict__ Fp,
                 const double *__restrict__ Gp, double a, int n, int64_t ne,
                 const int32_t *__restrict__ n_open, double *K, int64_t ldk, double *ws,
                 int64_t ws_slot, const CUtensorMap *views, int32_t *status, int open_rows_only) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  MatchSmem &sm = *reinterpret_cast<MatchSmem *>(smem_raw);
  const MatchLayout L = match_layout(n);
  const int ldm = static_cast<int>(L.ldm), npad = static_cast<int>(L.npad);
  double *slot = ws + static_cast<int64_t>(blockIdx.x) * ws_slot;
  const MatView Mv{views + (blockIdx.x * 2 + 0) * NVIEW, slot + L.m_off, ldm, n};
  const MatView Tv{views + (blockIdx.x * 2 + 1) * NVIEW, slot + L.tg_off, TG, TG};
  double *Mw = Mv.base;
  // LU sub-panel staging: shared memory up to kSmemPanelChannels, the slot's scratch beyond (generic
  // addressing: the same panel_lu code; __syncthreads orders the global accesses within the CTA)
  double *spbuf = (n <= kSmemPanelChannels) ? sm.gemm : slot + L.sp_off;
  double *smg = sm.gemm;
  GemmSync *gs = &sm.gs;

  for (int64_t e = blockIdx.x; e < ne; e += gridDim.x) {
    int o = n_open ? n_open[e] : n;
    o = o < 0 ? 0 : (o > n ? n : o);
    const int ncols = npad + o;
    const double *Re = R + e * static_cast<int64_t>(n) * ldr;
    const double *Fe = F + e * n, *Ge = G + e * n, *Fpe = Fp + e * n, *Gpe = Gp + e * n;
#ifdef RMX_PHASES
    unsigned long long ph_t0 = clock64();
#endif
    // unknowns ordered closed channels first, open last: column q of A holds channel
    // jq = (q < nc) ? o + q : q - nc, so the open unknowns are the LAST rows of the triangular
    // solve and back substitution for K_oo can stop after them (SURVEY §8(a) S4 flops:
    // (2/3)n^3 + n^2 n_o + n_o^3 instead of (2/3)n^3 + 2 n^2 n_o)
    const int nc = n - o;

    // ---- S3: A_ij = G_i d_ij - a R_ij G'_j ; B_ij = F_i d_ij - a R_ij F'_j (16 loads in flight) ----
    for (int i = warp_id(); i < n; i += NW) {
      const double *Ri = Re + static_cast<int64_t>(i) * ldr;
      double *Mi = Mw + static_cast<int64_t>(i) * ldm;
      constexpr int U = 8;
      for (int j0 = lane_id(); j0 < ncols; j0 += 32 * U) {
        double rv[U], sv[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int j = j0 + 32 * q;
          rv[q] = 0.0;
          sv[q] = 0.0;
          if (j < n) {
            const int jc = (j < nc) ? o + j : j - nc;
            rv[q] = Ri[jc];
            sv[q] = Gpe[jc];
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
            if (j < n && ((j < nc) ? o + j : j - nc) == i) v += Ge[i];
            if (j - npad == i) v += Fe[i];
            Mi[j] = v;
          }
        }
      }
    }
    __syncthreads();

    PH_MARK(0);  // formation pass
    // ---- S4a: blocked right-looking LU with partial pivoting on [A | B_open] ----
    // Outer blocks of 256 columns made of two 128-wide sub-blocks a, b. A sub-block is factored as
    // four 32-wide panels (each followed by a K = 32 update of the sub-block's remaining columns);
    // U12a = L11a^{-1} A12 as ONE in-place DMMA GEMM with the explicit 128 x 128 inverse (one
    // 128-row tile row) over every column right of a; sub-block b's columns are updated and factored
    // (its row interchanges run over the whole block, L21a included, while the trailing columns of
    // all rows below a still wait for a's update), b's U rows get a's update and U12b; then ONE
    // trailing update with K = 256 (C read and written once per 256 columns instead of twice).
    int singular = 0;
    auto factor_sub = [&](int c0, int Wblk, int sc0) {
      for (int q0 = 0; q0 < Wblk; q0 += PB) {
        const int c = c0 + q0, wq = min(PB, Wblk - q0), rem = Wblk - q0 - wq;
        singular |= panel_lu(Mw, ldm, n, c, wq, sc0, ncols, sm.ipiv + q0, spbuf, sm.ubuf, sm.redv,
                             sm.redi);
        if (rem > 0) {
          // sub-block columns right of this panel: U rows = L_qq^{-1} A ; rows below -= L U
          tri_inv64(Mw, ldm, c, wq, TRI_UNIT_LOWER, sm.tri, Tv.base, TG);
          gemm_set(wq, rem, wq, opk(Tv, 0, 0), opn(Mv, c, c + wq), Mv, c, c + wq, false, 0.0, smg, gs);
          gemm_sub(n - c - wq, rem, wq, opk(Mv, c + wq, c), opn(Mv, c, c + wq), Mv, c + wq, c + wq,
                   false, smg, gs);
        }
      }
    };
    for (int P0 = 0; P0 < n; P0 += 2 * NB) {
      const int W = min(2 * NB, n - P0), Wa = min(NB, W), Wb = W - Wa, ca = P0 + Wa;
      // trailing columns (A part and right-hand sides); when the last block ends on an odd n the
      // zero pad column n is skipped so that every C row stays 16-byte aligned
      const int ct = min((P0 + W + 1) & ~1, ncols);
      const int nt = ncols - ct;
      factor_sub(P0, Wa, P0);
      PH_MARK(1);  // panels (panel_lu + in-block K = 32 updates)
      if (Wb == 0 && nt == 0) continue;
      tri_inv128(Mv, P0, Wa, TRI_UNIT_LOWER, Tv, smg, gs);  // L11a^{-1}
      PH_MARK(5);
      const int c2 = Wb > 0 ? ca : ct;  // ca = P0 + 128 is even when Wb > 0
      gemm_set(Wa, ncols - c2, Wa, opk(Tv, 0, 0), opn(Mv, P0, c2), Mv, P0, c2, false, 0.0, smg, gs);
      PH_MARK(2);
      if (Wb > 0) {
        gemm_sub(n - ca, Wb, Wa, opk(Mv, ca, P0), opn(Mv, P0, ca), Mv, ca, ca, false, smg, gs);
        PH_MARK(2);
        factor_sub(ca, Wb, P0);
        PH_MARK(1);
        if (nt > 0) {
          gemm_sub(Wb, nt, Wa, opk(Mv, ca, P0), opn(Mv, P0, ct), Mv, ca, ct, false, smg, gs);
          PH_MARK(2);
          tri_inv128(Mv, ca, Wb, TRI_UNIT_LOWER, Tv, smg, gs);  // L22b^{-1}
          PH_MARK(5);
          gemm_set(Wb, nt, Wb, opk(Tv, 0, 0), opn(Mv, ca, ct), Mv, ca, ct, false, 0.0, smg, gs);
        }
      }
      if (nt > 0 && P0 + W < n)
        gemm_sub(n - P0 - W, nt, W, opk(Mv, P0 + W, P0), opn(Mv, P0, ct), Mv, P0 + W, ct, false, smg, gs);
      PH_MARK(2);  // U12 + K = 256 trailing update
    }

    // ---- S4b: blocked back substitution U Y = L^{-1} P B_open (Y = columns [npad, npad+o)) ----
    // rows_needed: the open unknowns [nc, n) only (sweep), or all (K's closed rows are outputs of
    // rmx_match_K); the blocks and the update order of rows >= nc are the same either way, so
    // K_oo is bitwise identical in both modes
    const int rlo = open_rows_only ? nc : 0;
    // 128-row blocks taken in pairs (a above b) from the bottom, the pairing independent of rlo:
    // Y_b = U_bb^{-1} Y_b; Y_a -= U_ab Y_b; Y_a = U_aa^{-1} Y_a; then ONE update of the rows above
    // the pair with K = 256 (the C rows read and written once per 256 solved rows)
    if (o > 0) {
      for (int Pb = ((n - 1) / NB) * NB; Pb >= 0 && Pb + NB > rlo; Pb -= 2 * NB) {
        const int Wb = min(NB, n - Pb), Pa = Pb - NB;
        const bool has_a = Pa >= 0 && Pa + NB > rlo;
        PH_MARK(3);
        tri_inv128(Mv, Pb, Wb, TRI_UPPER, Tv, smg, gs);  // U_bb^{-1}
        PH_MARK(6);
        gemm_set(Wb, o, Wb, opk(Tv, 0, 0), opn(Mv, Pb, npad), Mv, Pb, npad, false, 0.0, smg, gs);
        if (has_a) {
          gemm_sub(NB, o, Wb, opk(Mv, Pa, Pb), opn(Mv, Pb, npad), Mv, Pa, npad, false, smg, gs);
          PH_MARK(3);
          tri_inv128(Mv, Pa, NB, TRI_UPPER, Tv, smg, gs);  // U_aa^{-1}
          PH_MARK(6);
          gemm_set(NB, o, NB, opk(Tv, 0, 0), opn(Mv, Pa, npad), Mv, Pa, npad, false, 0.0, smg, gs);
          if (Pa > rlo)
            gemm_sub(Pa - rlo, o, NB + Wb, opk(Mv, rlo, Pa), opn(Mv, Pa, npad), Mv, rlo, npad, false, smg, gs);
        } else if (Pb > rlo) {
          gemm_sub(Pb - rlo, o, Wb, opk(Mv, rlo, Pb), opn(Mv, Pb, npad), Mv, rlo, npad, false, smg, gs);
        }
      }
    }

    PH_MARK(3);  // back substitution
    // ---- output: K = -Y (open columns), -e_j (closed columns); status ----
    int bad = 0;
    double *Ke = K + e * static_cast<int64_t>(n) * ldk;
    const int nrows = open_rows_only ? o : n;
    const int ncolk = open_rows_only ? o : n;
    for (int i = warp_id(); i < nrows; i += NW) {
      const int qi = (i < o) ? nc + i : i - o;  // solution row of channel i
      const double *Yi = Mw + static_cast<int64_t>(qi) * ldm + npad;
      double *Ki = Ke + static_cast<int64_t>(i) * ldk;
      constexpr int U = 8;  // U independent loads in flight per lane
      for (int j0 = lane_id(); j0 < ncolk; j0 += 32 * U) {
        double y[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + 32 * u;
          y[u] = (j < o && j < ncolk) ? Yi[j] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + 32 * u;
          if (j >= ncolk) continue;
          double v;
          if (j < o) {
            v = -y[u];
            if (i < o && !isfinite(v)) bad = 1;
          } else {
            v = (i == j) ? -1.0 : 0.0;
          }
          Ki[j] = v;
        }
      }
    }
    bad = __syncthreads_or(bad);
    PH_MARK(4);  // output
    if (threadIdx.x == 0) {
      if (singular)
        set_status(status, e, RMX_E_SINGULAR);
      else if (bad)
        set_status(status, e, RMX_E_NONFINITE);
    }
  }
}

int64_t match_ws_doubles_per_slot(int64_t nch) { return match_layout(nch).slot; }

#ifdef RMX_PHASES
extern "C" int rmx_debug_match_phases(unsigned long long *out) {
  cudaDeviceSynchronize();
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_match_phase, sizeof(g_match_phase)));
}
// panel_lu sub-steps: staging, factor, write-back + interchanges, rank-w update
extern "C" int rmx_debug_panel_phases(unsigned long long *out) {
  cudaDeviceSynchronize();
  return static_cast<int>(cudaMemcpyFromSymbol(out, la::g_panel_phase, 6 * sizeof(unsigned long long)));
}
#endif

// Matrices of one slot whose TMA descriptors the kernel uses: (M, Tg), NVIEW box shapes each.
void match_view_specs(int64_t nch, std::vector<MatSpec> &specs) {
  const MatchLayout L = match_layout(nch);
  specs = {MatSpec{L.m_off, nch, L.ldm, L.ldm}, MatSpec{L.tg_off, TG, TG, TG}};
}

cudaError_t launch_match(const double *R, const double *F, const double *G, const double *Fp,
                         const double *Gp, double a, int64_t nch, int64_t ne, const int32_t *n_open,
                         double *K, double *ws, int64_t ws_slot, const CUtensorMap *views, int64_t ws_slots,
                         int32_t *status, cudaStream_t st, int open_rows_only) {
  cudaError_t ce = ensure_smem_attr(reinterpret_cast<const void *>(match_kernel), sizeof(MatchSmem));
  if (ce != cudaSuccess) return ce;
  const int grid = static_cast<int>(ne < ws_slots ? ne : ws_slots);
  match_kernel<<<grid, NT, sizeof(MatchSmem), st>>>(R, nch, F, G, Fp, Gp, a, static_cast<int>(nch),
                                                    ne, n_open, K, nch, ws, ws_slot, views, status,
                                                    open_rows_only);
  return cudaGetLastError();
}

}  // namespace rmx
