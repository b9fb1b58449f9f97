// tepi.cu - S5 of the sweep: T = 2i K_oo (I - i K_oo)^{-1} and |T_ij|^2 (BASELINE.json:5).
// Real SPD route (reading T2): with K_oo symmetric,
//   (I - iK)^{-1} = (I + iK)(I + K^2)^{-1}  =>  T = 2iX - 2KX,  X = (I + K K^T)^{-1} K
// so Re T = -2P, Im T = 2X with P = K X, and |T_ij|^2 = 4 (X_ij^2 + P_ij^2). Per energy (one CTA,
// persistent over energies): S = I + K K^T (lower, DMMA GEMM), blocked Cholesky S = L L^T, two
// blocked triangular solves for X, P = K X (DMMA GEMM), then an epilogue pass writing |T|^2
// (optional) and the row sums sum_j |T_ij|^2 in a fixed order (deterministic).
// |T|^2 and the row sums are invariant under K -> -K, so the sweep may pass Y = -K directly.
#include "cta_la.cuh"
#include "rmx_internal.h"

namespace rmx {

using namespace la;

struct TepiSmem {
  double gemm[GEMM_SMEM_DOUBLES];
  double tri[TRI_SMEM_DOUBLES];
  GemmSync gs;
};

// Factorisation / solves use outer blocks of NB = 64 (two inner 32-wide triangles) so that the
// big updates run with K = 64.
__global__ void __launch_bounds__(NT, 1)
    tepi_kernel(const double *K, int64_t ldk, int64_t kstride, int n, int64_t ne,
                const int32_t *__restrict__ n_open, double *T2, const int64_t *t2_slot,
                double *rowsum, double *ws, int64_t ws_slot, int ldo, int32_t *status) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  TepiSmem &sm = *reinterpret_cast<TepiSmem *>(smem_raw);
  gemm_sync_init(&sm.gs);
  double *S = ws + static_cast<int64_t>(blockIdx.x) * ws_slot;  // o x ldo; later holds P
  double *X = S + static_cast<int64_t>(n) * ldo;                // o x ldo
  double *Kc = X + static_cast<int64_t>(n) * ldo;               // o x ldo: aligned copy of K_oo
  double *Tg = Kc + static_cast<int64_t>(n) * ldo + 32;          // PB x PB diagonal-block inverse
  auto Sp = [&](int r, int c) { return S + static_cast<int64_t>(r) * ldo + c; };
  auto Xr = [&](int r) { return X + static_cast<int64_t>(r) * ldo; };

  for (int64_t e = blockIdx.x; e < ne; e += gridDim.x) {
    int o = n_open ? n_open[e] : n;
    o = o < 0 ? 0 : (o > n ? n : o);
    const double *Ke = K + e * kstride;
    double *T2e = nullptr;
    if (T2) {
      const int64_t slot = t2_slot ? t2_slot[e] : e;
      if (slot >= 0) T2e = T2 + slot * static_cast<int64_t>(n) * n;
    }
    int bad = 0;
    if (o > 0) {
      // Kc = X = K_oo (16-byte aligned, even pitch: operands of the bulk-copy GEMM pipeline)
      for (int i = warp_id(); i < o; i += NW)
        for (int j = lane_id(); j < o; j += 32) {
          const double v = Ke[static_cast<int64_t>(i) * ldk + j];
          Kc[static_cast<int64_t>(i) * ldo + j] = v;
          Xr(i)[j] = v;
        }
      __syncthreads();
      // S = I + K_oo K_oo^T (lower tiles)
      gemm<true, true>(o, o, o, Kc, ldo, Kc, ldo, true, sm.gemm, &sm.gs, EpiStore{S, ldo, 1.0});
      // blocked Cholesky S = L L^T (lower); panel solves L21 = S21 L11^{-T} as in-place GEMMs
      for (int P0 = 0; P0 < o; P0 += NB) {
        const int W = min(NB, o - P0), w1 = min(PB, W), w2 = W - w1;
        bad |= chol_diag(S, ldo, P0, w1, sm.tri);
        tri_inv(S, ldo, P0, w1, TRI_LOWER, sm.tri, Tg);
        if (P0 + w1 < o)
          gemm<true, true>(o - P0 - w1, w1, w1, Sp(P0 + w1, P0), ldo, Tg, PB, false, sm.gemm, &sm.gs,
                           EpiStore{Sp(P0 + w1, P0), ldo, 0.0});
        if (w2 > 0) {
          gemm<true, true>(o - P0 - w1, w2, w1, Sp(P0 + w1, P0), ldo, Sp(P0 + w1, P0), ldo, false,
                           sm.gemm, &sm.gs, EpiSub{Sp(P0 + w1, P0 + w1), ldo});
          bad |= chol_diag(S, ldo, P0 + w1, w2, sm.tri);
          if (P0 + W < o) {
            tri_inv(S, ldo, P0 + w1, w2, TRI_LOWER, sm.tri, Tg);
            gemm<true, true>(o - P0 - W, w2, w2, Sp(P0 + W, P0 + w1), ldo, Tg, PB, false, sm.gemm,
                             &sm.gs, EpiStore{Sp(P0 + W, P0 + w1), ldo, 0.0});
          }
        }
        if (P0 + W < o) {
          const int m2 = o - P0 - W;
          gemm<true, true>(m2, m2, W, Sp(P0 + W, P0), ldo, Sp(P0 + W, P0), ldo, true, sm.gemm, &sm.gs,
                           EpiSub{Sp(P0 + W, P0 + W), ldo});
        }
      }
      // forward: L Z = K  (X holds K_oo)
      for (int P0 = 0; P0 < o; P0 += NB) {
        const int W = min(NB, o - P0), w1 = min(PB, W), w2 = W - w1;
        tri_inv(S, ldo, P0, w1, TRI_LOWER, sm.tri, Tg);
        gemm<true, false>(w1, o, w1, Tg, PB, Xr(P0), ldo, false, sm.gemm, &sm.gs, EpiStore{Xr(P0), ldo, 0.0});
        if (w2 > 0) {
          gemm<true, false>(w2, o, w1, Sp(P0 + w1, P0), ldo, Xr(P0), ldo, false, sm.gemm, &sm.gs,
                            EpiSub{Xr(P0 + w1), ldo});
          tri_inv(S, ldo, P0 + w1, w2, TRI_LOWER, sm.tri, Tg);
          gemm<true, false>(w2, o, w2, Tg, PB, Xr(P0 + w1), ldo, false, sm.gemm, &sm.gs,
                            EpiStore{Xr(P0 + w1), ldo, 0.0});
        }
        if (P0 + W < o)
          gemm<true, false>(o - P0 - W, o, W, Sp(P0 + W, P0), ldo, Xr(P0), ldo, false, sm.gemm, &sm.gs,
                            EpiSub{Xr(P0 + W), ldo});
      }
      // backward: L^T X = Z
      for (int P0 = ((o - 1) / NB) * NB; P0 >= 0; P0 -= NB) {
        const int W = min(NB, o - P0), w1 = min(PB, W), w2 = W - w1;
        if (w2 > 0) {
          tri_inv(S, ldo, P0 + w1, w2, TRI_LOWER, sm.tri, Tg);
          // X_b = L_bb^{-T} X_b : A(m,k) = Tg[k][m] -> [K][M]
          gemm<false, false>(w2, o, w2, Tg, PB, Xr(P0 + w1), ldo, false, sm.gemm, &sm.gs,
                             EpiStore{Xr(P0 + w1), ldo, 0.0});
          // X_a -= (L[P0+w1:P0+W, P0:P0+w1])^T X_b
          gemm<false, false>(w1, o, w2, Sp(P0 + w1, P0), ldo, Xr(P0 + w1), ldo, false, sm.gemm, &sm.gs,
                             EpiSub{Xr(P0), ldo});
        }
        tri_inv(S, ldo, P0, w1, TRI_LOWER, sm.tri, Tg);
        gemm<false, false>(w1, o, w1, Tg, PB, Xr(P0), ldo, false, sm.gemm, &sm.gs, EpiStore{Xr(P0), ldo, 0.0});
        if (P0 > 0)
          // X[0:P0] -= (L[P0:P0+W, 0:P0])^T X[P0:P0+W]; A(i,k) = S[(P0+k)*ldo + i] -> [K][M]
          gemm<false, false>(P0, o, W, Sp(P0, 0), ldo, Xr(P0), ldo, false, sm.gemm, &sm.gs,
                             EpiSub{X, ldo});
      }
      // P = K_oo X  (into S's storage)
      gemm<true, false>(o, o, o, Kc, ldo, X, ldo, false, sm.gemm, &sm.gs, EpiStore{S, ldo, 0.0});
    }
    // epilogue: |T|^2 = 4 (X^2 + P^2), row sums in fixed order
    for (int i = warp_id(); i < n; i += NW) {
      double s = 0.0;
      for (int j = lane_id(); j < n; j += 32) {
        double v = 0.0;
        if (i < o && j < o) {
          const double x = Xr(i)[j];
          const double p = *Sp(i, j);
          v = 4.0 * fma(x, x, p * p);
          if (!isfinite(v)) bad = 1;
        }
        if (T2e) T2e[static_cast<int64_t>(i) * n + j] = v;
        s += v;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (rowsum && lane_id() == 0) rowsum[e * n + i] = s;
    }
    bad = __syncthreads_or(bad);
    if (bad && threadIdx.x == 0) set_status(status, e, RMX_E_NONFINITE);
  }
}

int64_t tepi_ws_doubles_per_slot(int64_t nch) {
  const int64_t npad = (nch + 1) & ~1LL;
  return 3 * nch * npad + 32 + 32 * 32 + 32;  // + tail padding for 16-byte bulk copies of odd-width C tiles
}

cudaError_t launch_tepi(const double *K, int64_t ldk, int64_t kstride, int64_t nch, int64_t ne,
                        const int32_t *n_open, double *T2, const int64_t *t2_slot, double *rowsum,
                        double *ws, int64_t ws_slots, int32_t *status, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t ce = cudaFuncSetAttribute(tepi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(sizeof(TepiSmem)));
    if (ce != cudaSuccess) return ce;
    attr = true;
  }
  const int64_t npad = (nch + 1) & ~1LL;
  const int grid = static_cast<int>(ne < ws_slots ? ne : ws_slots);
  tepi_kernel<<<grid, NT, sizeof(TepiSmem), st>>>(K, ldk, kstride, static_cast<int>(nch), ne, n_open,
                                                  T2, t2_slot, rowsum, ws,
                                                  tepi_ws_doubles_per_slot(nch),
                                                  static_cast<int>(npad), status);
  return cudaGetLastError();
}

}  // namespace rmx
