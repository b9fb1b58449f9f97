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
  union {  // the triangle scratch is only used between gemm calls
    double gemm[GEMM_SMEM_DOUBLES];
    double tri[TRI_SMEM_DOUBLES];
  };
  GemmSync gs;
};


// P[j][i] = P[i][j] for j > i (upper triangle from the lower one), 32x32 blocks staged through
// shared memory so that both the reads and the writes are coalesced row segments.
__device__ __forceinline__ void mirror_lower(double *P, int64_t ld, int o, double *smem) {
  constexpr int TL = 33;
  const int nb = (o + 31) / 32;
  double *tile = smem + warp_id() * 32 * TL;  // one 32x33 tile per warp
  const int lane = lane_id();
  __syncthreads();
  for (int b = warp_id(); b < nb * (nb + 1) / 2; b += NW) {
    int bi = 0, rem = b;
    while (rem > bi) {
      rem -= bi + 1;
      ++bi;
    }
    const int bj = rem;  // bj <= bi: lower block (bi, bj) -> upper block (bj, bi)
    for (int r = 0; r < 32; ++r) {
      const int gi = bi * 32 + r, gj = bj * 32 + lane;
      tile[r * TL + lane] = (gi < o && gj < o) ? P[static_cast<int64_t>(gi) * ld + gj] : 0.0;
    }
    __syncwarp();
    for (int r = 0; r < 32; ++r) {  // row r of the upper block = column r of the lower block
      const int gi = bj * 32 + r, gj = bi * 32 + lane;
      if (gi < o && gj < o && gj > gi) P[static_cast<int64_t>(gi) * ld + gj] = tile[lane * TL + r];
    }
    __syncwarp();
  }
  __syncthreads();
}

// Workspace slot: S (then P) [o][ldo], X [o][ldo], Kc [o][ldo] (aligned copy of K_oo),
// Tg [32][32] (inverse of a 32x32 diagonal block of L: triangular solves run as DMMA GEMMs).
// Factorisation / solves use outer blocks of NB = 64 (two inner 32-wide triangles) so that the
// big updates run with K = 64.
__global__ void __launch_bounds__(NT, 1)
    tepi_kernel(const double *K, int64_t ldk, int64_t kstride, int n, int64_t ne,
                const int32_t *__restrict__ n_open, double *T2, const int64_t *t2_slot,
                double *rowsum, LevelSums lv, PhotoArgs pa, double *ws, int64_t ws_slot,
                const CUtensorMap *views, int32_t *status) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  TepiSmem &sm = *reinterpret_cast<TepiSmem *>(smem_raw);
  const TepiLayout L = tepi_layout(n);
  const int ldo = static_cast<int>(L.ldo);
  double *slot = ws + static_cast<int64_t>(blockIdx.x) * ws_slot;
  const CUtensorMap *vw = views + blockIdx.x * 5 * NVIEW;
  const MatView Sv{vw + 0 * NVIEW, slot + L.s_off, ldo};
  const MatView Xv{vw + 1 * NVIEW, slot + L.x_off, ldo};
  const MatView Kv{vw + 2 * NVIEW, slot + L.k_off, ldo};
  const MatView Tv{vw + 3 * NVIEW, slot + L.tg_off, TG};
  const MatView Ttv{vw + 4 * NVIEW, slot + L.tt_off, ldo};
  double *S = Sv.base;
  double *smg = sm.gemm;
  GemmSync *gs = &sm.gs;

  for (int64_t e = blockIdx.x; e < ne; e += gridDim.x) {
    int o = n_open ? n_open[e] : n;
    o = o < 0 ? 0 : (o > n ? n : o);
    const double *Ke = K + e * kstride;
    double *T2e = nullptr;
    if (T2) {
      const int64_t ts = t2_slot ? t2_slot[e] : e;
      if (ts >= 0) T2e = T2 + ts * static_cast<int64_t>(n) * n;
    }
    int bad = 0;
    if (o > 0) {
      // Kc = K_oo (aligned, even pitch: operand of the TMA GEMM pipeline); X = 0 (Z = L^{-1} is
      // built there, its strict upper part must stay zero)
      for (int i = warp_id(); i < o; i += NW) {
        const double *src = Ke + static_cast<int64_t>(i) * ldk;
        double *dk = Kv.at(i, 0), *dx = Xv.at(i, 0);
        constexpr int U = 8;  // 8 independent loads in flight per lane
        for (int j0 = lane_id(); j0 < o; j0 += 32 * U) {
          double v[U];
#pragma unroll
          for (int q = 0; q < U; ++q) v[q] = (j0 + 32 * q < o) ? src[j0 + 32 * q] : 0.0;
#pragma unroll
          for (int q = 0; q < U; ++q)
            if (j0 + 32 * q < o) {
              dk[j0 + 32 * q] = v[q];
              dx[j0 + 32 * q] = 0.0;
            }
        }
      }
      if (pa.g) {
        // NEXT-1 (10): v_j = (1/2)(g_j F'_j + sum_i g_i G'_i K_ij) into Kc column o; gG_i staged in
        // shared memory, i ascending
        const double *ge = pa.g + e * n, *Fpe = pa.Fp + e * n, *Gpe = pa.Gp + e * n;
        double *gG = sm.gemm;
        for (int i = threadIdx.x; i < n; i += NT) gG[i] = ge[i] * Gpe[i];
        __syncthreads();
        for (int j = threadIdx.x; j < o; j += NT) {
          double s = ge[j] * Fpe[j];
          for (int i = 0; i < n; ++i) s = fma(gG[i], Ke[static_cast<int64_t>(i) * ldk + j], s);
          *Kv.at(j, o) = 0.5 * s;
        }
      }
      __syncthreads();
      // S = I + K_oo K_oo^T (lower tiles)
      gemm_set(o, o, o, opk(Kv, 0, 0), opk(Kv, 0, 0), Sv, 0, 0, true, 1.0, smg, gs);
      // blocked Cholesky S = L L^T (lower), 128-wide blocks: diagonal block in smem, then
      // L21 = S21 L11^{-T} as one in-place GEMM with the explicit inverse, then the K = 128 update
      for (int P0 = 0; P0 < o; P0 += NB) {
        const int W = min(NB, o - P0);
        bad |= chol_diag_blk(S, ldo, P0, W, sm.tri);
        if (P0 + W < o) {
          tri_inv128(Sv, P0, W, TRI_LOWER, Tv, smg, gs);
          // L21^T = L11^{-1} S21^T (stored transposed, in place): one 128-row tile row, so each
          // output tile depends only on its own rows of S21
          gemm_set_t(W, o - P0 - W, W, opk(Tv, 0, 0), opk(Sv, P0 + W, P0), Sv, P0 + W, P0, smg, gs);
          const int m2 = o - P0 - W;
          gemm_sub(m2, m2, W, opk(Sv, P0 + W, P0), opk(Sv, P0 + W, P0), Sv, P0 + W, P0 + W, true,
                   smg, gs);
        }
      }
      // Z = L^{-1} (lower, in X) block row by block row:  Z_bb = L_bb^{-1} (128 x 128 inverse),
      // Z_{b,0:b} = -Z_bb (L_{b,0:b} Z_{0:b,0:b}); the triangular factor Z of the product skips its
      // zero k slices (kband 2), so the step costs (1/3) o^3 in total
      for (int R0 = 0; R0 < o; R0 += NB) {
        const int W = min(NB, o - R0);
        tri_inv128(Sv, R0, W, TRI_LOWER, Tv, smg, gs);
        if (R0 > 0) {
          gemm_set_kb(W, R0, R0, opk(Sv, R0, 0), opn(Xv, 0, 0), Ttv, 0, 0, false, 2, smg, gs);
          gemm_sub(W, R0, W, opk(Tv, 0, 0), opn(Ttv, 0, 0), Xv, R0, 0, false, smg, gs);
        }
        for (int q = threadIdx.x; q < W * W; q += NT) {
          const int r = q / W, cc = q % W;
          *Xv.at(R0 + r, R0 + cc) = Tv.base[r * TG + cc];  // upper part of Tv is zero
        }
        __syncthreads();
      }
      // S^{-1} = Z^T Z (lower tiles, kband 1: Z(k, i) = 0 for k < i), over L, then mirrored
      gemm_set_kb(o, o, o, opn(Xv, 0, 0), opn(Xv, 0, 0), Sv, 0, 0, true, 1, smg, gs);
      mirror_lower(S, ldo, o, sm.gemm);
      // X = S^{-1} K_oo = (I + K^2)^{-1} K: symmetric (K_oo symmetric, reading M1), lower tiles then
      // mirrored; overwrites Z
      gemm_set(o, o, o, opk(Sv, 0, 0), opn(Kv, 0, 0), Xv, 0, 0, true, 0.0, smg, gs);
      mirror_lower(Xv.base, ldo, o, sm.gemm);
      if (pa.g) {
        // NEXT-1 (11): y = S^{-1} v into X column o (v in Kc column o)
        double *vs = sm.gemm;
        for (int j = threadIdx.x; j < o; j += NT) vs[j] = *Kv.at(j, o);
        __syncthreads();
        for (int i = warp_id(); i < o; i += NW) {
          const double *sr = Sv.at(i, 0);
          double t = 0.0;
          for (int j = lane_id(); j < o; j += 32) t = fma(sr[j], vs[j], t);
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
          if (lane_id() == 0) *Xv.at(i, o) = t;
        }
      }
      // P = K_oo X = K S^{-1} K = I - S^{-1} (K and S commute): in place of S^{-1}
      __syncthreads();
      for (int i = warp_id(); i < o; i += NW) {
        double *pr = Sv.at(i, 0);
        for (int j = lane_id(); j < o; j += 32) pr[j] = (i == j ? 1.0 : 0.0) - pr[j];
      }
      __syncthreads();
    }
    // epilogue: |T|^2 = 4 (X^2 + P^2), row sums in fixed order
    for (int i = warp_id(); i < n; i += NW) {
      double s = 0.0;
      const double *xr = Xv.at(i, 0), *pr = Sv.at(i, 0);
      constexpr int U = 4;  // 2U independent loads in flight per lane
      for (int j0 = lane_id(); j0 < n; j0 += 32 * U) {
        double xv[U], pv[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int j = j0 + 32 * q;
          const bool in = i < o && j < o;
          xv[q] = in ? xr[j] : 0.0;
          pv[q] = in ? pr[j] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int j = j0 + 32 * q;
          if (j < n) {
            const double v = 4.0 * fma(xv[q], xv[q], pv[q] * pv[q]);
            if (!isfinite(v)) bad = 1;
            if (T2e) T2e[static_cast<int64_t>(i) * n + j] = v;
            s += v;
          }
        }
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (rowsum && lane_id() == 0) rowsum[e * n + i] = s;
    }
    if (pa.g) {
      // NEXT-1 (11)-(12): y = X[:, o] = (I + K_oo^2)^{-1} v; M = y + i K_oo y; |M_j|^2; sigma.
      // Row sums in a fixed order: warp w takes rows w, w + NW, ...; warps combined in order.
      double *ys = sm.gemm, *wsum = sm.gemm + n + 1;
      __syncthreads();
      for (int j = threadIdx.x; j < o; j += NT) ys[j] = *Xv.at(j, o);
      __syncthreads();
      double part = 0.0;
      for (int i = warp_id(); i < n; i += NW) {
        double m2 = 0.0;
        if (i < o) {
          const double *kr = Kv.at(i, 0);
          double t = 0.0;
          for (int j = lane_id(); j < o; j += 32) t = fma(kr[j], ys[j], t);
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
          m2 = fma(ys[i], ys[i], t * t);
        }
        if (!isfinite(m2)) bad = 1;
        if (pa.mabs2 && lane_id() == 0) pa.mabs2[e * n + i] = m2;
        part += m2;
      }
      if (lane_id() == 0) wsum[warp_id()] = part;
      __syncthreads();
      if (threadIdx.x == 0) {
        double s = 0.0;
        for (int q = 0; q < NW; ++q) s += wsum[q];
        pa.sigma[e] = pa.C * (pa.E[e] - pa.E0) * s;
      }
      __syncthreads();
    }
    if (lv.omega && o > 0) {
      // NEXT-2: level-pair collision strengths
      //   Omega_ab += g sum_{i in a} sum_{j in b} |T_ij|^2
      // for the open levels (channel ranges [ls[a], ls[a+1]) inside [0, o)). One warp per level
      // a, one lane per level b; i ascending, then j ascending (fixed order, no atomics).
      int nlo = 0;
      while (nlo < lv.nlevel && lv.level_start[nlo + 1] <= o) ++nlo;
      double *Om = lv.omega + e * lv.nlevel * lv.nlevel;
      for (int la = warp_id(); la < nlo; la += NW) {
        const int i0 = lv.level_start[la], i1 = lv.level_start[la + 1];
        for (int lb = lane_id(); lb < nlo; lb += 32) {
          const int j0 = lv.level_start[lb], j1 = lv.level_start[lb + 1];
          double acc = 0.0;
          for (int i = i0; i < i1; ++i) {
            const double *xr = Xv.at(i, 0), *pr = Sv.at(i, 0);
            for (int j = j0; j < j1; ++j) acc += 4.0 * fma(xr[j], xr[j], pr[j] * pr[j]);
          }
          Om[static_cast<int64_t>(la) * lv.nlevel + lb] += lv.g * acc;
        }
      }
    }
    bad = __syncthreads_or(bad);
    if (bad && threadIdx.x == 0) set_status(status, e, RMX_E_NONFINITE);
  }
}

int64_t tepi_ws_doubles_per_slot(int64_t nch) { return tepi_layout(nch).slot; }

// Matrices of one slot whose TMA descriptors the kernel uses: (S, X, Kc, Tg, Tt), NVIEW boxes each.
void tepi_view_specs(int64_t nch, std::vector<MatSpec> &specs) {
  const TepiLayout L = tepi_layout(nch);
  specs = {MatSpec{L.s_off, nch, L.ldo, L.ldo}, MatSpec{L.x_off, nch, L.ldo, L.ldo},
           MatSpec{L.k_off, nch, L.ldo, L.ldo}, MatSpec{L.tg_off, TG, TG, TG},
           MatSpec{L.tt_off, NB, L.ldo, L.ldo}};
}

cudaError_t launch_tepi(const double *K, int64_t ldk, int64_t kstride, int64_t nch, int64_t ne,
                        const int32_t *n_open, double *T2, const int64_t *t2_slot, double *rowsum,
                        const LevelSums &lv, const PhotoArgs &pa, double *ws, int64_t ws_slot,
                        const CUtensorMap *views, int64_t ws_slots, int32_t *status, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t ce = cudaFuncSetAttribute(tepi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(sizeof(TepiSmem)));
    if (ce != cudaSuccess) return ce;
    attr = true;
  }
  const int grid = static_cast<int>(ne < ws_slots ? ne : ws_slots);
  tepi_kernel<<<grid, NT, sizeof(TepiSmem), st>>>(K, ldk, kstride, static_cast<int>(nch), ne, n_open,
                                                  T2, t2_slot, rowsum, lv, pa, ws, ws_slot, views, status);
  return cudaGetLastError();
}

}  // namespace rmx
