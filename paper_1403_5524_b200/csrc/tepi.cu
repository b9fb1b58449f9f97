// tepi.cu - S5 of the sweep: T = 2i K_oo (I - i K_oo)^{-1} and |T_ij|^2 (BASELINE.json:5).
//
// Route (reading T2). With A = I - iK_oo (complex symmetric, K_oo real symmetric by
// reading M1), iK = I - A, so 2iK A^{-1} = 2(I - A) A^{-1} = 2(A^{-1} - I):
//   T = 2 (A^{-1} - I),   |T_ij|^2 = 4 |(A^{-1})_ij - delta_ij|^2,
// and only the inverse of A is needed. A's Hermitian part is I, so A has an LDL^T factorisation
// without pivoting whose pivots satisfy Re d_j >= 1 (Schur complements of a matrix with Hermitian
// part >= I keep Hermitian part >= I); the forward error of A^{-1} then grows like u ||K||, as for the
// oracle's pivoted complex elimination - unlike the real SPD route through I + K^2 of round 1,
// whose error grew like u ||K||^2 (1.5e-7 in |T|^2 at darc mesh 50169).
//
// Per energy (one CTA, persistent over energies, workspace slot = blockIdx.x); complex matrices are
// two real planes (re, im) and every complex product is two real DMMA GEMMs whose k range covers
// both halves (GemmArgs::nseg = 2):
//   0. Ar = I, Ai = -K_oo
//   1. blocked right-looking LDL^T, outer blocks of 256 made of 64-wide sub-blocks: each 64 x 64
//      diagonal block is factored in shared memory together with the inverse of its unit-lower
//      factor, Tinv_b = L_bb^{-1} (written over the block, D to a vector); W21 = A21 Tinv_b^T
//      (= L21 D_b), L21 = W21 D_b^{-1}; the outer block's later columns are updated inside the
//      panel, and the trailing matrix once per 256 columns, A22 -= W21 L21^T (lower tiles, K = 256)
//   2. Z = L^{-1} in place, 128-row block rows: the 128 x 128 diagonal inverse from the two 64
//      inverses, Z_{B,0:B} = -Tinv_B (L_{B,0:B} Z_{0:B,0:B})
//   3. Y = D^{-1} Z
//   4. A^{-1} = Z^T Y (lower tiles; Re into the P plane, Im in place over Y_i)
//   5. mirror, |T_ij|^2 = 4 (Im^2 + (delta_ij - Re)^2), row sums in a fixed order (deterministic)
// Executed flops ~ 4 o^3 (SURVEY §8(d) counts (16/3) o^3 as algorithmic).
// |T|^2 and the row sums are invariant under K -> -K (A -> conj(A)).
#include "cta_cgemm.cuh"
#include "rmx_internal.h"
#include <cstdlib>

namespace rmx {

using namespace la;

#ifdef RMX_PHASES
// per-phase clock64 totals of block 0 (diagnostic build: python -m paper_1403_5524_b200.build --phases)
__device__ unsigned long long g_tepi_phase[8];
#define TPH_MARK(k)                                                         \
  do {                                                                      \
    __syncthreads();                                                        \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                              \
      const unsigned long long now_ = clock64();                            \
      g_tepi_phase[k] += now_ - ph_t0;                                      \
      ph_t0 = now_;                                                         \
    }                                                                       \
  } while (0)
#else
#define TPH_MARK(k) \
  do {              \
  } while (0)
#endif

constexpr int CB = 64;          // block width of the complex LDL^T
constexpr int CB_LD = CB + 1;   // smem pitch of the diagonal block

struct TepiSmem {
  union {  // the diagonal-block scratch is only used between gemm calls
    double gemm[GEMM_SMEM_DOUBLES];
    double tri[2 * CB * CB_LD + 6 * CB];
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

// |T|^2 = 4 (Im^2 + (delta - Re)^2) and the row sums straight from the LOWER triangles of Re A^{-1} (P)
// and Im A^{-1} (X), 32 x 32 tiles staged through shared memory (the mirror passes are not needed):
// tile (bi, bj), bi >= bj, yields |T|^2 of its own elements and of the mirrored tile (bj, bi) (on a
// diagonal tile the upper half is filled from the lower one: bitwise symmetric |T|^2), its row sums
// go to part[bj][i] and its column sums to part[bi][j]; then rowsum_i = sum_q part[q][i] in q order
// (fixed order: deterministic). part: nb x o scratch (pitch o). Returns the non-finite flag.
__device__ __noinline__ int tiled_t2(const double *P, const double *X, int64_t ld, int o, int n, double *T2e,
                                     double *rowsum, double *part, double *smem) {
  constexpr int TL = 33;
  const int nb = (o + 31) / 32, lane = lane_id();
  double *tile = smem + warp_id() * 32 * TL;
  int bad = 0;
  __syncthreads();
  for (int b = warp_id(); b < nb * (nb + 1) / 2; b += NW) {
    int bi = 0, rem = b;
    while (rem > bi) {
      rem -= bi + 1;
      ++bi;
    }
    const int bj = rem;
    const bool diag = bi == bj;
    for (int r0 = 0; r0 < 32; r0 += 8) {  // 16 independent loads in flight per lane
      double xv[8], pv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = r0 + u, gi = bi * 32 + r, gj = bj * 32 + lane;
        const bool ok = gi < o && gj < o && (!diag || lane <= r);
        xv[u] = ok ? X[static_cast<int64_t>(gi) * ld + gj] : 0.0;
        pv[u] = ok ? P[static_cast<int64_t>(gi) * ld + gj] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int r = r0 + u, gi = bi * 32 + r, gj = bj * 32 + lane;
        double v = 0.0;
        if (gi < o && gj < o && (!diag || lane <= r)) {
          const double p = (gi == gj ? 1.0 : 0.0) - pv[u];
          v = 4.0 * fma(xv[u], xv[u], p * p);
        }
        tile[r * TL + lane] = v;
      }
    }
    __syncwarp();
    if (diag)
      for (int r = 0; r < 32; ++r)
        if (lane > r) tile[r * TL + lane] = tile[lane * TL + r];  // upper half from the lower one
    __syncwarp();
    // row sums of the tile (lane = row) and of its mirror (lane = column)
    double rs = 0.0, cs = 0.0;
#pragma unroll 8
    for (int q = 0; q < 32; ++q) {
      rs += tile[lane * TL + q];
      cs += tile[q * TL + lane];
    }
    if (!isfinite(rs)) bad = 1;
    const int gi = bi * 32 + lane, gj = bj * 32 + lane;
    if (gi < o) part[static_cast<int64_t>(bj) * o + gi] = rs;
    if (!diag && gj < o) part[static_cast<int64_t>(bi) * o + gj] = cs;
    if (T2e) {
      for (int r = 0; r < 32; ++r) {
        const int ri = bi * 32 + r, cj = bj * 32 + lane;
        if (ri < o && cj < o) T2e[static_cast<int64_t>(ri) * n + cj] = tile[r * TL + lane];
        const int rj = bj * 32 + r, ci = bi * 32 + lane;
        if (!diag && rj < o && ci < o) T2e[static_cast<int64_t>(rj) * n + ci] = tile[lane * TL + r];
      }
    }
    __syncwarp();
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += NT) {
    double s = 0.0;
    if (i < o)
      for (int q = 0; q < nb; ++q) s += part[static_cast<int64_t>(q) * o + i];
    if (rowsum) rowsum[i] = s;
  }
  if (T2e) {  // closed rows / columns: zero
    for (int i = warp_id(); i < n; i += NW)
      for (int j = lane; j < n; j += 32)
        if (i >= o || j >= o) T2e[static_cast<int64_t>(i) * n + j] = 0.0;
  }
  return bad;
}

// LDL^T of the W x W (W <= 64) complex symmetric diagonal block A[p0.., p0..] (lower triangle of
// the planes ar, ai) without pivoting, fused with the inverse of its unit-lower factor: in shared
// memory row r holds X = L^{-1} in columns < c and the not yet eliminated part of A in columns
// >= c, so elimination step c (X <- (I - l_c e_c^T) X, A22 -= l_c w_c^T) is one update of the
// rows below c:  M[r][k] -= l_r u_k with u_k = X[c][k] (k < c) or A[k][c] (k > c), M[r][c] = -l_r.
// On return the block holds Tinv = L^{-1} (unit lower, explicit zeros above the diagonal) and
// d[p0 .. p0+W) the pivots (re, im). All NT threads.
__device__ __noinline__ void diag_ldlt_inv(const MatView &ar, const MatView &ai, int p0, int W,
                                           double *dr_out, double *di_out, double *sm) {
  double *Mr = sm, *Mi = sm + CB * CB_LD;
  double *lr = Mi + CB * CB_LD, *li = lr + CB, *ur = li + CB, *ui = ur + CB;
  __syncthreads();
  for (int q = threadIdx.x; q < W * CB; q += NT) {
    const int r = q / CB, k = q % CB;
    if (k <= r && k < W) {
      Mr[r * CB_LD + k] = *ar.at(p0 + r, p0 + k);
      Mi[r * CB_LD + k] = *ai.at(p0 + r, p0 + k);
    }
  }
  for (int c = 0; c < W; ++c) {
    __syncthreads();
    const double dr = Mr[c * CB_LD + c], di = Mi[c * CB_LD + c];
    const double den = fma(dr, dr, di * di);
    const double ir = dr / den, ii = -di / den;  // 1/d (|d| >= Re d >= 1 in exact arithmetic)
    for (int t = threadIdx.x; t < W; t += NT) {
      if (t > c) {
        const double xr = Mr[t * CB_LD + c], xi = Mi[t * CB_LD + c];
        lr[t] = xr * ir - xi * ii;
        li[t] = fma(xr, ii, xi * ir);
        ur[t] = xr;
        ui[t] = xi;
      } else if (t < c) {
        ur[t] = Mr[c * CB_LD + t];
        ui[t] = Mi[c * CB_LD + t];
      }
    }
    if (threadIdx.x == 0) {
      dr_out[p0 + c] = dr;
      di_out[p0 + c] = di;
    }
    __syncthreads();
    const int nrow = W - c - 1;
    for (int e = threadIdx.x; e < nrow * CB; e += NT) {
      const int r = c + 1 + e / CB, k = e % CB;
      if (k > r) continue;
      const double a = lr[r], b = li[r];
      if (k == c) {
        Mr[r * CB_LD + c] = -a;
        Mi[r * CB_LD + c] = -b;
      } else {
        const double xr = ur[k], xi = ui[k];
        Mr[r * CB_LD + k] = fma(-a, xr, fma(b, xi, Mr[r * CB_LD + k]));
        Mi[r * CB_LD + k] = fma(-a, xi, fma(-b, xr, Mi[r * CB_LD + k]));
      }
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < W * W; q += NT) {
    const int r = q / W, k = q % W;
    *ar.at(p0 + r, p0 + k) = k < r ? Mr[r * CB_LD + k] : (k == r ? 1.0 : 0.0);
    *ai.at(p0 + r, p0 + k) = k < r ? Mi[r * CB_LD + k] : 0.0;
  }
  __syncthreads();
}

// L = W D^{-1}: dst[(dr0 + i, dc0 + j)] = src[(sr0 + i, sc0 + j)] / d_j (complex), i < m, j < w <= 64.
__device__ __forceinline__ void scale_cols(const MatView &sr, const MatView &si, int sr0, int sc0,
                                           const MatView &tr, const MatView &ti, int dr0, int dc0, int m, int w,
                                           const double *dre, const double *dim, double *sm) {
  double *idr = sm, *idi = sm + 64;
  __syncthreads();
  for (int j = threadIdx.x; j < w; j += NT) {
    const double a = dre[j], b = dim[j], den = fma(a, a, b * b);
    idr[j] = a / den;
    idi[j] = -b / den;
  }
  __syncthreads();
  constexpr int U = 8;  // 2U independent loads in flight per thread (the pass is latency-bound)
  for (int q0 = threadIdx.x; q0 < m * 64; q0 += NT * U) {
    double xr[U], xi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = q0 + u * NT, i = q >> 6, j = q & 63;
      const bool ok = q < m * 64 && j < w;
      xr[u] = ok ? *sr.at(sr0 + i, sc0 + j) : 0.0;
      xi[u] = ok ? *si.at(sr0 + i, sc0 + j) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = q0 + u * NT, i = q >> 6, j = q & 63;
      if (q < m * 64 && j < w) {
        *tr.at(dr0 + i, dc0 + j) = xr[u] * idr[j] - xi[u] * idi[j];
        *ti.at(dr0 + i, dc0 + j) = fma(xr[u], idi[j], xi[u] * idr[j]);
      }
    }
  }
}

// Complex product into the planes (cr, ci) at (r0, c0): C = alpha * (A.B) (set) or C -= A.B (sub),
// A = (a_re, a_im), B = (b_re, b_im) given as operand pairs of one layout.
__device__ __forceinline__ void cgemm(int M, int N, int K, const Op &are, const Op &aim, const Op &bre,
                                      const Op &bim, const MatView &cr, const MatView &ci, int r0, int c0,
                                      bool lower, bool sub, double alpha, int kband, double *smem,
                                      GemmSync *gs) {
  // Re = Ar.Br - Ai.Bi
  GemmArgs g{are, bre, cr.at(r0, c0), cr.ld, M, N, K, lower, sub, false, 0.0, kband};
  g.a2 = aim;
  g.b2 = bim;
  g.nseg = 2;
  g.neg2 = true;
  g.alpha = alpha;
  g.c_end = cr.end();
  gemm_rt(g, gemm_smem_align(smem), gs);
  // Im = Ar.Bi + Ai.Br
  g.b = bim;
  g.b2 = bre;
  g.neg2 = false;
  g.C = ci.at(r0, c0);
  g.ldc = ci.ld;
  g.c_end = ci.end();
  gemm_rt(g, gemm_smem_align(smem), gs);
}

// Workspace slot (tepi_layout): planes Ar, Ai (A, then L / Tinv blocks, then Z), Yr, Yi (scratch,
// then Y = D^{-1} Z, then Im A^{-1} in place), P (Re A^{-1}); vectors d (re, im) and v.
__global__ void __launch_bounds__(NT, 1)
    tepi_kernel(const double *K, int64_t ldk, int64_t kstride, int n, int64_t ne,
                const int32_t *__restrict__ n_open, double *T2, const int64_t *t2_slot,
                double *rowsum, LevelSums lv, PhotoArgs pa, double *ws, int64_t ws_slot,
                const CUtensorMap *views, int32_t *status, int c4m) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  TepiSmem &sm = *reinterpret_cast<TepiSmem *>(smem_raw);
  const TepiLayout L = tepi_layout(n);
  const int ldo = static_cast<int>(L.ldo);
  double *slot = ws + static_cast<int64_t>(blockIdx.x) * ws_slot;
  const CUtensorMap *vw = views + blockIdx.x * 5 * NVIEW;
  const MatView Arv{vw + 0 * NVIEW, slot + L.ar_off, ldo, n};
  const MatView Aiv{vw + 1 * NVIEW, slot + L.ai_off, ldo, n};
  const MatView Yrv{vw + 2 * NVIEW, slot + L.yr_off, ldo, n};
  const MatView Yiv{vw + 3 * NVIEW, slot + L.yi_off, ldo, n};
  const MatView Pv{vw + 4 * NVIEW, slot + L.p_off, ldo, n};
  double *dr = slot + L.d_off, *di = dr + n, *vv = di + n;
  double *smg = sm.gemm;
  GemmSync *gs = &sm.gs;
  // complex products: the products that write C (C = alpha A.B) by the 3M single pass
  // (cta_cgemm.cuh); the trailing updates C -= A.B (K = 128 per tile, C read and written per tile) by
  // the 4-product two-pass form of gemm_impl, whose 128 x 64 C tiles are staged through shared memory
  // one tile ahead (3M measured +40 % there with C read in its epilogue, +33 % with staged C).
  // RMX_TEPI_4M: the 4-product form everywhere (A/B switch).
  auto cg = [&](int M, int N, int K, const Op &are, const Op &aim, const Op &bre, const Op &bim,
                const MatView &cr, const MatView &ci, int r0, int c0, bool lower, bool sub, double alpha,
                int kband) {
    if (c4m || sub)
      cgemm(M, N, K, are, aim, bre, bim, cr, ci, r0, c0, lower, sub, alpha, kband, smg, gs);
    else
      cgemm3(M, N, K, are, aim, bre, bim, cr, ci, r0, c0, lower, sub, alpha, kband, smg, gs);
  };

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
#ifdef RMX_PHASES
    unsigned long long ph_t0 = clock64();
#endif
    if (o > 0) {
      if (pa.g) {
        // NEXT-1 (10): v_j = (1/2)(g_j F'_j + sum_i g_i G'_i K_ij) (j < o); gG_i staged in shared
        // memory, i ascending
        const double *ge = pa.g + e * n, *Fpe = pa.Fp + e * n, *Gpe = pa.Gp + e * n;
        double *gG = sm.gemm;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += NT) gG[i] = ge[i] * Gpe[i];
        __syncthreads();
        for (int j = threadIdx.x; j < o; j += NT) {
          double s = ge[j] * Fpe[j];
          for (int i = 0; i < n; ++i) s = fma(gG[i], Ke[static_cast<int64_t>(i) * ldk + j], s);
          vv[j] = 0.5 * s;
        }
      }
      // 0. Ar = I, Ai = -K_oo
      for (int i = warp_id(); i < o; i += NW) {
        const double *src = Ke + static_cast<int64_t>(i) * ldk;
        double *pr = Arv.at(i, 0), *pi = Aiv.at(i, 0);
        constexpr int U = 8;  // 8 independent loads in flight per lane
        for (int j0 = lane_id(); j0 < o; j0 += 32 * U) {
          double v[U];
#pragma unroll
          for (int q = 0; q < U; ++q) v[q] = (j0 + 32 * q < o) ? src[j0 + 32 * q] : 0.0;
#pragma unroll
          for (int q = 0; q < U; ++q) {
            const int j = j0 + 32 * q;
            if (j < o) {
              pi[j] = -v[q];
              pr[j] = (i == j) ? 1.0 : 0.0;
            }
          }
        }
      }
      TPH_MARK(0);  // copy (+ photo v)
      // 1. blocked LDL^T, outer blocks of OB = 256 columns made of 64-wide sub-blocks (diagonal factor
      // + inverse in shared memory each; W21, L21 and the update of the block's remaining columns
      // per sub-block); the trailing matrix is updated once per outer block (K = OB per product)
      constexpr int OB = 4 * CB;
      for (int P0 = 0; P0 < o; P0 += OB) {
        const int W = min(OB, o - P0), m = o - P0 - W;
        // Y scratch row q <-> global row P0 + CB + q; column range of sub-block s: [s*CB, s*CB + ws)
        for (int S = P0; S < P0 + W; S += CB) {
          const int ws = min(CB, P0 + W - S), mb = o - S - ws, yr = S + ws - (P0 + CB), yc = S - P0;
          const int rest = P0 + W - S - ws;  // columns of the outer block right of this sub-block
          diag_ldlt_inv(Arv, Aiv, S, ws, dr, di, sm.tri);
          TPH_MARK(1);  // diagonal blocks
          if (mb == 0) break;
          // W21 = A21 Tinv^T (= L21 D) for all rows below the sub-block
          cg(mb, ws, ws, opk(Arv, S + ws, S), opk(Aiv, S + ws, S), opk(Arv, S, S), opk(Aiv, S, S), Yrv, Yiv,
             yr, yc, false, false, 1.0, 0);
          TPH_MARK(2);  // W21 = A21 Tinv^T
          scale_cols(Yrv, Yiv, yr, yc, Arv, Aiv, S + ws, S, mb, ws, dr + S, di + S, sm.tri);
          TPH_MARK(3);  // L21 scaling
          if (rest > 0) {
            // the outer block's remaining columns: A[S+ws:, S+ws:P0+W] -= W21 L21[0:rest]^T
            cg(mb, rest, ws, opk(Yrv, yr, yc), opk(Yiv, yr, yc), opk(Arv, S + ws, S), opk(Aiv, S + ws, S), Arv,
               Aiv, S + ws, S + ws, false, true, 1.0, 0);
            TPH_MARK(4);
          }
        }
        if (m > 0) {
          // A22 -= [W21 ...] [L21 ...]^T over the whole outer block (lower tiles), K = W per product
          cg(m, m, W, opk(Yrv, W - CB, 0), opk(Yiv, W - CB, 0), opk(Arv, P0 + W, P0), opk(Aiv, P0 + W, P0), Arv,
             Aiv, P0 + W, P0 + W, true, true, 1.0, 0);
          TPH_MARK(4);  // trailing updates
        }
      }
      // 2. Z = L^{-1} in place, 128-row block rows
      for (int R0 = 0; R0 < o; R0 += 2 * CB) {
        const int W = min(2 * CB, o - R0), W2 = W - CB;
        if (W2 > 0) {
          // the upper-right 64-block of the diagonal 128-block is zero in Tinv_128 (the trailing
          // updates of step 1 left values there: their lower tiles overhang the diagonal)
          for (int q = threadIdx.x; q < CB * W2; q += NT) {
            *Arv.at(R0 + q / W2, R0 + CB + q % W2) = 0.0;
            *Aiv.at(R0 + q / W2, R0 + CB + q % W2) = 0.0;
          }
          // Tinv_128 = [[T1, 0], [-T2 L21 T1, T2]]: Q1 = L21 T1 -> Y, then -T2 Q1 over L21
          cg(W2, CB, CB, opk(Arv, R0 + CB, R0), opk(Aiv, R0 + CB, R0), opn(Arv, R0, R0), opn(Aiv, R0, R0),
             Yrv, Yiv, 0, 0, false, false, 1.0, 0);
          cg(W2, CB, W2, opk(Arv, R0 + CB, R0 + CB), opk(Aiv, R0 + CB, R0 + CB), opn(Yrv, 0, 0),
             opn(Yiv, 0, 0), Arv, Aiv, R0 + CB, R0, false, false, -1.0, 0);
        }
        if (R0 > 0) {
          // Tt = L_{B,0:R0} Z_{0:R0,0:R0} -> Y (Z lower triangular: kband 2); Z_B = -Tinv_128 Tt
          cg(W, R0, R0, opk(Arv, R0, 0), opk(Aiv, R0, 0), opn(Arv, 0, 0), opn(Aiv, 0, 0), Yrv, Yiv, 0, 0,
             false, false, 1.0, 2);
          cg(W, R0, W, opk(Arv, R0, R0), opk(Aiv, R0, R0), opn(Yrv, 0, 0), opn(Yiv, 0, 0), Arv, Aiv, R0,
             0, false, false, -1.0, 0);
        }
      }
      TPH_MARK(5);  // Z = L^{-1}
      // 3. Y = D^{-1} Z (zeros above the diagonal); Z's strict upper part inside its 128 x 128
      // diagonal blocks is zeroed too (both are read as explicit zeros by the k-band GEMM below)
      for (int i = warp_id(); i < o; i += NW) {
        const double a = dr[i], b = di[i], den = fma(a, a, b * b);
        const double ir = a / den, ii = -b / den;
        double *zr = Arv.at(i, 0), *zi = Aiv.at(i, 0), *yr = Yrv.at(i, 0), *yi = Yiv.at(i, 0);
        const int zend = min(o, (i / (2 * CB) + 1) * (2 * CB));
        constexpr int U = 8;  // 2U independent loads in flight per lane (the pass is latency-bound)
        for (int j0 = lane_id(); j0 <= i; j0 += 32 * U) {
          double xr[U], xi[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = j0 + 32 * u;
            xr[u] = j <= i ? zr[j] : 0.0;
            xi[u] = j <= i ? zi[j] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int j = j0 + 32 * u;
            if (j <= i) {
              yr[j] = xr[u] * ir - xi[u] * ii;
              yi[j] = fma(xr[u], ii, xi[u] * ir);
            }
          }
        }
        for (int j = i + 1 + lane_id(); j < o; j += 32) {
          yr[j] = 0.0;
          yi[j] = 0.0;
          if (j < zend) {
            zr[j] = 0.0;
            zi[j] = 0.0;
          }
        }
      }
      // 4. A^{-1} = Z^T Y (lower tiles; A(i,k) = Z(k,i) = 0 for k < i: kband 1). Re -> P, then Im
      // in place over Y_i: an output tile is stored after its own reads, and later tiles read only
      // rows >= their first row or other columns (row-major tile order).
      if (c4m) {
        GemmArgs g{opn(Arv, 0, 0), opn(Yrv, 0, 0), Pv.base, Pv.ld, o, o, o, true, false, false, 0.0, 1};
        g.c_end = Pv.end();
        g.a2 = opn(Aiv, 0, 0);
        g.b2 = opn(Yiv, 0, 0);
        g.nseg = 2;
        g.neg2 = true;
        gemm_rt(g, gemm_smem_align(smg), gs);
        g.b = opn(Yiv, 0, 0);
        g.b2 = opn(Yrv, 0, 0);
        g.neg2 = false;
        g.C = Yiv.base;
        g.c_end = Yiv.end();
        gemm_rt(g, gemm_smem_align(smg), gs);
      } else {
        // one pass: Re -> P, Im in place over Y_i (each tile stores after its own reads)
        cgemm3(o, o, o, opn(Arv, 0, 0), opn(Aiv, 0, 0), opn(Yrv, 0, 0), opn(Yiv, 0, 0), Pv, Yiv, 0, 0, true,
               false, 1.0, 1, smg, gs);
      }
      TPH_MARK(6);  // Y = D^{-1} Z and A^{-1} = Z^T Y
      // 5. symmetric A^{-1}: upper triangles from the lower ones - needed only by the NEXT-1 / NEXT-2
      // options, which read whole rows; |T|^2 and the row sums come from the lower triangles alone
      if (pa.g || lv.omega) {
        mirror_lower(Pv.base, ldo, o, sm.gemm);
        mirror_lower(Yiv.base, ldo, o, sm.gemm);
      }
    }
    const bool tiled = !(pa.g || lv.omega) && o > 0;
    if (tiled)  // the Yr plane (free after step 4) holds the partial row sums
      bad |= tiled_t2(Pv.base, Yiv.base, ldo, o, n, T2e, rowsum ? rowsum + e * n : nullptr, Yrv.base, sm.gemm);
    // epilogue: |T|^2 = 4 (Im^2 + (delta - Re)^2), row sums in fixed order
    for (int i = warp_id(); i < (tiled ? 0 : n); i += NW) {
      double s = 0.0;
      const double *xr = Yiv.at(i, 0), *pr = Pv.at(i, 0);
      constexpr int U = 4;  // 2U independent loads in flight per lane
      for (int j0 = lane_id(); j0 < n; j0 += 32 * U) {
        double xv[U], pv[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int j = j0 + 32 * q;
          const bool in = i < o && j < o;
          xv[q] = in ? xr[j] : 0.0;
          pv[q] = in ? (i == j ? 1.0 : 0.0) - pr[j] : 0.0;
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
      // NEXT-1 (11)-(12): M = A^{-1} v = (Re A^{-1}) v + i (Im A^{-1}) v; |M_j|^2; sigma.
      // Row sums in a fixed order: warp w takes rows w, w + NW, ...; warps combined in order.
      double *vs = sm.gemm, *wsum = sm.gemm + n + 1;
      __syncthreads();
      for (int j = threadIdx.x; j < o; j += NT) vs[j] = vv[j];
      __syncthreads();
      double part = 0.0;
      for (int i = warp_id(); i < n; i += NW) {
        double m2 = 0.0;
        if (i < o) {
          const double *pr = Pv.at(i, 0), *xr = Yiv.at(i, 0);
          double tr = 0.0, ti = 0.0;
          for (int j = lane_id(); j < o; j += 32) {
            tr = fma(pr[j], vs[j], tr);
            ti = fma(xr[j], vs[j], ti);
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) {
            tr += __shfl_xor_sync(0xffffffffu, tr, off);
            ti += __shfl_xor_sync(0xffffffffu, ti, off);
          }
          m2 = fma(tr, tr, ti * ti);
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
            const double *xr = Yiv.at(i, 0), *pr = Pv.at(i, 0);
            for (int j = j0; j < j1; ++j) {
              const double p = (i == j ? 1.0 : 0.0) - pr[j];
              acc += 4.0 * fma(xr[j], xr[j], p * p);
            }
          }
          Om[static_cast<int64_t>(la) * lv.nlevel + lb] += lv.g * acc;
        }
      }
    }
    bad = __syncthreads_or(bad);
    if (bad && threadIdx.x == 0) set_status(status, e, RMX_E_NONFINITE);
    TPH_MARK(7);  // mirror + epilogue (+ photo, levels)
  }
}

#ifdef RMX_PHASES
extern "C" int rmx_debug_tepi_phases(unsigned long long *out) {
  cudaDeviceSynchronize();
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_tepi_phase, sizeof(g_tepi_phase)));
}
#endif

#ifdef RMX_CHECKS
// Self-test of the bounds-checked build: an index one row past a 4 x 4 view must trap.
__global__ void checks_selftest_kernel(double *buf, int row) {
  const MatView v{nullptr, buf, 4, 4};
  *v.at(row, 0) = 1.0;
}
extern "C" int rmx_debug_checks_selftest(int row) {
  double *buf = nullptr;
  if (cudaMalloc(&buf, 64 * sizeof(double)) != cudaSuccess) return -1;
  checks_selftest_kernel<<<1, 1>>>(buf, row);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaFree(buf);
  return static_cast<int>(e);
}
#endif

int64_t tepi_ws_doubles_per_slot(int64_t nch) { return tepi_layout(nch).slot; }

// Matrices of one slot whose TMA descriptors the kernel uses: (Ar, Ai, Yr, Yi, P), NVIEW boxes each.
void tepi_view_specs(int64_t nch, std::vector<MatSpec> &specs) {
  const TepiLayout L = tepi_layout(nch);
  specs = {MatSpec{L.ar_off, nch, L.ldo, L.ldo}, MatSpec{L.ai_off, nch, L.ldo, L.ldo},
           MatSpec{L.yr_off, nch, L.ldo, L.ldo}, MatSpec{L.yi_off, nch, L.ldo, L.ldo},
           MatSpec{L.p_off, nch, L.ldo, L.ldo}};
}

cudaError_t launch_tepi(const double *K, int64_t ldk, int64_t kstride, int64_t nch, int64_t ne,
                        const int32_t *n_open, double *T2, const int64_t *t2_slot, double *rowsum,
                        const LevelSums &lv, const PhotoArgs &pa, double *ws, int64_t ws_slot,
                        const CUtensorMap *views, int64_t ws_slots, int32_t *status, cudaStream_t st) {
  cudaError_t ce = ensure_smem_attr(reinterpret_cast<const void *>(tepi_kernel), sizeof(TepiSmem));
  if (ce != cudaSuccess) return ce;
  const int grid = static_cast<int>(ne < ws_slots ? ne : ws_slots);
  static const int c4m = getenv("RMX_TEPI_4M") != nullptr;  // A/B switch: 4-product complex GEMMs
  tepi_kernel<<<grid, NT, sizeof(TepiSmem), st>>>(K, ldk, kstride, static_cast<int>(nch), ne, n_open,
                                                  T2, t2_slot, rowsum, lv, pa, ws, ws_slot, views, status, c4m);
  return cudaGetLastError();
}

}  // namespace rmx
