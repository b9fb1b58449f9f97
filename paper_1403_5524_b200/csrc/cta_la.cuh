// cta_la.cuh - CTA-level dense FP64 linear algebra on one matrix in global memory, used by the
// per-energy matching (LU) and T-epilogue (Cholesky) kernels. Every routine is executed by all NT
// threads of one CTA; there is no inter-CTA communication (one CTA owns one energy, SURVEY.md
// §8(a) S4/S5 and BASELINE.json:5 "one CTA ... per energy").
//
//   gemm      : C op= A.B over a tile loop, 128x64 CTA tiles, FP64 DMMA (mma.m8n8k4.f64) with a
//               2-stage cp.async pipeline; A stored [M][K] or [K][M], B stored [N][K] or [K][N]
//   panel_lu  : unblocked LU with partial pivoting of an n x bw panel (pivot = max |a|, ties ->
//               lowest row, the oracle's rule), rank-1 updates fused with the next pivot search
//   trsm_*    : small (bw <= 32) triangular solves, one thread per column / row
//   chol_diag : unblocked Cholesky of a bw x bw diagonal block in shared memory
#pragma once
#include "rmx_common.cuh"

namespace rmx {
namespace la {

constexpr int NT = 256;  // threads per CTA
constexpr int NW = NT / 32;
constexpr int BM = 128, BN = 64, BK = 16, WM = 4, WN = 2;
constexpr int WTM = BM / WM, WTN = BN / WN;  // 32 x 32 warp tile
constexpr int MI = WTM / 8, NI = WTN / 8;    // 4 x 4 DMMA fragments
constexpr int PB = 32;                        // inner panel / triangle width of the factorizations
constexpr int NB = 2 * PB;                    // outer block width (K of the big trailing GEMMs)
constexpr int A_ELEMS = (BM * (BK + 4) > BK * (BM + 4)) ? BM * (BK + 4) : BK * (BM + 4);
constexpr int B_ELEMS = (BN * (BK + 4) > BK * (BN + 4)) ? BN * (BK + 4) : BK * (BN + 4);
constexpr int CS_LD = BN + 8;  // C tile pitch in smem: conflict-free 16-byte fragment reads
constexpr int C_ELEMS = BM * CS_LD;
constexpr int GEMM_SMEM_DOUBLES = 2 * (A_ELEMS + B_ELEMS) + C_ELEMS;
constexpr int TRI_LD = PB + 1;                // padded pitch of a bw x bw triangle in smem
constexpr int TRI_SMEM_DOUBLES = PB * TRI_LD;

__device__ __forceinline__ int cdiv(int a, int b) { return (a + b - 1) / b; }

// ------------------------------------------------------------------------------------------------
// cp.async staging of one BK-slice of an operand tile
//   KC  : global element (r, k) at G[r*ld + k]  -> smem [ROWS][BK+4]
//   !KC : global element (r, k) at G[k*ld + r]  -> smem [BK][ROWS+4]
// rows >= R or k >= K are zero-filled. al16: ld even and G 16-byte aligned.
template <bool KC, int ROWS>
__device__ __forceinline__ void stage_operand(double *s, const double *G, int64_t ld, int r0,
                                              int k0, int R, int K, bool al16) {
  const uint32_t sb = smem_u32(s);
  if (KC) {
    constexpr int CPR = BK / 2;  // 16-byte chunks per row
    for (int q = threadIdx.x; q < ROWS * CPR; q += NT) {
      const int r = q / CPR, kc = (q % CPR) * 2;
      const int gr = r0 + r, gk = k0 + kc;
      int nv = (gr < R) ? K - gk : 0;
      nv = nv < 0 ? 0 : (nv > 2 ? 2 : nv);
      const double *src = nv ? G + static_cast<int64_t>(gr) * ld + gk : G;
      const uint32_t dst = sb + (r * (BK + 4) + kc) * 8;
      if (al16) {
        cp_async16(dst, src, nv * 8);
      } else {
        cp_async8(dst, src, nv > 0 ? 8 : 0);
        cp_async8(dst + 8, nv > 1 ? src + 1 : G, nv > 1 ? 8 : 0);
      }
    }
  } else {
    constexpr int CPR = ROWS / 2;
    for (int q = threadIdx.x; q < BK * CPR; q += NT) {
      const int kk = q / CPR, rc = (q % CPR) * 2;
      const int gk = k0 + kk, gr = r0 + rc;
      int nv = (gk < K) ? R - gr : 0;
      nv = nv < 0 ? 0 : (nv > 2 ? 2 : nv);
      const double *src = nv ? G + static_cast<int64_t>(gk) * ld + gr : G;
      const uint32_t dst = sb + (kk * (ROWS + 4) + rc) * 8;
      if (al16) {
        cp_async16(dst, src, nv * 8);
      } else {
        cp_async8(dst, src, nv > 0 ? 8 : 0);
        cp_async8(dst + 8, nv > 1 ? src + 1 : G, nv > 1 ? 8 : 0);
      }
    }
  }
}

// Epilogues. kReadC: the accumulator starts from C (staged into shared memory by bulk async
// copies, one tile ahead of its use); init() maps a C value to the initial accumulator and store2
// writes the final pair (col, col+1) with the valid masks v0/v1 (r < M && c < N).
struct EpiSub {  // C -= A.B   (acc = -C ; acc += A.B ; C = -acc : exact sign flips)
  static constexpr bool kReadC = true;
  double *C;
  int64_t ldc;
  __device__ __forceinline__ double init(double c) const { return -c; }
  __device__ __forceinline__ void store2(int r, int c, bool v0, bool v1, double a0, double a1) const {
    double *p = C + static_cast<int64_t>(r) * ldc + c;
    if (v0) p[0] = -a0;
    if (v1) p[1] = -a1;
  }
};

struct EpiStore {  // C = A.B + diag_add * I
  static constexpr bool kReadC = false;
  double *C;
  int64_t ldc;
  double diag_add;
  __device__ __forceinline__ double init(double) const { return 0.0; }
  __device__ __forceinline__ void store2(int r, int c, bool v0, bool v1, double a0, double a1) const {
    double *p = C + static_cast<int64_t>(r) * ldc + c;
    if (v0) p[0] = a0 + (r == c ? diag_add : 0.0);
    if (v1) p[1] = a1 + (r == c + 1 ? diag_add : 0.0);
  }
};

// Per-kernel shared state of the C-tile bulk-copy pipeline (one mbarrier, phase carried across calls).
struct GemmSync {
  uint64_t cbar;
  uint32_t cphase;
  uint32_t pad;
};
__device__ __forceinline__ void gemm_sync_init(GemmSync *gs) {
  if (threadIdx.x == 0) {
    mbar_init(&gs->cbar, 1);
    gs->cphase = 0;
    fence_barrier_init();
  }
  __syncthreads();
}

// Tile enumeration (row-major over tm); lower = only tiles holding some element with row >= col.
__device__ __forceinline__ int tiles_in_row(int tm, int tiles_n, bool lower) {
  if (!lower) return tiles_n;
  const int last_col_tile = (tm * BM + BM - 1) / BN;
  return min(tiles_n, last_col_tile + 1);
}

// Warp 0: bulk-copy the valid rows of C tile (tm, tn) into Cs (pitch CS_LD), completion on cbar.
// Rows are copied as whole 16-byte chunks (may read <= 8 bytes past the last column: workspaces are
// padded for this).
__device__ __forceinline__ void issue_c_tile(const double *C, int64_t ldc, int M, int N, int tm,
                                             int tn, double *Cs, uint64_t *cbar) {
  const int lane = lane_id();
  const int r0 = tm * BM, c0 = tn * BN;
  const int rows = min(BM, M - r0), cols = min(BN, N - c0);
  const uint32_t rb = static_cast<uint32_t>((cols * 8 + 15) & ~15);
  if (lane == 0) mbar_arrive_expect_tx(cbar, rb * static_cast<uint32_t>(rows));
  __syncwarp();
  for (int r = lane; r < rows; r += 32)
    bulk_g2s(smem_u32(Cs + r * CS_LD), C + static_cast<int64_t>(r0 + r) * ldc + c0, rb, cbar);
}

// C[M x N] op= A[M x K] . B[K x N] on the calling CTA. smem: GEMM_SMEM_DOUBLES doubles (A/B
// double buffer for cp.async, plus the C tile buffer). Begins and ends with __syncthreads().
// Pipeline: A/B k-slices (BK) double-buffered with cp.async groups; the next tile's C is fetched by
// cp.async.bulk into Cs as soon as the current tile's accumulators have been initialised from it,
// so its latency overlaps a whole tile of DMMA work.
template <bool A_KC, bool B_KC, class Epi>
__device__ __noinline__ void gemm(int M, int N, int K, const double *A, int64_t lda, const double *B,
                                  int64_t ldb, bool lower, double *smem, GemmSync *gs,
                                  const Epi &epi) {
  __syncthreads();
  if (M <= 0 || N <= 0) return;
  const int tiles_m = cdiv(M, BM), tiles_n = cdiv(N, BN);
  const int nkc = K > 0 ? cdiv(K, BK) : 1;
  int ntiles = 0;
  for (int tm = 0; tm < tiles_m; ++tm) ntiles += tiles_in_row(tm, tiles_n, lower);
  const int total = ntiles * nkc;
  const bool al16 = ((lda | ldb) & 1) == 0 &&
                    ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0;
  bool bulk_c = false;
  if constexpr (Epi::kReadC)
    bulk_c = (epi.ldc & 1) == 0 && (reinterpret_cast<uintptr_t>(epi.C) & 15) == 0;
  double *As[2] = {smem, smem + A_ELEMS};
  double *Bs[2] = {smem + 2 * A_ELEMS, smem + 2 * A_ELEMS + B_ELEMS};
  double *Cs = smem + 2 * (A_ELEMS + B_ELEMS);
  uint32_t ph = gs->cphase;

  const int warp = warp_id(), lane = lane_id();
  const int wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, t = lane & 3;

  auto decode_tile = [&](int tile, int &tm, int &tn) {
    tm = 0;
    int cnt;
    while (tile >= (cnt = tiles_in_row(tm, tiles_n, lower))) {
      tile -= cnt;
      ++tm;
    }
    tn = tile;
  };
  auto issue_ab = [&](int it) {
    int tm, tn;
    decode_tile(it / nkc, tm, tn);
    const int kc = it % nkc, buf = it & 1;
    stage_operand<A_KC, BM>(As[buf], A, lda, tm * BM, kc * BK, M, K, al16);
    stage_operand<B_KC, BN>(Bs[buf], B, ldb, tn * BN, kc * BK, N, K, al16);
    cp_async_commit();
  };

  if (bulk_c && warp == 0) {
    int tm, tn;
    decode_tile(0, tm, tn);
    issue_c_tile(epi.C, epi.ldc, M, N, tm, tn, Cs, &gs->cbar);
  }
  issue_ab(0);
  double acc[MI][NI][2];
  for (int it = 0; it < total; ++it) {
    const int tile = it / nkc, kc = it % nkc;
    int tm, tn;
    decode_tile(tile, tm, tn);
    if (it + 1 < total) issue_ab(it + 1);
    if (kc == 0) {
      if (bulk_c) {
        mbar_wait(&gs->cbar, ph);
        ph ^= 1;
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const int rl = wm * WTM + mi * 8 + g;
        const int r = tm * BM + rl;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const int cl = wn * WTN + ni * 8 + 2 * t;
          const int c = tn * BN + cl;
          double c0v = 0.0, c1v = 0.0;
          if constexpr (Epi::kReadC) {
            if (bulk_c) {
              c0v = Cs[rl * CS_LD + cl];
              c1v = Cs[rl * CS_LD + cl + 1];
            } else {
              const double *p = epi.C + static_cast<int64_t>(r) * epi.ldc + c;
              if (r < M && c < N) c0v = p[0];
              if (r < M && c + 1 < N) c1v = p[1];
            }
          }
          acc[mi][ni][0] = epi.init(c0v);
          acc[mi][ni][1] = epi.init(c1v);
        }
      }
    }
    if (it + 1 < total)
      cp_async_wait<1>();
    else
      cp_async_wait<0>();
    __syncthreads();
    if (kc == 0 && bulk_c && tile + 1 < ntiles && warp == 0) {
      int tm2, tn2;
      decode_tile(tile + 1, tm2, tn2);
      fence_proxy_async();
      issue_c_tile(epi.C, epi.ldc, M, N, tm2, tn2, Cs, &gs->cbar);
    }
    if (K > 0) {
      const double *as = As[it & 1], *bs = Bs[it & 1];
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        const int k = ks * 4 + t;
        double a[MI], b[NI];
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          const int m = wm * WTM + mi * 8 + g;
          a[mi] = A_KC ? as[m * (BK + 4) + k] : as[k * (BM + 4) + m];
        }
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const int n = wn * WTN + ni * 8 + g;
          b[ni] = B_KC ? bs[n * (BK + 4) + k] : bs[k * (BN + 4) + n];
        }
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi], b[ni]);
      }
    }
    __syncthreads();
    if (kc == nkc - 1) {
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const int r = tm * BM + wm * WTM + mi * 8 + g;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const int c = tn * BN + wn * WTN + ni * 8 + 2 * t;
          epi.store2(r, c, r < M && c < N, r < M && c + 1 < N, acc[mi][ni][0], acc[mi][ni][1]);
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) gs->cphase = ph;
}

// ------------------------------------------------------------------------------------------------
// Block-wide argmax of |value| with ties -> lowest index. red: smem [2*NW] scratch.
__device__ __forceinline__ void block_argmax(double &v, int &idx, double *redv, int *redi) {
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
  const int warp = warp_id(), lane = lane_id();
  __syncthreads();
  if (lane == 0) {
    redv[warp] = v;
    redi[warp] = idx;
  }
  __syncthreads();
  v = redv[0];
  idx = redi[0];
  for (int w = 1; w < NW; ++w) {
    const double ov = redv[w];
    const int oi = redi[w];
    if (ov > v || (ov == v && oi < idx)) {
      v = ov;
      idx = oi;
    }
  }
}

// LU with partial pivoting of the panel M[p0:n, p0:p0+bw] (bw <= 32), in place: multipliers
// below the diagonal, U on and above. Each interchange swaps the two rows over the columns
// [sc0, sc1) (the whole augmented row right of the current outer block, so the trailing matrix,
// the right-hand sides and the outer block's earlier multipliers stay consistent); the pivot rows
// are also recorded in ipiv[0..bw). Returns 1 on an exact zero pivot. The rank-1 update of column
// j is fused with the pivot search of column j+1 (one pass over the rows per column).
// Pivot rule: max |a_ij|, ties -> lowest row (the oracle's rule).
static __device__ __noinline__ int panel_lu(double *M, int64_t ld, int n, int p0, int bw, int sc0,
                                            int sc1, int *ipiv, double *redv, int *redi) {
  const int warp = warp_id(), lane = lane_id();
  int singular = 0;
  double best = -1.0;
  int besti = n;
  for (int i = p0 + threadIdx.x; i < n; i += NT) {
    const double v = fabs(M[static_cast<int64_t>(i) * ld + p0]);
    if (v > best) {
      best = v;
      besti = i;
    }
  }
  block_argmax(best, besti, redv, redi);
  for (int jj = 0; jj < bw; ++jj) {
    const int j = p0 + jj;
    const int pr = besti < n ? besti : j;  // all-NaN column (e.g. a pole energy): no interchange
    if (pr != j) {
      double *a = M + static_cast<int64_t>(j) * ld;
      double *b = M + static_cast<int64_t>(pr) * ld;
      constexpr int SU = 4;
      for (int c0 = sc0 + threadIdx.x; c0 < sc1; c0 += NT * SU) {
        double va[SU], vb[SU];
#pragma unroll
        for (int q = 0; q < SU; ++q) {
          const int c = c0 + q * NT;
          if (c < sc1) {
            va[q] = a[c];
            vb[q] = b[c];
          }
        }
#pragma unroll
        for (int q = 0; q < SU; ++q) {
          const int c = c0 + q * NT;
          if (c < sc1) {
            a[c] = vb[q];
            b[c] = va[q];
          }
        }
      }
    }
    if (threadIdx.x == 0) ipiv[jj] = pr;
    __syncthreads();
    const double u = lane < bw ? M[static_cast<int64_t>(j) * ld + p0 + lane] : 0.0;
    const double piv = __shfl_sync(0xffffffffu, u, jj);
    const bool zero = (piv == 0.0);
    singular |= zero;
    const double rpiv = zero ? 0.0 : 1.0 / piv;
    best = -1.0;
    besti = n;
    const bool track = (jj + 1 < bw);
    // rows j+1 .. n-1, warp-strided, UNR rows in flight per warp
    constexpr int UNR = 8;
    for (int i0 = j + 1 + warp; i0 < n; i0 += NW * UNR) {
      double x[UNR];
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const int i = i0 + q * NW;
        x[q] = (i < n && lane < bw) ? M[static_cast<int64_t>(i) * ld + p0 + lane] : 0.0;
      }
#pragma unroll
      for (int q = 0; q < UNR; ++q) {
        const int i = i0 + q * NW;
        const double xj = __shfl_sync(0xffffffffu, x[q], jj);
        const double l = xj * rpiv;
        double y = x[q];
        if (lane == jj)
          y = zero ? xj : l;
        else if (lane > jj)
          y = fma(-l, u, y);
        if (i < n && lane >= jj && lane < bw) M[static_cast<int64_t>(i) * ld + p0 + lane] = y;
        if (track) {
          const double v = fabs(__shfl_sync(0xffffffffu, y, jj + 1));
          if (i < n && v > best) {
            best = v;
            besti = i;
          }
        }
      }
    }
    if (track) block_argmax(best, besti, redv, redi);
    __syncthreads();
  }
  return singular;
}

// U12 = L11^{-1} A12 for the rows [p0, p0+bw) and columns [c0, c1), L11 = unit lower part of
// M[p0:p0+bw, p0:p0+bw] (bw <= 32). One thread per column.
static __device__ __noinline__ void trsm_unit_lower_cols(double *M, int64_t ld, int p0, int bw,
                                                         int c0, int c1, double *tri) {
  for (int q = threadIdx.x; q < PB * PB; q += NT) {
    const int r = q / PB, c = q % PB;
    tri[r * TRI_LD + c] = (r < bw && c < r) ? M[static_cast<int64_t>(p0 + r) * ld + p0 + c] : 0.0;
  }
  __syncthreads();
  for (int c = c0 + threadIdx.x; c < c1; c += NT) {
    double x[PB];
#pragma unroll
    for (int r = 0; r < PB; ++r) x[r] = r < bw ? M[static_cast<int64_t>(p0 + r) * ld + c] : 0.0;
#pragma unroll
    for (int r = 1; r < PB; ++r) {
      double s = x[r];
#pragma unroll
      for (int q = 0; q < r; ++q) s = fma(-tri[r * TRI_LD + q], x[q], s);
      x[r] = s;
    }
#pragma unroll
    for (int r = 0; r < PB; ++r)
      if (r < bw) M[static_cast<int64_t>(p0 + r) * ld + c] = x[r];
  }
  __syncthreads();
}

// X[p0:p0+bw, c0:c1) = U^{-1} X for the upper-triangular (non-unit) U = M[p0:p0+bw, p0:p0+bw];
// X lives at Xb + r*ldx + c (row r relative to p0 in the same row numbering). Thread per column.
static __device__ __noinline__ void trsm_upper_cols(const double *M, int64_t ld, int p0, int bw, double *Xb,
                                int64_t ldx, int ncols, double *tri) {
  for (int q = threadIdx.x; q < bw * bw; q += NT) {
    const int r = q / bw, c = q % bw;
    tri[r * TRI_LD + c] = M[static_cast<int64_t>(p0 + r) * ld + p0 + c];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ncols; c += NT) {
    double x[PB];
#pragma unroll
    for (int r = 0; r < PB; ++r) x[r] = r < bw ? Xb[static_cast<int64_t>(p0 + r) * ldx + c] : 0.0;
#pragma unroll
    for (int r = PB - 1; r >= 0; --r) {
      if (r < bw) {
        double s = x[r];
#pragma unroll
        for (int q = r + 1; q < PB; ++q)
          if (q < bw) s = fma(-tri[r * TRI_LD + q], x[q], s);
        x[r] = s / tri[r * TRI_LD + r];
      }
    }
#pragma unroll
    for (int r = 0; r < PB; ++r)
      if (r < bw) Xb[static_cast<int64_t>(p0 + r) * ldx + c] = x[r];
  }
  __syncthreads();
}

// Lower triangle L = S[p0:p0+bw, p0:p0+bw] -> tri (full bw x bw, upper part zero).
__device__ __forceinline__ void load_lower_tri(const double *S, int64_t ld, int p0, int bw,
                                               double *tri) {
  for (int q = threadIdx.x; q < bw * bw; q += NT) {
    const int r = q / bw, c = q % bw;
    tri[r * TRI_LD + c] = c <= r ? S[static_cast<int64_t>(p0 + r) * ld + p0 + c] : 0.0;
  }
  __syncthreads();
}

// X[p0:p0+bw, :] = L^{-1} X  (L lower non-unit in tri). Thread per column.
static __device__ __noinline__ void trsm_lower_cols(const double *tri, int bw, double *X, int64_t ldx, int p0,
                                int ncols) {
  for (int c = threadIdx.x; c < ncols; c += NT) {
    double x[PB];
#pragma unroll
    for (int r = 0; r < PB; ++r) x[r] = r < bw ? X[static_cast<int64_t>(p0 + r) * ldx + c] : 0.0;
#pragma unroll
    for (int r = 0; r < PB; ++r) {
      if (r < bw) {
        double s = x[r];
#pragma unroll
        for (int q = 0; q < r; ++q) s = fma(-tri[r * TRI_LD + q], x[q], s);
        x[r] = s / tri[r * TRI_LD + r];
      }
    }
#pragma unroll
    for (int r = 0; r < PB; ++r)
      if (r < bw) X[static_cast<int64_t>(p0 + r) * ldx + c] = x[r];
  }
  __syncthreads();
}

// X[p0:p0+bw, :] = L^{-T} X  (L lower non-unit in tri). Thread per column.
static __device__ __noinline__ void trsm_lower_t_cols(const double *tri, int bw, double *X, int64_t ldx, int p0,
                                  int ncols) {
  for (int c = threadIdx.x; c < ncols; c += NT) {
    double x[PB];
#pragma unroll
    for (int r = 0; r < PB; ++r) x[r] = r < bw ? X[static_cast<int64_t>(p0 + r) * ldx + c] : 0.0;
#pragma unroll
    for (int r = PB - 1; r >= 0; --r) {
      if (r < bw) {
        double s = x[r];
#pragma unroll
        for (int q = r + 1; q < PB; ++q)
          if (q < bw) s = fma(-tri[q * TRI_LD + r], x[q], s);
        x[r] = s / tri[r * TRI_LD + r];
      }
    }
#pragma unroll
    for (int r = 0; r < PB; ++r)
      if (r < bw) X[static_cast<int64_t>(p0 + r) * ldx + c] = x[r];
  }
  __syncthreads();
}

// Rows [r0, r1) of the panel S[:, p0:p0+bw]: L21 = S21 L11^{-T} (L11 lower in tri). Thread per row.
static __device__ __noinline__ void trsm_rows_lt(const double *tri, int bw, double *S, int64_t ld, int p0, int r0,
                             int r1) {
  for (int r = r0 + threadIdx.x; r < r1; r += NT) {
    double *row = S + static_cast<int64_t>(r) * ld + p0;
    double x[PB];
#pragma unroll
    for (int c = 0; c < PB; ++c) x[c] = c < bw ? row[c] : 0.0;
#pragma unroll
    for (int c = 0; c < PB; ++c) {
      if (c < bw) {
        double s = x[c];
#pragma unroll
        for (int q = 0; q < c; ++q) s = fma(-x[q], tri[c * TRI_LD + q], s);
        x[c] = s / tri[c * TRI_LD + c];
      }
    }
#pragma unroll
    for (int c = 0; c < PB; ++c)
      if (c < bw) row[c] = x[c];
  }
  __syncthreads();
}

// Unblocked Cholesky of S[p0:p0+bw, p0:p0+bw] (lower) in tri, written back to S.
// Returns 1 if a non-positive pivot appears (S is SPD by construction: I + K K^T).
static __device__ __noinline__ int chol_diag(double *S, int64_t ld, int p0, int bw, double *tri) {
  load_lower_tri(S, ld, p0, bw, tri);
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  if (warp_id() == 0) {
    const int lane = lane_id();
    for (int c = 0; c < bw; ++c) {
      // lane r (r >= c) holds column c of row r
      double d = tri[c * TRI_LD + c];
      if (lane == 0 && !(d > 0.0)) bad = 1;
      d = sqrt(d);
      __syncwarp();
      if (lane >= c && lane < bw) {
        const double v = (lane == c) ? d : tri[lane * TRI_LD + c] / d;
        tri[lane * TRI_LD + c] = v;
      }
      __syncwarp();
      if (lane > c && lane < bw) {
        const double lr = tri[lane * TRI_LD + c];
        for (int q = c + 1; q <= lane; ++q) tri[lane * TRI_LD + q] = fma(-lr, tri[q * TRI_LD + c], tri[lane * TRI_LD + q]);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < bw * bw; q += NT) {
    const int r = q / bw, c = q % bw;
    if (c <= r) S[static_cast<int64_t>(p0 + r) * ld + p0 + c] = tri[r * TRI_LD + c];
  }
  __syncthreads();
  return bad;
}

}  // namespace la
}  // namespace rmx
