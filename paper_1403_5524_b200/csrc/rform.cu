// rform.cu - S1+S2 of the sweep: R_ij(E) = (1/2a) sum_k w_ik w_jk / (E_k - E)
// (§6 Eq. 1-2 "R = X x Y" with X_ik = w_ik/(E - E_k), Y = w_kj; written in the
// north_star convention of BASELINE.json:5). B200 design:
//   * one CTA per (energy, upper-triangle tile pair (I <= J)); the grid enumerates energies fastest,
//     so the CTAs resident at any time are (mostly) one tile pair for ~148 energies and stream the
//     same two W slabs through L2 in lock step (W read from HBM about once per wave);
//   * the term of the pole nearest to E is left out of the k loop (d_k* = 0) and added in the
//     epilogue (reading N1);
//   * a producer warp issues 2D TMA loads (SWIZZLE_128B, 16 doubles x BM rows per box) of the W rows of
//     tile I and tile J into a STAGES-deep mbarrier ring, and computes the stage's denominators
//     d_k = 1/(E_k - E) on chip (X of Eq. 2 is never materialised) plus the pole guard;
//   * consumer warps run FP64 tensor-core MMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4, the only FP64
//     MMA on sm_100a; tcgen05 has no f64 kind), scaling the A fragment by d_k in registers;
//   * fragment rows are permuted inside each 8-row group (g -> (g>>1) + 4(g&1)) so that the 16-byte
//     fragment loads from the 128B-swizzled tiles are bank-conflict free;
//   * epilogue scales by 1/2a and stores the tile and its mirror image: R is bitwise symmetric.
#include "rmx_common.cuh"
#include "rmx_internal.h"
#include <cstdlib>

namespace rmx {

template <int BM_, int STAGES_, bool PRODUCER_ = true>
struct RformCfg {
  static constexpr int BM = BM_, STAGES = STAGES_;
  // PRODUCER: a dedicated TMA/denominator warp (9 warps: 3 on one SM sub-partition caps the
  // register file at 168 per thread and the pair mode spills); otherwise the consumer warps refill
  // the ring in turn (8 warps, up to 255 registers, no spills).
  static constexpr bool PRODUCER = PRODUCER_;
  static constexpr int BK = 32;    // k per pipeline stage
  static constexpr int BOXK = 16;  // doubles per TMA box row (128 B = swizzle span)
  static constexpr int NB = BM / 32;                       // 32 x 32 blocks per tile dimension
  static constexpr int NCW = (NB * NB / 2 > 4) ? NB * NB / 2 : 4;  // consumer warps, <= 2 blocks each
  static constexpr int NT = (NCW + (PRODUCER ? 1 : 0)) * 32;
  static constexpr int BOX_BYTES = BM * BOXK * 8;
  static constexpr int OP_BYTES = 2 * BOX_BYTES;   // one operand, one stage
  static constexpr int STAGE_BYTES = 2 * OP_BYTES;  // tile I + tile J
  static constexpr int SMEM_BYTES =
      1024 + STAGES * STAGE_BYTES + STAGES * BK * 8 + 2 * STAGES * 8 + 16;
  static_assert(BOX_BYTES % 1024 == 0, "swizzle-128B boxes must stay 1024-byte aligned");
  static_assert(NB * NB <= 2 * NCW, "at most two 32x32 blocks per consumer warp");
};

__device__ __forceinline__ int frag_row_perm(int g) { return (g >> 1) + 4 * (g & 1); }

// Decode upper-triangle tile pair index -> (ti, tj), ti <= tj, row-major over ti.
__device__ __forceinline__ void decode_pair(int p, int ntiles, int &ti, int &tj) {
  ti = 0;
  while (p >= ntiles - ti) {
    p -= ntiles - ti;
    ++ti;
  }
  tj = ti + p;
}

// Work split inside a tile: the useful 32x32 blocks (inside nch, and c >= r on a diagonal tile) of
// each block row are cut into chunks of two adjacent blocks (one 32 x 64 warp tile, A fragments
// shared) plus a single block when the row count is odd. Chunks are listed pairs first, then
// singles, and dealt snake-wise to the four SM sub-partitions (warp w runs on sub-partition w % 4):
// chunk i -> warp i for i < 4, warp 11 - i for i >= 4. A full tile (8 pairs) keeps the plain 4 x 2
// warp grid; a diagonal tile (4 pairs + 2 singles) or a ragged edge tile costs the largest
// sub-partition load (3 of 4 blocks) instead of a full tile. With NCW == 4 (64-row tiles) every
// chunk is a single block. Returns the number of blocks (0, 1, 2) of this warp's chunk at (r, c).
template <int NB, int NCW>
__device__ __forceinline__ int rform_chunk(int warp, int rbm, int cbm, bool diag, int &r, int &c) {
  constexpr bool PAIRS = NCW >= 8;
  const int want = PAIRS ? ((warp < 4) ? warp : 11 - warp) : warp;
  int idx = 0;
  r = c = 0;
  if (PAIRS) {
    for (int rr = 0; rr < rbm; ++rr)
      for (int cc = diag ? rr : 0; cc + 1 < cbm; cc += 2, ++idx)
        if (idx == want) { r = rr; c = cc; return 2; }
  }
  for (int rr = 0; rr < rbm; ++rr) {
    const int c0 = diag ? rr : 0;
    for (int cc = PAIRS ? (((cbm - c0) & 1) ? cbm - 1 : cbm) : c0; cc < cbm; ++cc, ++idx)
      if (idx == want) { r = rr; c = cc; return 1; }
  }
  return 0;
}

// One k-slab of DMMA for a warp owning block(s) of 32x32.
//   MODE 0: two adjacent blocks of one block row (A fragments shared, 4 x 8 fragments, 64 DMMA / kk)
//   MODE 2: one block (4 x 4 fragments, 32 DMMA / kk)
template <int MODE>
__device__ __forceinline__ void rform_slab(double (&acc)[2][4][4][2], uint32_t abase, uint32_t bbase,
                                           uint32_t dbase, int box_bytes, const uint32_t (&arow)[2],
                                           const uint32_t (&brow)[2], int t, int prow) {
#pragma unroll
  for (int kb = 0; kb < 2; ++kb) {
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      // this lane's two k values: k = kb*16 + kk*8 + 2t + {0,1}; 16-byte chunk c = kk*4 + t
      const uint32_t chunk = static_cast<uint32_t>(((kk * 4 + t) ^ prow) << 4);
      double d0, d1;
      lds128(d0, d1, dbase + (kb * 16 + kk * 8 + 2 * t) * 8);
      if (MODE == 0) {
        // two blocks of one block row: A fragments shared (4 A + 8 B fragments, 64 DMMA)
        double a[4][2], b[2][4][2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) {
          lds128(a[mi][0], a[mi][1], abase + kb * box_bytes + arow[0] + mi * 1024 + chunk);
          a[mi][0] *= d0;
          a[mi][1] *= d1;
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
            lds128(b[u][ni][0], b[u][ni][1], bbase + kb * box_bytes + brow[u] + ni * 1024 + chunk);
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 4; ++ni)
                dmma(acc[u][mi][ni][0], acc[u][mi][ni][1], a[mi][h], b[u][ni][h]);
      } else {
        // one block, or two blocks of different block rows done one after the other (keeps the
        // live fragment set at 4 A + 4 B)
#pragma unroll
        for (int u = 0; u < (MODE == 1 ? 2 : 1); ++u) {
          double a[4][2], b[4][2];
#pragma unroll
          for (int mi = 0; mi < 4; ++mi) {
            lds128(a[mi][0], a[mi][1], abase + kb * box_bytes + arow[u] + mi * 1024 + chunk);
            a[mi][0] *= d0;
            a[mi][1] *= d1;
          }
#pragma unroll
          for (int ni = 0; ni < 4; ++ni)
            lds128(b[ni][0], b[ni][1], bbase + kb * box_bytes + brow[u] + ni * 1024 + chunk);
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int mi = 0; mi < 4; ++mi)
#pragma unroll
              for (int ni = 0; ni < 4; ++ni)
                dmma(acc[u][mi][ni][0], acc[u][mi][ni][1], a[mi][h], b[ni][h]);
        }
      }
    }
  }
}

// Fill ring slot s with k-slab kt: d_k = 1/(E_k - E) for the slab's 32 k (one per lane) + pole guard,
// then (lane 0) expect-tx and the 2 or 4 TMA boxes of W rows of tiles I and J. Whole warp.
template <class C>
__device__ __forceinline__ void rform_fill(uint8_t *smem, const CUtensorMap *wmap,
                                           const double *__restrict__ Ek, double Ee, int nlev,
                                           int kt, bool diag, int ti, int tj, int kstar) {
  double *dsm = reinterpret_cast<double *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *full = reinterpret_cast<uint64_t *>(dsm + C::STAGES * C::BK);
  uint64_t *empty = full + C::STAGES;
  int *pole_flag = reinterpret_cast<int *>(empty + C::STAGES);
  const int s = kt % C::STAGES, lane = lane_id();
  const int k = kt * C::BK + lane;  // BK == 32 == warp size
  double dv = 0.0;
  if (k < nlev) {
    const double diff = __ldg(Ek + k) - Ee;
    if (fabs(diff) < kPoleGuard) *pole_flag = 1;
    dv = (k == kstar) ? 0.0 : 1.0 / diff;  // the nearest pole's term is added in the epilogue
  }
  dsm[s * C::BK + lane] = dv;
  __syncwarp();
  if (lane == 0) {
    const uint32_t bytes = diag ? C::OP_BYTES : 2 * C::OP_BYTES;
    mbar_arrive_expect_tx(&full[s], bytes);
    const uint32_t base = smem_u32(smem + s * C::STAGE_BYTES);
    const int k0 = kt * C::BK;
    tma_load_2d(base, wmap, &full[s], k0, ti * C::BM);
    tma_load_2d(base + C::BOX_BYTES, wmap, &full[s], k0 + C::BOXK, ti * C::BM);
    if (!diag) {
      tma_load_2d(base + C::OP_BYTES, wmap, &full[s], k0, tj * C::BM);
      tma_load_2d(base + C::OP_BYTES + C::BOX_BYTES, wmap, &full[s], k0 + C::BOXK, tj * C::BM);
    }
  }
}

// One consumer warp: its chunk's k loop and epilogue (MODE 0: two blocks (r, c), (r, c + 1);
// MODE 2: one block; MODE 3: no block, only releases the stages). Templated whole so that each
// mode's accumulators get their own register allocation.
template <class C, int MODE>
__device__ __forceinline__ void rform_consumer(uint8_t *smem, int nk, bool diag, int rb0, int cb0,
                                               int ti, int tj, int nch, int64_t e, int pair,
                                               double inv2a, double *__restrict__ R,
                                               int32_t *__restrict__ status, const CUtensorMap *wmap,
                                               const double *__restrict__ Ek, double Ee, int nlev,
                                               const double *__restrict__ w, int64_t ldw, int kstar) {
  double *dsm = reinterpret_cast<double *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *full = reinterpret_cast<uint64_t *>(dsm + C::STAGES * C::BK);
  uint64_t *empty = full + C::STAGES;
  const int *pole_flag = reinterpret_cast<const int *>(empty + C::STAGES);
  const int lane = lane_id();
  const int g = lane >> 2, t = lane & 3;
  const int prow = frag_row_perm(g);
  constexpr int NBLK = MODE == 0 ? 2 : (MODE == 2 ? 1 : 0);
  double acc[2][4][4][2];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) acc[u][mi][ni][0] = acc[u][mi][ni][1] = 0.0;
  // byte offsets of this lane's fragment rows inside a box (row * 128); swizzle xor = prow
  // (fragment mi / ni of a block sits 8 rows = 1024 bytes further)
  const uint32_t arow[2] = {static_cast<uint32_t>((rb0 * 32 + prow) * 128), 0u};
  const uint32_t brow[2] = {static_cast<uint32_t>((cb0 * 32 + prow) * 128),
                            static_cast<uint32_t>((cb0 * 32 + 32 + prow) * 128)};

  for (int kt = 0; kt < nk; ++kt) {
    const int s = kt % C::STAGES;
    mbar_wait(&full[s], (kt / C::STAGES) & 1);
    if (MODE != 3) {
      const uint32_t abase = smem_u32(smem + s * C::STAGE_BYTES);
      const uint32_t bbase = diag ? abase : abase + C::OP_BYTES;
      const uint32_t dbase = smem_u32(dsm + s * C::BK);
      rform_slab<MODE>(acc, abase, bbase, dbase, C::BOX_BYTES, arow, brow, t, prow);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (!C::PRODUCER && warp_id() == kt % C::NCW && kt + C::STAGES < nk) {
      // this warp's turn: once every warp has released slab kt, refill its slot with kt + STAGES
      mbar_wait(&empty[s], (kt / C::STAGES) & 1);
      rform_fill<C>(smem, wmap, Ek, Ee, nlev, kt + C::STAGES, diag, ti, tj, kstar);
    }
  }

  // ===================== epilogue: scale, store tile + mirror =====================
  const bool pole = (*reinterpret_cast<const volatile int *>(pole_flag)) != 0;
  if (pole && pair == 0 && threadIdx.x == 0) set_status(status, e, RMX_E_POLE);
  double *Re = R + e * static_cast<int64_t>(nch) * nch;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  // the nearest pole's term w_ik* w_jk* d_k* / 2a, added last (reading N1)
  const double dsc = inv2a / (__ldg(Ek + kstar) - Ee);
#pragma unroll
  for (int u = 0; u < NBLK; ++u) {
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int row = ti * C::BM + rb0 * 32 + mi * 8 + prow;
      if (row >= nch) continue;
      const double wr = __ldg(w + static_cast<int64_t>(row) * ldw + kstar);
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = tj * C::BM + (cb0 + u) * 32 + ni * 8 + t + 4 * h;
          if (col >= nch) continue;
          if (diag && row > col) continue;  // lower half of a diagonal tile comes from its mirror
          const double wc = __ldg(w + static_cast<int64_t>(col) * ldw + kstar);
          const double v = pole ? nan : fma(acc[u][mi][ni][h], inv2a, (wr * wc) * dsc);
          Re[static_cast<int64_t>(row) * nch + col] = v;
          if (row != col) Re[static_cast<int64_t>(col) * nch + row] = v;
        }
      }
    }
  }
}

template <class C>
__global__ void __launch_bounds__(C::NT, 1)
    rform_dmma_kernel(const __grid_constant__ CUtensorMap wmap, const double *__restrict__ w, int64_t ldw,
                      const double *__restrict__ Ek, const double *__restrict__ E, int nch, int nlev,
                      int ntiles, int nen, double inv2a, double *__restrict__ R,
                      int32_t *__restrict__ status) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  double *dsm = reinterpret_cast<double *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *full = reinterpret_cast<uint64_t *>(dsm + C::STAGES * C::BK);
  uint64_t *empty = full + C::STAGES;
  int *pole_flag = reinterpret_cast<int *>(empty + C::STAGES);
  int *kstar_s = pole_flag + 1;

  // energies fastest: the CTAs resident at any moment are (mostly) one tile pair for up to ~148
  // energies, so they stream the same two 128-row slabs of W in lock step and W is fetched from
  // HBM about once per wave (whole-W working set per wave otherwise: DRAM ~1.3 TB/launch).
  const int pair = blockIdx.x / nen;
  const int64_t e = blockIdx.x % nen;
  int ti, tj;
  decode_pair(pair, ntiles, ti, tj);
  const bool diag = (ti == tj);
  const double Ee = E[e];
  const int nk = (nlev + C::BK - 1) / C::BK;
  const int warp = warp_id(), lane = lane_id();

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    *pole_flag = 0;
    *kstar_s = nearest_pole(Ek, nlev, Ee);
    fence_barrier_init();
  }
  __syncthreads();
  const int kstar = *kstar_s;

  if (!C::PRODUCER) {
    // prologue: warp 0 fills the first STAGES slabs; afterwards the consumers refill in turn
    if (warp == 0) {
      tma_prefetch_desc(&wmap);
      for (int kt = 0; kt < C::STAGES && kt < nk; ++kt)
        rform_fill<C>(smem, &wmap, Ek, Ee, nlev, kt, diag, ti, tj, kstar);
    }
  } else if (warp == C::NCW) {
    // ===================== producer warp: TMA + denominators =====================
    if (lane == 0) tma_prefetch_desc(&wmap);
    int found_pole = 0;
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % C::STAGES;
      if (kt >= C::STAGES) mbar_wait(&empty[s], ((kt / C::STAGES) - 1) & 1);
      const int k = kt * C::BK + lane;  // BK == 32 == warp size
      double dv = 0.0;
      if (k < nlev) {
        const double diff = __ldg(Ek + k) - Ee;
        if (fabs(diff) < kPoleGuard) found_pole = 1;
        dv = (k == kstar) ? 0.0 : 1.0 / diff;  // the nearest pole's term is added in the epilogue
      }
      dsm[s * C::BK + lane] = dv;
      if (found_pole) *pole_flag = 1;
      __syncwarp();
      if (lane == 0) {
        const uint32_t bytes = diag ? C::OP_BYTES : 2 * C::OP_BYTES;
        mbar_arrive_expect_tx(&full[s], bytes);
        const uint32_t base = smem_u32(smem + s * C::STAGE_BYTES);
        const int k0 = kt * C::BK;
        tma_load_2d(base, &wmap, &full[s], k0, ti * C::BM);
        tma_load_2d(base + C::BOX_BYTES, &wmap, &full[s], k0 + C::BOXK, ti * C::BM);
        if (!diag) {
          tma_load_2d(base + C::OP_BYTES, &wmap, &full[s], k0, tj * C::BM);
          tma_load_2d(base + C::OP_BYTES + C::BOX_BYTES, &wmap, &full[s], k0 + C::BOXK,
                      tj * C::BM);
        }
      }
    }
    return;
  }

  // ===================== consumer warps: FP64 DMMA =====================
  const int rbm = min(C::NB, (nch - ti * C::BM + 31) / 32);
  const int cbm = min(C::NB, (nch - tj * C::BM + 31) / 32);
  int rb0, cb0;
  const int nblk = rform_chunk<C::NB, C::NCW>(warp, rbm, cbm, diag, rb0, cb0);
  if (nblk == 2)
    rform_consumer<C, 0>(smem, nk, diag, rb0, cb0, ti, tj, nch, e, pair, inv2a, R, status, &wmap,
                         Ek, Ee, nlev, w, ldw, kstar);
  else if (nblk == 1)
    rform_consumer<C, 2>(smem, nk, diag, rb0, cb0, ti, tj, nch, e, pair, inv2a, R, status, &wmap,
                         Ek, Ee, nlev, w, ldw, kstar);
  else
    rform_consumer<C, 3>(smem, nk, diag, rb0, cb0, ti, tj, nch, e, pair, inv2a, R, status, &wmap,
                         Ek, Ee, nlev, w, ldw, kstar);
}

// Small-channel path (nch <= 32, e.g. BASELINE.json:7 'tiny'): one CTA per energy, each thread owns
// up to 3 upper-triangle entries (nch(nch+1)/2 <= 528 <= 3*256), denominators staged through shared
// memory in chunks. Launch-bound by construction (SURVEY.md §7 hard part 8).
__global__ void __launch_bounds__(256) rform_small_kernel(const double *__restrict__ w, int64_t ldw,
                                                          const double *__restrict__ Ek,
                                                          const double *__restrict__ E, int nch,
                                                          int nlev, double inv2a,
                                                          double *__restrict__ R,
                                                          int32_t *__restrict__ status) {
  constexpr int PPT = 3;
  __shared__ double ds[1024];
  __shared__ int pole, kstar_s;
  const int64_t e = blockIdx.x;
  const double Ee = E[e];
  if (threadIdx.x == 0) {
    pole = 0;
    kstar_s = nearest_pole(Ek, nlev, Ee);
  }
  __syncthreads();
  const int kstar = kstar_s;
  const int npair = nch * (nch + 1) / 2;
  int pi[PPT], pj[PPT];
  double s[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    pi[q] = -1;
    pj[q] = -1;
    s[q] = 0.0;
    int p = threadIdx.x + q * blockDim.x;
    if (p < npair) {
      int i = 0;
      while (p >= nch - i) {
        p -= nch - i;
        ++i;
      }
      pi[q] = i;
      pj[q] = i + p;
    }
  }
  for (int k0 = 0; k0 < nlev; k0 += 1024) {
    __syncthreads();
    for (int k = threadIdx.x; k < 1024; k += blockDim.x) {
      double dv = 0.0;
      if (k0 + k < nlev) {
        const double diff = Ek[k0 + k] - Ee;
        if (fabs(diff) < kPoleGuard) pole = 1;
        dv = (k0 + k == kstar) ? 0.0 : 1.0 / diff;  // nearest pole added last (reading N1)
      }
      ds[k] = dv;
    }
    __syncthreads();
    const int kn = min(1024, nlev - k0);
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      if (pi[q] < 0) continue;
      const double *wi = w + pi[q] * ldw + k0, *wj = w + pj[q] * ldw + k0;
      double acc = s[q];
      for (int k = 0; k < kn; ++k) acc = fma(wi[k] * ds[k], wj[k], acc);
      s[q] = acc;
    }
  }
  __syncthreads();
  double *Re = R + e * static_cast<int64_t>(nch) * nch;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  const double dsc = inv2a / (Ek[kstar] - Ee);
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    if (pi[q] < 0) continue;
    const double v = pole ? nan : fma(s[q], inv2a, (w[pi[q] * ldw + kstar] * w[pj[q] * ldw + kstar]) * dsc);
    Re[pi[q] * nch + pj[q]] = v;
    Re[pj[q] * nch + pi[q]] = v;
  }
  if (pole && threadIdx.x == 0) set_status(status, e, RMX_E_POLE);
}

// ------------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                      const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                      const cuuint32_t *, CUtensorMapInterleave,
                                      CUtensorMapSwizzle, CUtensorMapL2promotion,
                                      CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t get_encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled_t>(p);
  }
  return fn;
}

bool encode_tmap_f64(CUtensorMap *map, const double *base, int64_t rows, int64_t cols, int64_t ld,
                     int box_rows, std::string &err) {
  PFN_encodeTiled_t enc = get_encode_fn();
  if (!enc) {
    err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 8};
  cuuint32_t box[2] = {16, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "cuTensorMapEncodeTiled failed (code " + std::to_string(static_cast<int>(r)) + ")";
    return false;
  }
  return true;
}

template <class C>
static cudaError_t launch_rform_cfg(const double *w, int64_t ldw, const double *Ek, int nch,
                                    int nlev, double a, const double *E, int64_t ne, double *R,
                                    int32_t *status, cudaStream_t st, std::string &err) {
  PFN_encodeTiled_t enc = get_encode_fn();
  if (!enc) {
    err = "cuTensorMapEncodeTiled unavailable";
    return cudaErrorNotSupported;
  }
  CUtensorMap map;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(nlev), static_cast<cuuint64_t>(nch)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldw) * 8};
  cuuint32_t box[2] = {C::BOXK, C::BM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(w), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "cuTensorMapEncodeTiled failed (code " + std::to_string(static_cast<int>(r)) + ")";
    return cudaErrorInvalidValue;
  }
  {
    cudaError_t ce = ensure_smem_attr(reinterpret_cast<const void *>(rform_dmma_kernel<C>), C::SMEM_BYTES);
    if (ce != cudaSuccess) return ce;
  }
  const int ntiles = (nch + C::BM - 1) / C::BM;
  const int npairs = ntiles * (ntiles + 1) / 2;
  const double inv2a = 1.0 / (2.0 * a);
  // grid.x <= 2^31-1: chunk the energies
  const int64_t max_e = (static_cast<int64_t>(1) << 30) / npairs;
  for (int64_t e0 = 0; e0 < ne; e0 += max_e) {
    const int64_t n = (ne - e0 < max_e) ? ne - e0 : max_e;
    rform_dmma_kernel<C><<<static_cast<unsigned>(n * npairs), C::NT, C::SMEM_BYTES, st>>>(
        map, w, ldw, Ek, E + e0, nch, nlev, ntiles, static_cast<int>(n), inv2a,
        R + e0 * static_cast<int64_t>(nch) * nch, status ? status + e0 : nullptr);
    cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) return ce;
  }
  return cudaSuccess;
}

// Rform128 (dedicated producer warp) and Rform128R (consumers refill in turn, no spills) measure the
// same on darc (87.5 % vs 87.2 % of peak, profiles/r01_summary.md); RMX_RFORM_PRODUCER=0 selects R.
using Rform128 = RformCfg<128, 3, true>;
using Rform128R = RformCfg<128, 3, false>;
using Rform64 = RformCfg<64, 3, false>;

int rform_tile_for(int64_t nch) {
  if (nch <= 32) return 0;
  if (nch <= 96) return 64;
  // pick the tile that wastes the fewest MMA lanes on ragged / diagonal tiles
  auto waste = [&](int bm) {
    int64_t nt = (nch + bm - 1) / bm;
    double computed = static_cast<double>(nt * (nt + 1) / 2) * bm * bm;
    return computed / (0.5 * nch * (nch + 1));
  };
  return waste(128) <= 1.08 * waste(64) ? 128 : 64;
}

cudaError_t launch_rform(const double *w, int64_t ldw, const double *Ek, int64_t nch, int64_t nlev,
                         double a, const double *E, int64_t ne, double *R, int32_t *status,
                         cudaStream_t st, std::string &err) {
  const int bm = rform_tile_for(nch);
  if (bm == 0) {
    rform_small_kernel<<<static_cast<unsigned>(ne), 256, 0, st>>>(
        w, ldw, Ek, E, static_cast<int>(nch), static_cast<int>(nlev), 1.0 / (2.0 * a), R, status);
    return cudaGetLastError();
  }
  if (bm == 64)
    return launch_rform_cfg<Rform64>(w, ldw, Ek, static_cast<int>(nch), static_cast<int>(nlev), a,
                                     E, ne, R, status, st, err);
  static const bool rotating = [] {
    const char *v = std::getenv("RMX_RFORM_PRODUCER");
    return v && v[0] == '0';
  }();
  if (rotating)
    return launch_rform_cfg<Rform128R>(w, ldw, Ek, static_cast<int>(nch), static_cast<int>(nlev), a,
                                       E, ne, R, status, st, err);
  return launch_rform_cfg<Rform128>(w, ldw, Ek, static_cast<int>(nch), static_cast<int>(nlev), a,
                                    E, ne, R, status, st, err);
}

}  // namespace rmx
