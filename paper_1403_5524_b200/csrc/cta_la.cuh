// cta_la.cuh - CTA-level dense FP64 linear algebra on one matrix in global memory, used by the
// per-energy matching (LU) and T-epilogue (complex LDL^T, tepi.cu) kernels. Every routine is executed by all NT
// threads of one CTA; there is no inter-CTA communication (one CTA owns one energy, SURVEY.md
// §8(a) S4/S5 and BASELINE.json:5 "one CTA ... per energy").
//
//   gemm      : C op= A.B over a tile loop, 128x64 CTA tiles, FP64 DMMA (mma.m8n8k4.f64) fed by a
//               warp-specialised cp.async.bulk + mbarrier pipeline; A stored [M][K] or [K][M],
//               B stored [N][K] or [K][N]; C read (C -= A.B) or written (C = A.B)
//   panel_lu  : unblocked LU with partial pivoting of an n x bw panel (pivot = max |a|, ties ->
//               lowest row, the oracle's rule), rank-1 updates fused with the next pivot search
//   tri_inv128: inverse of a 128 x 128 triangular diagonal block (64 x 64 halves by substitution in
//               shared memory, the off-diagonal block by two DMMA GEMMs); the triangular solves
//               of the LU are then DMMA GEMMs with it (MAGMA-style inverted diagonal blocks)
#pragma once
#include "rmx_common.cuh"

namespace rmx {
namespace la {

constexpr int NT = 288;  // threads per CTA: 8 DMMA consumer warps + 1 TMA-producer warp
constexpr int NW = NT / 32;
constexpr int NCW = 8;          // consumer warps inside gemm(); warp NCW is the producer
constexpr int BM = 128, BN = 64, BK = 32, WM = 4, WN = 2;
constexpr int WTM = BM / WM, WTN = BN / WN;  // 32 x 32 warp tile
constexpr int MI = WTM / 8, NI = WTN / 8;    // 4 x 4 DMMA fragments
constexpr int PB = 32;                        // inner panel / triangle width of the factorizations
constexpr int NB = 4 * PB;                    // outer block width (K of the big trailing GEMMs)
constexpr int STAGES = 3;                     // A/B ring depth
// TMA boxes are 16 doubles (128 B, the SWIZZLE_128B span) wide:
//   view 0: {16, 128} rows   k-contiguous A slices (2 boxes per BK = 32)
//   view 1: {16, 64}  rows   k-contiguous B slices (2 boxes)
//   view 2: {16, 32}  rows   m/n-contiguous slices, 32 k-rows (8 boxes for A, 4 for B)
constexpr int NVIEW = 3;
constexpr int A_STAGE_BYTES = BM * BK * 8, B_STAGE_BYTES = BN * BK * 8;
constexpr int STAGE_BYTES = A_STAGE_BYTES + B_STAGE_BYTES;
constexpr int CS_LD = BN + 2;  // C tile pitch (bulk row copies): 4 rows = 64 mod 128 bytes apart
constexpr int C_ELEMS = BM * CS_LD;
constexpr int GEMM_SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + C_ELEMS * 8;  // + 1024 alignment slack
constexpr int GEMM_SMEM_DOUBLES = GEMM_SMEM_BYTES / 8;
constexpr int TB = 64;                        // edge of the smem-computed triangular inverses
constexpr int TB_LD = TB + 1;
constexpr int TG = NB;                        // edge (and pitch) of the global inverse Tg (128)
constexpr int TRI_SMEM_DOUBLES = 2 * TB * TB_LD;  // tri_inv64 scratch

// A matrix of a workspace slot: raw pointer + leading dimension, and its TMA descriptors
// (NVIEW box shapes, see above; the tensor extent is the matrix allocation, out-of-range
// boxes are zero filled).
struct MatView {
  const CUtensorMap *tm;
  double *base;
  int64_t ld;
  int64_t rows = 0;  // rows of the allocation (bounds-checked build; 0 = unchecked)
  __device__ __forceinline__ double *at(int r, int c) const {
    RMX_CHECK(r >= 0 && c >= 0 && c < ld && (rows == 0 || r < rows));
    return base + static_cast<int64_t>(r) * ld + c;
  }
  __device__ __forceinline__ const double *end() const { return rows ? base + rows * ld : nullptr; }
};
// An operand: the submatrix of `v` starting at (r0, c0). kc: element (i, k) of the operand is
// v(r0 + i, c0 + k) (k contiguous); otherwise v(r0 + k, c0 + i).
struct Op {
  MatView v;
  int r0, c0;
  bool kc;
};
__device__ __forceinline__ Op opk(const MatView &v, int r0, int c0) { return Op{v, r0, c0, true}; }
__device__ __forceinline__ Op opn(const MatView &v, int r0, int c0) { return Op{v, r0, c0, false}; }

__device__ __forceinline__ int cdiv(int a, int b) { return (a + b - 1) / b; }

// mbarriers of the gemm pipeline (re-initialised at every gemm call).
struct GemmSync {
  uint64_t full[STAGES], empty[STAGES], cfull, cempty;
};

// Tile enumeration (row-major over tm); lower = only tiles holding some element with row >= col.
__device__ __forceinline__ int tiles_in_row(int tm, int tiles_n, bool lower) {
  if (!lower) return tiles_n;
  const int last_col_tile = (tm * BM + BM - 1) / BN;
  return min(tiles_n, last_col_tile + 1);
}

__device__ __forceinline__ uint32_t round16(int bytes) { return static_cast<uint32_t>((bytes + 15) & ~15); }
// first k slice of output tile (tm, tn) under the kband rule of GemmArgs
__device__ __forceinline__ int kc_first(int kband, int tm, int tn) {
  return kband == 1 ? (tm * BM) / BK : (kband == 2 ? (tn * BN) / BK : 0);
}
__device__ __forceinline__ int frag_perm(int g) { return (g >> 1) + 4 * (g & 1); }
// x with its sign bit xor-ed with the top bit of `sgn` (0 or 0x80000000)
__device__ __forceinline__ double flip_sign(double x, uint32_t sgn) {
  return __hiloint2double(__double2hiint(x) ^ static_cast<int>(sgn), __double2loint(x));
}

// Producer-warp helper: bulk-copy `nrows` rows of `rbytes` bytes (16-byte multiple) from
// G + r*ld to smem rows of pitch `ld_s` doubles; completion on bar.
__device__ __forceinline__ void bulk_rows(double *s, int ld_s, const double *G, int64_t ld,
                                          int nrows, uint32_t rbytes, uint64_t *bar) {
  for (int r = lane_id(); r < nrows; r += 32)
    bulk_g2s(smem_u32(s + r * ld_s), G + static_cast<int64_t>(r) * ld, rbytes, bar);
}

struct GemmArgs {
  Op a, b;
  double *C;      // C element (i, j) at C[i*ldc + j]   (trans_c: at C[j*ldc + i])
  int64_t ldc;
  int M, N, K;
  bool lower, read_c;  // read_c: C -= A.B (C must be 16-byte aligned, ldc even); else C = A.B + diag_add I
  bool trans_c;        // store the result transposed (only with read_c == false)
  double diag_add;
  // leading k range known to contribute zero (triangular operands): 0 none; 1 A(i, k) = 0 for
  // k < i (k starts at the output tile's first row); 2 B(j, k) = 0 for k < j (k starts at the
  // output tile's first column). Whole BK slices are skipped; the rest must hold explicit zeros.
  int kband;
  bool add_c;  // with read_c: C += A.B instead of C -= A.B (tools/gemm2_proto.cuh experiment only)
  // optional second product, summed into the first along k: A.B + (neg2 ? -1 : +1) A2.B2 (same
  // M, N, K, kband and operand layouts as (a, b)); a complex product is two such real GEMMs
  // (Re = Ar.Br - Ai.Bi, Im = Ar.Bi + Ai.Br), the k range doubling instead of C being re-read
  Op a2{}, b2{};
  int nseg = 1;
  bool neg2 = false;
  double alpha = 1.0;  // set mode (read_c false): C = alpha (A.B) + diag_add I
  const double *c_end = nullptr;  // one past C's allocation (bounds-checked build; nullptr = unchecked)
};

// C[M x N] op= A[M x K] . B[K x N] on the calling CTA (all NT threads call it).
// Warp-specialised, no CTA-wide barrier in the main loop: warp NCW streams BK-deep A/B slices with
// 2D TMA (SWIZZLE_128B boxes of the slot's tensor maps) into a STAGES-deep mbarrier ring, and each
// tile's C (C -= A.B) into a C buffer by bulk row copies one tile ahead; warps 0..NCW-1 run FP64
// DMMA on 32x32 warp tiles and store their part of the tile straight to global memory.
// k-contiguous fragments are read as 16-byte (k, k+1) pairs; within each 8-row group fragment row
// g maps to smem row (g>>1) + 4(g&1) so those reads are bank-conflict free under the swizzle.
// Partial k-slices are masked (both operands zeroed beyond K).
template <bool A_KC, bool B_KC>
static __device__ __noinline__ void gemm_impl(const GemmArgs &gar, uint8_t *smem_al, GemmSync *gs) {
  // argument block copied to registers once (it arrives by reference through the call ABI, i.e.
  // from local memory; re-reading it in the epilogue cost long-scoreboard stalls)
  const GemmArgs ga = gar;
  const int M = ga.M, N = ga.N, K = ga.K;
  const bool lower = ga.lower, readC = ga.read_c;
  __syncthreads();
  if (M <= 0 || N <= 0 || K <= 0) return;
  if (threadIdx.x == 0) {
    for (int st = 0; st < STAGES; ++st) {
      mbar_init(&gs->full[st], 1);
      mbar_init(&gs->empty[st], NCW);
    }
    mbar_init(&gs->cfull, 1);
    mbar_init(&gs->cempty, NCW);
    fence_barrier_init();
  }
  __syncthreads();
  const int tiles_m = cdiv(M, BM), tiles_n = cdiv(N, BN);
  const int nkc = cdiv(K, BK);
  int ntiles = 0;
  for (int tm = 0; tm < tiles_m; ++tm) ntiles += tiles_in_row(tm, tiles_n, lower);
  double *Cs = reinterpret_cast<double *>(smem_al + STAGES * STAGE_BYTES);
  const int warp = warp_id(), lane = lane_id();

  if (warp == NCW) {
    // ============================ producer warp ============================
    // generic-proxy global writes of earlier phases (made CTA-visible by the barrier above) must be
    // ordered before the async-proxy (TMA / bulk) reads issued below
    asm volatile("fence.proxy.async;\n" ::: "memory");
    const CUtensorMap *tmAs[2] = {ga.a.v.tm + (A_KC ? 0 : 2), ga.a2.v.tm + (A_KC ? 0 : 2)};
    const CUtensorMap *tmBs[2] = {ga.b.v.tm + (B_KC ? 1 : 2), ga.b2.v.tm + (B_KC ? 1 : 2)};
    if (lane == 0)
      for (int sg = 0; sg < ga.nseg; ++sg) {
        tma_prefetch_desc(tmAs[sg]);
        tma_prefetch_desc(tmBs[sg]);
      }
    int it = 0, tm = 0, tn = 0, rowcnt = tiles_in_row(0, tiles_n, lower);
    for (int tile = 0; tile < ntiles; ++tile) {
      if (tn == rowcnt) {
        tn = 0;
        rowcnt = tiles_in_row(++tm, tiles_n, lower);
      }
      if (readC) {
        if (tile > 0) mbar_wait(&gs->cempty, (tile - 1) & 1);
        const int rows = min(BM, M - tm * BM), cols = min(BN, N - tn * BN);
        const uint32_t rb = round16(cols * 8);
        if (lane == 0) mbar_arrive_expect_tx(&gs->cfull, rb * rows);
        __syncwarp();
        RMX_CHECK(!ga.c_end || ga.C + static_cast<int64_t>(tm * BM + rows - 1) * ga.ldc + tn * BN + cols <= ga.c_end);
        bulk_rows(Cs, CS_LD, ga.C + static_cast<int64_t>(tm * BM) * ga.ldc + tn * BN, ga.ldc, rows,
                  rb, &gs->cfull);
      }
      for (int sg = 0; sg < ga.nseg; ++sg) {
      const Op &oa = sg ? ga.a2 : ga.a, &ob = sg ? ga.b2 : ga.b;
      const CUtensorMap *tmA = tmAs[sg], *tmB = tmBs[sg];
      for (int kc = kc_first(ga.kband, tm, tn); kc < nkc; ++kc, ++it) {
        const int st = it % STAGES, use = it / STAGES;
        if (it >= STAGES) mbar_wait(&gs->empty[st], (use - 1) & 1);
        if (lane == 0) {
          const int k0 = kc * BK;
          uint64_t *bar = &gs->full[st];
          mbar_arrive_expect_tx(bar, STAGE_BYTES);
          const uint32_t sa = smem_u32(smem_al + st * STAGE_BYTES), sb = sa + A_STAGE_BYTES;
          if (A_KC) {
#pragma unroll
            for (int q = 0; q < 2; ++q)
              tma_load_2d(sa + q * (BM * 128), tmA, bar, oa.c0 + k0 + 16 * q, oa.r0 + tm * BM);
          } else {
#pragma unroll
            for (int q = 0; q < BM / 16; ++q)
              tma_load_2d(sa + q * (BK * 128), tmA, bar, oa.c0 + tm * BM + 16 * q, oa.r0 + k0);
          }
          if (B_KC) {
#pragma unroll
            for (int q = 0; q < 2; ++q)
              tma_load_2d(sb + q * (BN * 128), tmB, bar, ob.c0 + k0 + 16 * q, ob.r0 + tn * BN);
          } else {
#pragma unroll
            for (int q = 0; q < BN / 16; ++q)
              tma_load_2d(sb + q * (BK * 128), tmB, bar, ob.c0 + tn * BN + 16 * q, ob.r0 + k0);
          }
        }
        __syncwarp();
      }
      }
      ++tn;
    }
  } else {
    // ============================ consumer warps ============================
    const int wm = warp % WM, wn = warp / WM;
    const int g = lane >> 2, t = lane & 3;
    const int pg = frag_perm(g);
    // per-lane byte offsets of the fragment loads inside a stage (k8 = 0; add k8 terms below)
    //   KC  : box (k8>>1) at +k8h*box, row r (r & 7 = pg), 16-byte chunk ((k8&1)*4 + t) ^ pg
    //   !KC : box m>>4, row k = 8 k8 + 2t (+1) -> (k & 7) = 2t (+1) is k8-independent
    uint32_t aoff[MI][2], boff[NI][2];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
      if (A_KC) {
        const int r = wm * WTM + mi * 8 + pg;
        aoff[mi][0] = r * 128 + ((t ^ pg) << 4);
        aoff[mi][1] = r * 128 + (((4 + t) ^ pg) << 4);
      } else {
        const int m = wm * WTM + mi * 8 + g, j2 = (m & 15) >> 1;
        const uint32_t base = (m >> 4) * (BK * 128) + ((m & 1) << 3);
        aoff[mi][0] = base + (2 * t) * 128 + ((j2 ^ (2 * t)) << 4);
        aoff[mi][1] = base + (2 * t + 1) * 128 + ((j2 ^ (2 * t + 1)) << 4);
      }
    }
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      if (B_KC) {
        const int r = wn * WTN + ni * 8 + pg;
        boff[ni][0] = r * 128 + ((t ^ pg) << 4);
        boff[ni][1] = r * 128 + (((4 + t) ^ pg) << 4);
      } else {
        const int n = wn * WTN + ni * 8 + g, j2 = (n & 15) >> 1;
        const uint32_t base = (n >> 4) * (BK * 128) + ((n & 1) << 3);
        boff[ni][0] = base + (2 * t) * 128 + ((j2 ^ (2 * t)) << 4);
        boff[ni][1] = base + (2 * t + 1) * 128 + ((j2 ^ (2 * t + 1)) << 4);
      }
    }
    const int arow = A_KC ? pg : g;  // tile-local row offset of this lane's accumulator rows
    const uint32_t smem0 = smem_u32(smem_al);
    double acc[MI][NI][2];
    int it = 0, tm = 0, tn = 0, rowcnt = tiles_in_row(0, tiles_n, lower);
    for (int tile = 0; tile < ntiles; ++tile) {
      if (tn == rowcnt) {
        tn = 0;
        rowcnt = tiles_in_row(++tm, tiles_n, lower);
      }
      if (readC) {
        mbar_wait(&gs->cfull, tile & 1);
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          const double *cr = Cs + (wm * WTM + mi * 8 + arow) * CS_LD + wn * WTN;
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) {
            double c0, c1;
            if (B_KC) {
              c0 = cr[ni * 8 + t];
              c1 = cr[ni * 8 + t + 4];
            } else {
              lds128(c0, c1, smem_u32(cr + ni * 8 + 2 * t));
            }
            acc[mi][ni][0] = -c0;  // C -= A.B as acc = -C; acc += A.B; C = -acc (exact)
            acc[mi][ni][1] = -c1;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&gs->cempty);
      } else {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      }
      // lower mode: a warp tile entirely above the diagonal (its last row < its first column) only
      // keeps the ring protocol (waits and arrivals): no DMMA, no store - the callers never read
      // the strict upper part of a lower-tile result (DMMA pipe time on the diagonal tiles)
      const bool upper_only = lower && (tm * BM + wm * WTM + WTM - 1 < tn * BN + wn * WTN);
      for (int sg = 0; sg < ga.nseg; ++sg) {
      // sign of the second product: flip the sign bit of its A fragments (integer op, off the
      // FP64 pipe)
      const uint32_t sgn = (sg == 1 && ga.neg2) ? 0x80000000u : 0u;
      for (int kc = kc_first(ga.kband, tm, tn); kc < nkc; ++kc, ++it) {
        const int st = it % STAGES, use = it / STAGES;
        mbar_wait(&gs->full[st], use & 1);
        if (upper_only) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&gs->empty[st]);
          continue;
        }
        const int krem = min(BK, K - kc * BK);
        const uint32_t sa = smem0 + st * STAGE_BYTES, sb = sa + A_STAGE_BYTES;
        auto step = [&](const int k8, const bool partial) {
          double a[MI][2], b[NI][2];
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) {
            if (A_KC) {
              lds128(a[mi][0], a[mi][1], sa + (k8 >> 1) * (BM * 128) + aoff[mi][k8 & 1]);
            } else {
              a[mi][0] = lds64(sa + k8 * 1024 + aoff[mi][0]);
              a[mi][1] = lds64(sa + k8 * 1024 + aoff[mi][1]);
            }
          }
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) {
            if (B_KC) {
              lds128(b[ni][0], b[ni][1], sb + (k8 >> 1) * (BN * 128) + boff[ni][k8 & 1]);
            } else {
              b[ni][0] = lds64(sb + k8 * 1024 + boff[ni][0]);
              b[ni][1] = lds64(sb + k8 * 1024 + boff[ni][1]);
            }
          }
#pragma unroll
          for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int h = 0; h < 2; ++h) a[mi][h] = flip_sign(a[mi][h], sgn);
          if (partial) {  // zero both operands beyond K (stale smem may hold anything)
            const int k = k8 * 8 + 2 * t;
            const bool v0 = k < krem, v1 = k + 1 < krem;
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) {
              a[mi][0] = v0 ? a[mi][0] : 0.0;
              a[mi][1] = v1 ? a[mi][1] : 0.0;
            }
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
              b[ni][0] = v0 ? b[ni][0] : 0.0;
              b[ni][1] = v1 ? b[ni][1] : 0.0;
            }
          }
          // k-slot 0 for all 16 accumulators, then k-slot 1: dependent DMMAs are 16 issues apart
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
              for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], a[mi][h], b[ni][h]);
        };
        if (krem == BK) {
#pragma unroll
          for (int k8 = 0; k8 < BK / 8; ++k8) step(k8, false);
        } else {
#pragma unroll 1
          for (int k8 = 0; k8 * 8 < krem; ++k8) step(k8, true);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&gs->empty[st]);
      }
      }
      // epilogue: this warp's 32 x 32 part of the tile straight to global memory
#pragma unroll
      for (int mi = 0; mi < (upper_only ? 0 : MI); ++mi) {
        const int r = tm * BM + wm * WTM + mi * 8 + arow;
        if (r >= M) continue;
        double *crow = ga.C + static_cast<int64_t>(r) * ga.ldc;
        RMX_CHECK(!ga.c_end || crow + min(N, tn * BN + BN) <= ga.c_end);
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = tn * BN + wn * WTN + ni * 8 + (B_KC ? t + 4 * h : 2 * t + h);
            if (c >= N) continue;
            if (readC)
              crow[c] = -acc[mi][ni][h];
            else if (ga.trans_c)
              ga.C[static_cast<int64_t>(c) * ga.ldc + r] = acc[mi][ni][h];
            else
              crow[c] = ga.alpha * acc[mi][ni][h] + (r == c ? ga.diag_add : 0.0);
          }
      }
      ++tn;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void gemm_rt(const GemmArgs &ga, uint8_t *smem_al, GemmSync *gs) {
  if (ga.a.kc) {
    if (ga.b.kc)
      gemm_impl<true, true>(ga, smem_al, gs);
    else
      gemm_impl<true, false>(ga, smem_al, gs);
  } else {
    if (ga.b.kc)
      gemm_impl<false, true>(ga, smem_al, gs);
    else
      gemm_impl<false, false>(ga, smem_al, gs);
  }
}

// Front ends (one compiled instance of the pipeline for every call site).
__device__ __forceinline__ uint8_t *gemm_smem_align(double *smem) {
  return reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem) + 1023) &
                                     ~static_cast<uintptr_t>(1023));
}
// C -= A.B   (C = the submatrix of `c` at (r0, c0))
__device__ __forceinline__ void gemm_sub(int M, int N, int K, const Op &a, const Op &b,
                                         const MatView &c, int cr0, int cc0, bool lower,
                                         double *smem, GemmSync *gs) {
  GemmArgs ga{a, b, c.at(cr0, cc0), c.ld, M, N, K, lower, true, false, 0.0};
  ga.c_end = c.end();
  gemm_rt(ga, gemm_smem_align(smem), gs);
}
// C = A.B + diag_add I
__device__ __forceinline__ void gemm_set(int M, int N, int K, const Op &a, const Op &b,
                                         const MatView &c, int cr0, int cc0, bool lower,
                                         double diag_add, double *smem, GemmSync *gs) {
  GemmArgs ga{a, b, c.at(cr0, cc0), c.ld, M, N, K, lower, false, false, diag_add};
  ga.c_end = c.end();
  gemm_rt(ga, gemm_smem_align(smem), gs);
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
// below the diagonal, U on and above; pivot rows (absolute) in ipiv[0..bw). Returns 1 on an exact
// zero pivot. Pivot rule: max |a_ij| over the remaining rows, ties -> lowest row (the oracle's rule).
// The panel is processed in sub-panels of SPW = 8 columns held in shared memory (sp: >= (n-p0)*9
// doubles): each sub-panel is factored entirely in smem (pivot search, row swap, rank-1 update per
// column), written back, its interchanges are applied to the whole augmented rows [sc0, sc1) in
// order, and the panel's remaining columns get one rank-8 update pass (U rows by a unit-lower 8x8
// solve). Global memory is touched ~4 times per 32 columns instead of once per column.
constexpr int SPW = 8, SP_LD = SPW + 1;
constexpr int PERM_MAX = 2 * PB;
#ifdef RMX_PHASES
// panel_lu sub-step clock64 totals of block 0 (diagnostic build; rmx_debug_panel_phases)
static __device__ unsigned long long g_panel_phase[6];
#define PANEL_MARK(k)                                   \
  do {                                                  \
    __syncthreads();                                    \
    if (blockIdx.x == 0 && threadIdx.x == 0) {          \
      const unsigned long long now_ = clock64();        \
      g_panel_phase[k] += now_ - pp_t0;                 \
      pp_t0 = now_;                                     \
    }                                                   \
  } while (0)
#else
#define PANEL_MARK(k) \
  do {                \
  } while (0)
#endif
#ifndef RMX_PANEL_SU
#define RMX_PANEL_SU 16
#endif
  // rows touched by the interchanges of one panel

__device__ __forceinline__ int panel_lu(double *M, int64_t ld, int n, int p0, int bw, int sc0,
                                        int sc1, int *ipiv, double *sp, double *ubuf, double *redv,
                                        int *redi) {
  int singular = 0;
#ifdef RMX_PHASES
  unsigned long long pp_t0 = clock64();
#endif
  for (int s0 = 0; s0 < bw; s0 += SPW) {
    const int c0 = p0 + s0, w = min(SPW, bw - s0), nr = n - c0;
    // 1. stage the sub-panel rows c0..n-1, columns c0..c0+w (SU loads in flight per thread)
    constexpr int SU = RMX_PANEL_SU;
    __syncthreads();
    for (int q0 = threadIdx.x; q0 < nr * SPW; q0 += NT * SU) {
      double v[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int q = q0 + u * NT, r = q / SPW, c = q % SPW;
        v[u] = (q < nr * SPW && c < w) ? M[static_cast<int64_t>(c0 + r) * ld + c0 + c] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int q = q0 + u * NT;
        if (q < nr * SPW) sp[(q / SPW) * SP_LD + q % SPW] = v[u];
      }
    }
    __syncthreads();
    PANEL_MARK(0);
    // 2. factor in shared memory; each column's rank-1 update pass also searches the next
    // column's pivot (one pass over the rows and one barrier per column fewer)
    double best = -1.0;
    int besti = nr;
    for (int r = threadIdx.x; r < nr; r += NT) {
      const double v = fabs(sp[r * SP_LD]);
      if (v > best) {
        best = v;
        besti = r;
      }
    }
    for (int jj = 0; jj < w; ++jj) {
      block_argmax(best, besti, redv, redi);
      const int pr = besti < nr ? besti : jj;  // all-NaN column (e.g. a pole energy): no interchange
      if (threadIdx.x < SPW && pr != jj) {
        const double t0 = sp[jj * SP_LD + threadIdx.x];
        sp[jj * SP_LD + threadIdx.x] = sp[pr * SP_LD + threadIdx.x];
        sp[pr * SP_LD + threadIdx.x] = t0;
      }
      if (threadIdx.x == 0) ipiv[s0 + jj] = c0 + pr;
      __syncthreads();
      const double piv = sp[jj * SP_LD + jj];
      const bool zero = (piv == 0.0);
      singular |= zero;
      const double rpiv = zero ? 0.0 : 1.0 / piv;
      double u[SPW];
#pragma unroll
      for (int q = 0; q < SPW; ++q) u[q] = sp[jj * SP_LD + q];
      const int jn = jj + 1;  // next pivot column (searched over rows >= jn)
      best = -1.0;
      besti = nr;
      for (int r = jn + threadIdx.x; r < nr; r += NT) {
        double *row = sp + r * SP_LD;
        const double l = zero ? 0.0 : row[jj] * rpiv;
        if (!zero) row[jj] = l;
#pragma unroll
        for (int q = 0; q < SPW; ++q)
          if (q > jj) row[q] = fma(-l, u[q], row[q]);
        if (jn < w) {
          const double v = fabs(row[jn]);
          if (v > best) {
            best = v;
            besti = r;
          }
        }
      }
    }
    __syncthreads();
    PANEL_MARK(1);
    // 3. write the factored sub-panel back
    for (int q = threadIdx.x; q < nr * SPW; q += NT) {
      const int r = q / SPW, c = q % SPW;
      if (c < w) M[static_cast<int64_t>(c0 + r) * ld + c0 + c] = sp[r * SP_LD + c];
    }
    // 4. the sub-panel's interchanges, in order, on the rest of the augmented rows (a composed
    // permutation of the panel's rows, applied once per panel, measured slower: the pass is bound by
    // the rows' bytes)
    for (int jj = 0; jj < w; ++jj) {
      const int pr = ipiv[s0 + jj], j = c0 + jj;
      RMX_CHECK(pr >= j && pr < n && sc1 <= ld);
      if (pr != j) {
        double *ra = M + static_cast<int64_t>(j) * ld;
        double *rb = M + static_cast<int64_t>(pr) * ld;
        constexpr int SU = 4;
        for (int cb = sc0 + threadIdx.x; cb < sc1; cb += NT * SU) {
          double va[SU], vb[SU];
#pragma unroll
          for (int q = 0; q < SU; ++q) {
            const int c = cb + q * NT;
            const bool ok = c < sc1 && (c < c0 || c >= c0 + w);
            va[q] = ok ? ra[c] : 0.0;
            vb[q] = ok ? rb[c] : 0.0;
          }
#pragma unroll
          for (int q = 0; q < SU; ++q) {
            const int c = cb + q * NT;
            if (c < sc1 && (c < c0 || c >= c0 + w)) {
              ra[c] = vb[q];
              rb[c] = va[q];
            }
          }
        }
      }
      __syncthreads();
    }
    PANEL_MARK(2);
    // 5. rank-w update of the panel's remaining columns [c0+w, p0+bw)
    const int cr0 = c0 + w, nc = p0 + bw - cr0;
    if (nc > 0) {
      // U rows c0..c0+w-1: unit-lower solve with L_ss (sp), one thread per column
      if (threadIdx.x < nc) {
        const int c = cr0 + threadIdx.x;
        double x[SPW];
#pragma unroll
        for (int q = 0; q < SPW; ++q) {
          double v = q < w ? M[static_cast<int64_t>(c0 + q) * ld + c] : 0.0;
#pragma unroll
          for (int k = 0; k < q; ++k) v = fma(-sp[q * SP_LD + k], x[k], v);
          x[q] = v;
        }
#pragma unroll
        for (int q = 0; q < SPW; ++q) {
          ubuf[q * PB + threadIdx.x] = x[q];
          if (q < w) M[static_cast<int64_t>(c0 + q) * ld + c] = x[q];
        }
      }
      __syncthreads();
      // rows c0+w..n-1: M[i][c] -= sum_q L[i][q] U[q][c]; (row, column) elements dealt to all
      // threads, UNR independent loads in flight per thread (the pass is latency-bound)
      constexpr int UNR = 16;
      const int tot = (nr - w) * nc;
      for (int q0 = threadIdx.x; q0 < tot; q0 += NT * UNR) {
        double x[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int q = q0 + u * NT, r = w + q / nc, c = q % nc;
          x[u] = q < tot ? M[static_cast<int64_t>(c0 + r) * ld + cr0 + c] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
          const int q = q0 + u * NT, r = w + q / nc, c = q % nc;
          if (q < tot) {
            double v = x[u];
#pragma unroll
            for (int k = 0; k < SPW; ++k) v = fma(-sp[r * SP_LD + k], ubuf[k * PB + c], v);
            M[static_cast<int64_t>(c0 + r) * ld + cr0 + c] = v;
          }
        }
      }
    }
    PANEL_MARK(3);
  }
  __syncthreads();
  return singular;
}

enum { TRI_UNIT_LOWER = 0, TRI_LOWER = 1, TRI_UPPER = 2 };
// Inverse of the W x W (W <= 64) diagonal block of `src` at (p0, p0) written to Tg [64][64]
// (global, zero outside W x W): two 32 x 32 diagonal inverses by substitution (warps 0 and 1,
// lane = column), then the off-diagonal block from the 2 x 2 block formula
//   lower:  [[A, 0], [C, B]]^-1 = [[A^-1, 0], [-B^-1 C A^-1, B^-1]]
//   upper:  [[A, C], [0, B]]^-1 = [[A^-1, -A^-1 C B^-1], [0, B^-1]]
__device__ __forceinline__ void tri_inv64(const double *src, int64_t ld, int p0, int W, int kind,
                                          double *sm, double *Tg, int ldt = TB) {
  double *Lb = sm, *Tb = sm + TB * TB_LD;
  __syncthreads();
  for (int q = threadIdx.x; q < TB * TB; q += NT) {
    const int r = q / TB, c = q % TB;
    double v = 0.0;
    if (r < W && c < W) {
      const bool keep = kind == TRI_UPPER ? (c >= r) : (kind == TRI_LOWER ? (c <= r) : (c < r));
      if (keep) v = src[static_cast<int64_t>(p0 + r) * ld + p0 + c];
      if (kind == TRI_UNIT_LOWER && r == c) v = 1.0;
    } else if (r == c) {
      v = 1.0;  // identity padding keeps the fixed-size substitution finite
    }
    Lb[r * TB_LD + c] = v;
    Tb[r * TB_LD + c] = 0.0;
  }
  __syncthreads();
  if (warp_id() < 2) {
    const int o = 32 * warp_id(), c = lane_id();
    double x[32];
    if (kind != TRI_UPPER) {
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        double s = (r == c) ? 1.0 : 0.0;
#pragma unroll
        for (int q = 0; q < r; ++q) s = fma(-Lb[(o + r) * TB_LD + o + q], x[q], s);
        x[r] = (kind == TRI_LOWER) ? s / Lb[(o + r) * TB_LD + o + r] : s;
      }
    } else {
#pragma unroll
      for (int r = 31; r >= 0; --r) {
        double s = (r == c) ? 1.0 : 0.0;
#pragma unroll
        for (int q = r + 1; q < 32; ++q) s = fma(-Lb[(o + r) * TB_LD + o + q], x[q], s);
        x[r] = s / Lb[(o + r) * TB_LD + o + r];
      }
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) Tb[(o + r) * TB_LD + o + c] = x[r];
  }
  __syncthreads();
  // off-diagonal 32 x 32 block; P is staged in the block's unused (zero) quadrant of Tb
  const bool upper = kind == TRI_UPPER;
  for (int q = threadIdx.x; q < 32 * 32; q += NT) {
    const int i = q / 32, j = q % 32;
    double s = 0.0;
    if (!upper) {  // P = C A^-1, C = Lb[32+i][k], A^-1 = Tb[k][j] (lower: k >= j)
      for (int k = j; k < 32; ++k) s = fma(Lb[(32 + i) * TB_LD + k], Tb[k * TB_LD + j], s);
      Tb[i * TB_LD + 32 + j] = s;
    } else {       // P = C B^-1, C = Lb[i][32+k], B^-1 = Tb[32+k][32+j] (upper: k <= j)
      for (int k = 0; k <= j; ++k) s = fma(Lb[i * TB_LD + 32 + k], Tb[(32 + k) * TB_LD + 32 + j], s);
      Tb[(32 + i) * TB_LD + j] = s;
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < 32 * 32; q += NT) {
    const int i = q / 32, j = q % 32;
    double s = 0.0;
    if (!upper) {  // -B^-1 P, B^-1 = Tb[32+i][32+k] (k <= i), P[k][j] = Tb[k][32+j]
      for (int k = 0; k <= i; ++k) s = fma(Tb[(32 + i) * TB_LD + 32 + k], Tb[k * TB_LD + 32 + j], s);
      Lb[(32 + i) * TB_LD + j] = -s;  // result staged in Lb (its lower-left block is consumed)
    } else {       // -A^-1 P, A^-1 = Tb[i][k] (k >= i), P[k][j] = Tb[32+k][j]
      for (int k = i; k < 32; ++k) s = fma(Tb[i * TB_LD + k], Tb[(32 + k) * TB_LD + j], s);
      Lb[i * TB_LD + 32 + j] = -s;
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < TB * TB; q += NT) {
    const int r = q / TB, c = q % TB;
    double v = 0.0;
    if (r < W && c < W) {
      const bool off = upper ? (r < 32 && c >= 32) : (r >= 32 && c < 32);
      const bool zero = upper ? (r >= 32 && c < 32) : (r < 32 && c >= 32);
      v = off ? Lb[r * TB_LD + c] : (zero ? 0.0 : Tb[r * TB_LD + c]);
    }
    Tg[r * ldt + c] = v;
  }
  __syncthreads();
}

// Inverse of the W x W (W <= NB = 128) triangular diagonal block of `sv` at (p0, p0) into the
// global Tg [128][128] (view tv, zero outside W x W): 64 x 64 diagonal inverses in shared memory
// (tri_inv64) and the off-diagonal 64-block by two DMMA GEMMs with the 2 x 2 block formula
//   lower: T21 = -T2 (L21 T1)          upper: T12 = -T1 (U12 T2)
// (the product is staged in the quadrant that ends up zero, then cleared).
__device__ __forceinline__ void tri_inv128(const MatView &sv, int p0, int W, int kind,
                                           const MatView &tv, double *smem, GemmSync *gs) {
  double *Tg = tv.base;
  __syncthreads();
  for (int q = threadIdx.x; q < TG * TG; q += NT) Tg[q] = 0.0;
  const int W1 = min(W, TB), W2 = W - W1;
  tri_inv64(sv.base, sv.ld, p0, W1, kind, smem, Tg, TG);
  if (W2 > 0) {
    tri_inv64(sv.base, sv.ld, p0 + TB, W2, kind, smem, Tg + TB * TG + TB, TG);
    if (kind != TRI_UPPER) {
      // P = L21 T1 -> Tg[0:W2, 64:128); T21 = -T2 P -> Tg[64:64+W2, 0:64)
      gemm_set(W2, TB, TB, opk(sv, p0 + TB, p0), opn(tv, 0, 0), tv, 0, TB, false, 0.0, smem, gs);
      gemm_sub(W2, TB, W2, opk(tv, TB, TB), opn(tv, 0, TB), tv, TB, 0, false, smem, gs);
      for (int q = threadIdx.x; q < TB * TB; q += NT) Tg[(q / TB) * TG + TB + (q % TB)] = 0.0;
    } else {
      // P = U12 T2 -> Tg[64:128, 0:W2); T12 = -T1 P -> Tg[0:64, 64:64+W2)
      gemm_set(TB, W2, W2, opk(sv, p0, p0 + TB), opn(tv, TB, TB), tv, TB, 0, false, 0.0, smem, gs);
      gemm_sub(TB, W2, TB, opk(tv, 0, 0), opn(tv, TB, 0), tv, 0, TB, false, smem, gs);
      for (int q = threadIdx.x; q < TB * TB; q += NT) Tg[(TB + q / TB) * TG + (q % TB)] = 0.0;
    }
  }
  __syncthreads();
}

}  // namespace la
}  // namespace rmx
