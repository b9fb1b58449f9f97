// cta_cgemm.cuh - complex CTA GEMM of the T epilogue (tepi.cu) by the 3M (Gauss) scheme:
//     T1 = Ar Br,  T2 = Ai Bi,  T3 = (Ar + Ai)(Br + Bi)  ->  Re = T1 - T2,  Im = T3 - T1 - T2
// three real FP64 DMMA products per complex product instead of four (the T route's executed flops
// drop from 4 o^3 to 3 o^3), and both output planes from ONE pass over the four
// operand planes (the 2-pass real form loaded every operand twice).
// Same pipeline as cta_la.cuh gemm_impl (one TMA producer warp, 8 DMMA consumer warps, mbarrier
// ring, swizzled fragment loads); tile 128 x 32 with 32 x 16 warp tiles so that the three
// accumulator sets (48 registers) fit the 168-register budget of a 9-warp CTA; 2 stages of 80 KB
// (the four planes' k-slices); the sum operands (Ar + Ai), (Br + Bi) are formed in registers. The
// T epilogue uses it for the products that write C (C = alpha A.B); its sub mode (C -= A.B, C read in
// the epilogue) is kept for completeness - the trailing updates run the 4-product form of gemm_impl,
// whose 128 x 64 tiles amortise the staged C tile over twice the k range (tepi.cu).
// Rounding: Im = (T3 - T1) - T2; the error bound u (|Ar| + |Ai|)(|Br| + |Bi|) is that of the
// 4-product form up to a factor <= 2 (normwise).
#pragma once
#include "cta_la.cuh"

namespace rmx {
namespace la {

constexpr int C3_BN = 32, C3_WTN = C3_BN / WN, C3_NI = C3_WTN / 8;  // 32 x 16 warp tiles, 4 x 2 fragments
constexpr int C3_STAGES = 2;
constexpr int C3_A_BYTES = BM * BK * 8, C3_B_BYTES = C3_BN * BK * 8;
constexpr int C3_STAGE_BYTES = 2 * C3_A_BYTES + 2 * C3_B_BYTES;  // Ar, Ai, Br, Bi
static_assert(1024 + C3_STAGES * C3_STAGE_BYTES <= GEMM_SMEM_BYTES, "cgemm3 stages exceed the gemm smem");

struct CGemmArgs {
  Op ar, ai, br, bi;  // operands (re, im planes); a pair shares its layout flag
  double *Cr, *Ci;    // output planes at the submatrix origin
  int64_t ldc;
  const double *cr_end = nullptr, *ci_end = nullptr;  // bounds-checked build
  int M, N, K;
  bool lower, sub;  // sub: C -= A.B; else C = alpha A.B
  int kband;        // as GemmArgs::kband
  double alpha;
};

__device__ __forceinline__ int c3_tiles_in_row(int tm, int tiles_n, bool lower) {
  if (!lower) return tiles_n;
  return min(tiles_n, (tm * BM + BM - 1) / C3_BN + 1);
}
__device__ __forceinline__ int c3_kc_first(int kband, int tm, int tn) {
  return kband == 1 ? (tm * BM) / BK : (kband == 2 ? (tn * C3_BN) / BK : 0);
}

template <bool A_KC, bool B_KC>
static __device__ __noinline__ void cgemm3_impl(const CGemmArgs &gar, uint8_t *smem_al, GemmSync *gs) {
  // the argument block arrives by reference (local memory): each role copies only what it uses
  const int M = gar.M, N = gar.N, K = gar.K, kband = gar.kband;
  const bool lower = gar.lower;
  __syncthreads();
  if (M <= 0 || N <= 0 || K <= 0) return;
  if (threadIdx.x == 0) {
    for (int st = 0; st < C3_STAGES; ++st) {
      mbar_init(&gs->full[st], 1);
      mbar_init(&gs->empty[st], NCW);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int tiles_m = cdiv(M, BM), tiles_n = cdiv(N, C3_BN);
  const int nkc = cdiv(K, BK);
  int ntiles = 0;
  for (int tm = 0; tm < tiles_m; ++tm) ntiles += c3_tiles_in_row(tm, tiles_n, lower);
  const int warp = warp_id(), lane = lane_id();

  if (warp == NCW) {
    // ============================ producer warp ============================
    asm volatile("fence.proxy.async;\n" ::: "memory");
    // views: 0 = {16, 128} rows (A k-contiguous), 2 = {16, 32} rows (B k-contiguous; m/n-contiguous)
    const CUtensorMap *tA[2] = {gar.ar.v.tm + (A_KC ? 0 : 2), gar.ai.v.tm + (A_KC ? 0 : 2)};
    const CUtensorMap *tB[2] = {gar.br.v.tm + 2, gar.bi.v.tm + 2};
    const int ar0[2] = {gar.ar.r0, gar.ai.r0}, ac0[2] = {gar.ar.c0, gar.ai.c0};
    const int br0[2] = {gar.br.r0, gar.bi.r0}, bc0[2] = {gar.br.c0, gar.bi.c0};
    if (lane == 0)
      for (int p = 0; p < 2; ++p) {
        tma_prefetch_desc(tA[p]);
        tma_prefetch_desc(tB[p]);
      }
    int it = 0, tm = 0, tn = 0, rowcnt = c3_tiles_in_row(0, tiles_n, lower);
    for (int tile = 0; tile < ntiles; ++tile) {
      if (tn == rowcnt) {
        tn = 0;
        rowcnt = c3_tiles_in_row(++tm, tiles_n, lower);
      }
      for (int kc = c3_kc_first(kband, tm, tn); kc < nkc; ++kc, ++it) {
        const int st = it % C3_STAGES, use = it / C3_STAGES;
        if (it >= C3_STAGES) mbar_wait(&gs->empty[st], (use - 1) & 1);
        if (lane == 0) {
          const int k0 = kc * BK;
          uint64_t *bar = &gs->full[st];
          mbar_arrive_expect_tx(bar, C3_STAGE_BYTES);
          const uint32_t s0 = smem_u32(smem_al + st * C3_STAGE_BYTES);
#pragma unroll
          for (int p = 0; p < 2; ++p) {
            const uint32_t sa = s0 + p * C3_A_BYTES, sb = s0 + 2 * C3_A_BYTES + p * C3_B_BYTES;
            if (A_KC) {
#pragma unroll
              for (int q = 0; q < 2; ++q)
                tma_load_2d(sa + q * (BM * 128), tA[p], bar, ac0[p] + k0 + 16 * q, ar0[p] + tm * BM);
            } else {
#pragma unroll
              for (int q = 0; q < BM / 16; ++q)
                tma_load_2d(sa + q * (BK * 128), tA[p], bar, ac0[p] + tm * BM + 16 * q, ar0[p] + k0);
            }
            if (B_KC) {
#pragma unroll
              for (int q = 0; q < 2; ++q)
                tma_load_2d(sb + q * (C3_BN * 128), tB[p], bar, bc0[p] + k0 + 16 * q, br0[p] + tn * C3_BN);
            } else {
#pragma unroll
              for (int q = 0; q < C3_BN / 16; ++q)
                tma_load_2d(sb + q * (BK * 128), tB[p], bar, bc0[p] + tn * C3_BN + 16 * q, br0[p] + k0);
            }
          }
        }
        __syncwarp();
      }
      ++tn;
    }
  } else {
    // ============================ consumer warps ============================
    const int wm = warp % WM, wn = warp / WM;
    const int g = lane >> 2, t = lane & 3;
    const int pg = frag_perm(g);
    uint32_t aoff[MI][2], boff[C3_NI][2];
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
    for (int ni = 0; ni < C3_NI; ++ni) {
      if (B_KC) {
        const int r = wn * C3_WTN + ni * 8 + pg;
        boff[ni][0] = r * 128 + ((t ^ pg) << 4);
        boff[ni][1] = r * 128 + (((4 + t) ^ pg) << 4);
      } else {
        const int n = wn * C3_WTN + ni * 8 + g, j2 = (n & 15) >> 1;
        const uint32_t base = (n >> 4) * (BK * 128) + ((n & 1) << 3);
        boff[ni][0] = base + (2 * t) * 128 + ((j2 ^ (2 * t)) << 4);
        boff[ni][1] = base + (2 * t + 1) * 128 + ((j2 ^ (2 * t + 1)) << 4);
      }
    }
    const int arow = A_KC ? pg : g;
    const uint32_t smem0 = smem_u32(smem_al);
    double *const Cr = gar.Cr, *const Ci = gar.Ci;
    const int64_t ldc = gar.ldc;
    const bool sub = gar.sub;
    const double alpha = gar.alpha;
#ifdef RMX_CHECKS
    const double *cr_end = gar.cr_end, *ci_end = gar.ci_end;
#endif
    double t1[MI][C3_NI][2], t2[MI][C3_NI][2], t3[MI][C3_NI][2];
    int it = 0, tm = 0, tn = 0, rowcnt = c3_tiles_in_row(0, tiles_n, lower);
    for (int tile = 0; tile < ntiles; ++tile) {
      if (tn == rowcnt) {
        tn = 0;
        rowcnt = c3_tiles_in_row(++tm, tiles_n, lower);
      }
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < C3_NI; ++ni)
#pragma unroll
          for (int h = 0; h < 2; ++h) t1[mi][ni][h] = t2[mi][ni][h] = t3[mi][ni][h] = 0.0;
      // lower mode: a warp tile entirely above the diagonal keeps only the ring protocol
      const bool upper_only = lower && (tm * BM + wm * WTM + WTM - 1 < tn * C3_BN + wn * C3_WTN);
      for (int kc = c3_kc_first(kband, tm, tn); kc < nkc; ++kc, ++it) {
        const int st = it % C3_STAGES, use = it / C3_STAGES;
        mbar_wait(&gs->full[st], use & 1);
        if (upper_only) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&gs->empty[st]);
          continue;
        }
        const int krem = min(BK, K - kc * BK);
        const uint32_t s0 = smem0 + st * C3_STAGE_BYTES;
        const uint32_t sar = s0, sai = s0 + C3_A_BYTES, sbr = s0 + 2 * C3_A_BYTES, sbi = sbr + C3_B_BYTES;
        auto step = [&](const int k8, const bool partial) {
          double ar[MI][2], ai[MI][2], br[C3_NI][2], bi[C3_NI][2];
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) {
            if (A_KC) {
              lds128(ar[mi][0], ar[mi][1], sar + (k8 >> 1) * (BM * 128) + aoff[mi][k8 & 1]);
              lds128(ai[mi][0], ai[mi][1], sai + (k8 >> 1) * (BM * 128) + aoff[mi][k8 & 1]);
            } else {
              ar[mi][0] = lds64(sar + k8 * 1024 + aoff[mi][0]);
              ar[mi][1] = lds64(sar + k8 * 1024 + aoff[mi][1]);
              ai[mi][0] = lds64(sai + k8 * 1024 + aoff[mi][0]);
              ai[mi][1] = lds64(sai + k8 * 1024 + aoff[mi][1]);
            }
          }
#pragma unroll
          for (int ni = 0; ni < C3_NI; ++ni) {
            if (B_KC) {
              lds128(br[ni][0], br[ni][1], sbr + (k8 >> 1) * (C3_BN * 128) + boff[ni][k8 & 1]);
              lds128(bi[ni][0], bi[ni][1], sbi + (k8 >> 1) * (C3_BN * 128) + boff[ni][k8 & 1]);
            } else {
              br[ni][0] = lds64(sbr + k8 * 1024 + boff[ni][0]);
              br[ni][1] = lds64(sbr + k8 * 1024 + boff[ni][1]);
              bi[ni][0] = lds64(sbi + k8 * 1024 + boff[ni][0]);
              bi[ni][1] = lds64(sbi + k8 * 1024 + boff[ni][1]);
            }
          }
          if (partial) {  // zero both operands beyond K
            const int k = k8 * 8 + 2 * t;
            const bool v0 = k < krem, v1 = k + 1 < krem;
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) {
              ar[mi][0] = v0 ? ar[mi][0] : 0.0;
              ar[mi][1] = v1 ? ar[mi][1] : 0.0;
              ai[mi][0] = v0 ? ai[mi][0] : 0.0;
              ai[mi][1] = v1 ? ai[mi][1] : 0.0;
            }
#pragma unroll
            for (int ni = 0; ni < C3_NI; ++ni) {
              br[ni][0] = v0 ? br[ni][0] : 0.0;
              br[ni][1] = v1 ? br[ni][1] : 0.0;
              bi[ni][0] = v0 ? bi[ni][0] : 0.0;
              bi[ni][1] = v1 ? bi[ni][1] : 0.0;
            }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double bs[C3_NI];
#pragma unroll
            for (int ni = 0; ni < C3_NI; ++ni) bs[ni] = br[ni][h] + bi[ni][h];
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) {
              const double as = ar[mi][h] + ai[mi][h];
#pragma unroll
              for (int ni = 0; ni < C3_NI; ++ni) {
                dmma(t1[mi][ni][0], t1[mi][ni][1], ar[mi][h], br[ni][h]);
                dmma(t2[mi][ni][0], t2[mi][ni][1], ai[mi][h], bi[ni][h]);
                dmma(t3[mi][ni][0], t3[mi][ni][1], as, bs[ni]);
              }
            }
          }
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
      // epilogue: Re = T1 - T2, Im = (T3 - T1) - T2; straight to global memory
      if (!upper_only) {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi) {
          const int r = tm * BM + wm * WTM + mi * 8 + arow;
          if (r >= M) continue;
          double *crr = Cr + static_cast<int64_t>(r) * ldc;
          double *cri = Ci + static_cast<int64_t>(r) * ldc;
          RMX_CHECK(!cr_end || (crr + min(N, tn * C3_BN + C3_BN) <= cr_end &&
                                cri + min(N, tn * C3_BN + C3_BN) <= ci_end));
#pragma unroll
          for (int ni = 0; ni < C3_NI; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int c = tn * C3_BN + wn * C3_WTN + ni * 8 + (B_KC ? t + 4 * h : 2 * t + h);
              if (c >= N) continue;
              const double re = t1[mi][ni][h] - t2[mi][ni][h];
              const double im = (t3[mi][ni][h] - t1[mi][ni][h]) - t2[mi][ni][h];
              if (sub) {
                crr[c] -= re;
                cri[c] -= im;
              } else {
                crr[c] = alpha * re;
                cri[c] = alpha * im;
              }
            }
        }
      }
      ++tn;
    }
  }
  __syncthreads();
}

// Complex product into the planes (cr, ci) at (r0, c0): C = alpha (A.B) (set) or C -= A.B (sub).
// The operands of a pair (ar/ai, br/bi) share their layout (k-contiguous or not).
__device__ __forceinline__ void cgemm3(int M, int N, int K, const Op &ar, const Op &ai, const Op &br,
                                       const Op &bi, const MatView &cr, const MatView &ci, int r0, int c0,
                                       bool lower, bool sub, double alpha, int kband, double *smem,
                                       GemmSync *gs) {
  CGemmArgs g{ar, ai, br, bi, cr.at(r0, c0), ci.at(r0, c0), cr.ld, cr.end(), ci.end(), M, N, K, lower,
              sub, kband, alpha};
  uint8_t *s = gemm_smem_align(smem);
  if (ar.kc) {
    if (br.kc)
      cgemm3_impl<true, true>(g, s, gs);
    else
      cgemm3_impl<true, false>(g, s, gs);
  } else {
    if (br.kc)
      cgemm3_impl<false, true>(g, s, gs);
    else
      cgemm3_impl<false, false>(g, s, gs);
  }
}

}  // namespace la
}  // namespace rmx
