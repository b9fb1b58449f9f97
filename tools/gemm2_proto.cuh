// gemm2_proto.cuh - EXPERIMENT (tools only, not in librmx): an 8-warp variant of the per-CTA DMMA
// GEMM of cta_la.cuh with 128 x 128 CTA tiles and 64 x 32 warp tiles. Without the TMA-producer warp
// the CTA has 8 warps = 2 per SMSP, so each thread may use up to 255 registers (the 9-warp design is
// capped at 168 by the per-SMSP register file), which pays for 64 accumulators per lane; the larger
// tile halves the HBM/L2 bytes per flop of the streamed operand. Thread 0 issues the TMA loads
// (rotating refill, STAGES - 1 slices ahead). C = A.B only, K % 32 == 0, full tiles (bench shapes).
// Measured against la::gemm_set by tools/gemm_bench.cu (mode 2).
#pragma once
#include "../paper_1403_5524_b200/csrc/cta_la.cuh"

namespace rmx {
namespace proto {

constexpr int NT2 = 256, NW2 = 8;
constexpr int BM2 = 128, BN2 = 128, BK2 = 32, WM2 = 2, WN2 = 4;
constexpr int WTM2 = BM2 / WM2, WTN2 = BN2 / WN2;  // 64 x 32
constexpr int MI2 = WTM2 / 8, NI2 = WTN2 / 8;       // 8 x 4 DMMA fragments
constexpr int ST2 = 3;
constexpr int A2_BYTES = BM2 * BK2 * 8, B2_BYTES = BN2 * BK2 * 8, STAGE2 = A2_BYTES + B2_BYTES;
constexpr int SMEM2 = 1024 + ST2 * STAGE2 + 256;

struct Sync2 {
  uint64_t full[ST2], empty[ST2];
};

// views: index 0 = {16, 128} boxes (k-contiguous rows), 2 = {16, 32} boxes (m/n-contiguous, 32 k rows)
template <bool A_KC, bool B_KC>
__device__ __forceinline__ void gemm2_set(int M, int N, int K, const la::Op &a, const la::Op &b, double *C, int64_t ldc,
                          uint8_t *smem_al, Sync2 *sy) {
  const int warp = warp_id(), lane = lane_id();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST2; ++s) {
      mbar_init(&sy->full[s], 1);
      mbar_init(&sy->empty[s], NW2);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int tiles_m = M / BM2, tiles_n = N / BN2, nkc = K / BK2;
  const int total = tiles_m * tiles_n * nkc;  // flattened (tile, kc) slices, kc fastest
  const CUtensorMap *tmA = a.v.tm + (A_KC ? 0 : 2);
  const CUtensorMap *tmB = b.v.tm + (B_KC ? 0 : 2);
  auto load = [&](int sl) {  // thread 0 only
    const int st = sl % ST2;
    const int kc = sl % nkc, tile = sl / nkc, tm = tile / tiles_n, tn = tile % tiles_n;
    const int k0 = kc * BK2;
    uint64_t *bar = &sy->full[st];
    mbar_arrive_expect_tx(bar, STAGE2);
    const uint32_t sa = smem_u32(smem_al + st * STAGE2), sb = sa + A2_BYTES;
    if (A_KC) {
#pragma unroll
      for (int q = 0; q < 2; ++q) tma_load_2d(sa + q * (BM2 * 128), tmA, bar, a.c0 + k0 + 16 * q, a.r0 + tm * BM2);
    } else {
#pragma unroll
      for (int q = 0; q < BM2 / 16; ++q) tma_load_2d(sa + q * (BK2 * 128), tmA, bar, a.c0 + tm * BM2 + 16 * q, a.r0 + k0);
    }
    if (B_KC) {
#pragma unroll
      for (int q = 0; q < 2; ++q) tma_load_2d(sb + q * (BN2 * 128), tmB, bar, b.c0 + k0 + 16 * q, b.r0 + tn * BN2);
    } else {
#pragma unroll
      for (int q = 0; q < BN2 / 16; ++q) tma_load_2d(sb + q * (BK2 * 128), tmB, bar, b.c0 + tn * BN2 + 16 * q, b.r0 + k0);
    }
  };
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async;\n" ::: "memory");
    for (int sl = 0; sl < ST2 && sl < total; ++sl) load(sl);
  }
  const int wm = warp % WM2, wn = warp / WM2;
  const int g = lane >> 2, t = lane & 3;
  const int pg = la::frag_perm(g);
  uint32_t aoff[MI2][2], boff[NI2][2];
#pragma unroll
  for (int mi = 0; mi < MI2; ++mi) {
    if (A_KC) {
      const int r = wm * WTM2 + mi * 8 + pg;
      aoff[mi][0] = r * 128 + ((t ^ pg) << 4);
      aoff[mi][1] = r * 128 + (((4 + t) ^ pg) << 4);
    } else {
      const int m = wm * WTM2 + mi * 8 + g, j2 = (m & 15) >> 1;
      const uint32_t base = (m >> 4) * (BK2 * 128) + ((m & 1) << 3);
      aoff[mi][0] = base + (2 * t) * 128 + ((j2 ^ (2 * t)) << 4);
      aoff[mi][1] = base + (2 * t + 1) * 128 + ((j2 ^ (2 * t + 1)) << 4);
    }
  }
#pragma unroll
  for (int ni = 0; ni < NI2; ++ni) {
    if (B_KC) {
      const int r = wn * WTN2 + ni * 8 + pg;
      boff[ni][0] = r * 128 + ((t ^ pg) << 4);
      boff[ni][1] = r * 128 + (((4 + t) ^ pg) << 4);
    } else {
      const int n = wn * WTN2 + ni * 8 + g, j2 = (n & 15) >> 1;
      const uint32_t base = (n >> 4) * (BK2 * 128) + ((n & 1) << 3);
      boff[ni][0] = base + (2 * t) * 128 + ((j2 ^ (2 * t)) << 4);
      boff[ni][1] = base + (2 * t + 1) * 128 + ((j2 ^ (2 * t + 1)) << 4);
    }
  }
  const int arow = A_KC ? pg : g;
  const uint32_t smem0 = smem_u32(smem_al);
  double acc[MI2][NI2][2];
  int it = 0;
  for (int tile = 0; tile < tiles_m * tiles_n; ++tile) {
    const int tm = tile / tiles_n, tn = tile % tiles_n;
#pragma unroll
    for (int mi = 0; mi < MI2; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI2; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
    for (int kc = 0; kc < nkc; ++kc, ++it) {
      const int st = it % ST2;
      // rotating refill: thread 0 reloads the stage released by the previous slice
      if (threadIdx.x == 0 && it >= 1 && it - 1 + ST2 < total) {
        const int ps = (it - 1) % ST2;
        mbar_wait(&sy->empty[ps], ((it - 1) / ST2) & 1);
        load(it - 1 + ST2);
      }
      mbar_wait(&sy->full[st], (it / ST2) & 1);
      const uint32_t sa = smem0 + st * STAGE2, sb = sa + A2_BYTES;
#pragma unroll
      for (int k8 = 0; k8 < BK2 / 8; ++k8) {
        double af[MI2][2], bf[NI2][2];
#pragma unroll
        for (int mi = 0; mi < MI2; ++mi) {
          if (A_KC) {
            lds128(af[mi][0], af[mi][1], sa + (k8 >> 1) * (BM2 * 128) + aoff[mi][k8 & 1]);
          } else {
            af[mi][0] = lds64(sa + k8 * 1024 + aoff[mi][0]);
            af[mi][1] = lds64(sa + k8 * 1024 + aoff[mi][1]);
          }
        }
#pragma unroll
        for (int ni = 0; ni < NI2; ++ni) {
          if (B_KC) {
            lds128(bf[ni][0], bf[ni][1], sb + (k8 >> 1) * (BN2 * 128) + boff[ni][k8 & 1]);
          } else {
            bf[ni][0] = lds64(sb + k8 * 1024 + boff[ni][0]);
            bf[ni][1] = lds64(sb + k8 * 1024 + boff[ni][1]);
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int mi = 0; mi < MI2; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi][h], bf[ni][h]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sy->empty[st]);
    }
#pragma unroll
    for (int mi = 0; mi < MI2; ++mi) {
      const int r = tm * BM2 + wm * WTM2 + mi * 8 + arow;
      double *crow = C + static_cast<int64_t>(r) * ldc;
#pragma unroll
      for (int ni = 0; ni < NI2; ++ni)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = tn * BN2 + wn * WTN2 + ni * 8 + (B_KC ? t + 4 * h : 2 * t + h);
          crow[c] = acc[mi][ni][h];
        }
    }
  }
  __syncthreads();
}

// the same behind a non-inlined call (as la::gemm_impl is called): isolates the call-ABI cost
template <bool A_KC, bool B_KC>
static __device__ __noinline__ void gemm2_set_call(const la::GemmArgs &ga, uint8_t *smem_al, Sync2 *sy) {
  const la::GemmArgs g = ga;
  gemm2_set<A_KC, B_KC>(g.M, g.N, g.K, g.a, g.b, g.C, g.ldc, smem_al, sy);
}

// Full-featured variant (what cta_la needs): lower-triangle tile sets, k bands, partial M/N/K,
// C read (C -= A.B / C += A.B) into registers, transposed store, diag_add. Load cursor in registers.
template <bool A_KC, bool B_KC>
__device__ __forceinline__ void gemm3(const la::GemmArgs &gar, uint8_t *smem_al, Sync2 *sy) {
  const la::GemmArgs ga = gar;
  const int M = ga.M, N = ga.N, K = ga.K;
  const bool lower = ga.lower, readC = ga.read_c, addC = ga.add_c;
  const int warp = warp_id(), lane = lane_id();
  __syncthreads();
  if (M <= 0 || N <= 0 || K <= 0) return;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST2; ++s) {
      mbar_init(&sy->full[s], 1);
      mbar_init(&sy->empty[s], NW2);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int tiles_m = la::cdiv(M, BM2), tiles_n = la::cdiv(N, BN2), nkc = la::cdiv(K, BK2);
  auto row_tiles = [&](int tm) {
    if (!lower) return tiles_n;
    return min(tiles_n, (tm * BM2 + BM2 - 1) / BN2 + 1);
  };
  auto kfirst = [&](int tm, int tn) {
    return ga.kband == 1 ? (tm * BM2) / BK2 : (ga.kband == 2 ? (tn * BN2) / BK2 : 0);
  };
  int ntiles = 0;
  for (int tm = 0; tm < tiles_m; ++tm) ntiles += row_tiles(tm);
  const CUtensorMap *tmA = ga.a.v.tm + (A_KC ? 0 : 2);
  const CUtensorMap *tmB = ga.b.v.tm + (B_KC ? 0 : 2);
  // load cursor (used by thread 0)
  int ctile = 0, ctm = 0, ctn = 0, crc = row_tiles(0), ckc = kfirst(0, 0), lit = 0;
  auto settle = [&]() {
    while (ctile < ntiles && ckc >= nkc) {
      if (++ctile >= ntiles) break;
      if (++ctn == crc) {
        ctn = 0;
        crc = row_tiles(++ctm);
      }
      ckc = kfirst(ctm, ctn);
    }
  };
  auto load_next = [&]() {
    const int st = lit % ST2;
    const int k0 = ckc * BK2;
    uint64_t *bar = &sy->full[st];
    mbar_arrive_expect_tx(bar, STAGE2);
    const uint32_t sa = smem_u32(smem_al + st * STAGE2), sb = sa + A2_BYTES;
    if (A_KC) {
#pragma unroll
      for (int q = 0; q < 2; ++q) tma_load_2d(sa + q * (BM2 * 128), tmA, bar, ga.a.c0 + k0 + 16 * q, ga.a.r0 + ctm * BM2);
    } else {
#pragma unroll
      for (int q = 0; q < BM2 / 16; ++q) tma_load_2d(sa + q * (BK2 * 128), tmA, bar, ga.a.c0 + ctm * BM2 + 16 * q, ga.a.r0 + k0);
    }
    if (B_KC) {
#pragma unroll
      for (int q = 0; q < 2; ++q) tma_load_2d(sb + q * (BN2 * 128), tmB, bar, ga.b.c0 + k0 + 16 * q, ga.b.r0 + ctn * BN2);
    } else {
#pragma unroll
      for (int q = 0; q < BN2 / 16; ++q) tma_load_2d(sb + q * (BK2 * 128), tmB, bar, ga.b.c0 + ctn * BN2 + 16 * q, ga.b.r0 + k0);
    }
    ++lit;
    ++ckc;
    settle();
  };
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async;\n" ::: "memory");
    settle();
    for (int q = 0; q < ST2 && ctile < ntiles; ++q) load_next();
  }
  const int wm = warp % WM2, wn = warp / WM2;
  const int g = lane >> 2, t = lane & 3;
  const int pg = la::frag_perm(g);
  uint32_t aoff[MI2][2], boff[NI2][2];
#pragma unroll
  for (int mi = 0; mi < MI2; ++mi) {
    if (A_KC) {
      const int r = wm * WTM2 + mi * 8 + pg;
      aoff[mi][0] = r * 128 + ((t ^ pg) << 4);
      aoff[mi][1] = r * 128 + (((4 + t) ^ pg) << 4);
    } else {
      const int m = wm * WTM2 + mi * 8 + g, j2 = (m & 15) >> 1;
      const uint32_t base = (m >> 4) * (BK2 * 128) + ((m & 1) << 3);
      aoff[mi][0] = base + (2 * t) * 128 + ((j2 ^ (2 * t)) << 4);
      aoff[mi][1] = base + (2 * t + 1) * 128 + ((j2 ^ (2 * t + 1)) << 4);
    }
  }
#pragma unroll
  for (int ni = 0; ni < NI2; ++ni) {
    if (B_KC) {
      const int r = wn * WTN2 + ni * 8 + pg;
      boff[ni][0] = r * 128 + ((t ^ pg) << 4);
      boff[ni][1] = r * 128 + (((4 + t) ^ pg) << 4);
    } else {
      const int n = wn * WTN2 + ni * 8 + g, j2 = (n & 15) >> 1;
      const uint32_t base = (n >> 4) * (BK2 * 128) + ((n & 1) << 3);
      boff[ni][0] = base + (2 * t) * 128 + ((j2 ^ (2 * t)) << 4);
      boff[ni][1] = base + (2 * t + 1) * 128 + ((j2 ^ (2 * t + 1)) << 4);
    }
  }
  const int arow = A_KC ? pg : g;
  const uint32_t smem0 = smem_u32(smem_al);
  double acc[MI2][NI2][2];
  int it = 0, tm = 0, tn = 0, rowcnt = row_tiles(0);
  for (int tile = 0; tile < ntiles; ++tile) {
    if (tn == rowcnt) {
      tn = 0;
      rowcnt = row_tiles(++tm);
    }
    const bool cfull = (tm + 1) * BM2 <= M && (tn + 1) * BN2 <= N;
    if (readC && cfull) {
      const double sgn = addC ? 1.0 : -1.0;
#pragma unroll
      for (int mi = 0; mi < MI2; ++mi) {
        const int r = tm * BM2 + wm * WTM2 + mi * 8 + arow;
        const double *crow = ga.C + static_cast<int64_t>(r) * ga.ldc + tn * BN2 + wn * WTN2;
#pragma unroll
        for (int ni = 0; ni < NI2; ++ni) {
          if (B_KC) {
            acc[mi][ni][0] = sgn * crow[ni * 8 + t];
            acc[mi][ni][1] = sgn * crow[ni * 8 + t + 4];
          } else {
            const double2 v = *reinterpret_cast<const double2 *>(crow + ni * 8 + 2 * t);
            acc[mi][ni][0] = sgn * v.x;
            acc[mi][ni][1] = sgn * v.y;
          }
        }
      }
    } else
#pragma unroll
    for (int mi = 0; mi < MI2; ++mi) {
      const int r = tm * BM2 + wm * WTM2 + mi * 8 + arow;
      const double *crow = ga.C + static_cast<int64_t>(r) * ga.ldc;
#pragma unroll
      for (int ni = 0; ni < NI2; ++ni) {
        double c0 = 0.0, c1 = 0.0;
        if (readC && r < M) {
          const int cb = tn * BN2 + wn * WTN2 + ni * 8;
          if (B_KC) {
            if (cb + t < N) c0 = crow[cb + t];
            if (cb + t + 4 < N) c1 = crow[cb + t + 4];
          } else if (cb + 2 * t + 1 < N) {
            const double2 v = *reinterpret_cast<const double2 *>(crow + cb + 2 * t);
            c0 = v.x;
            c1 = v.y;
          } else if (cb + 2 * t < N) {
            c0 = crow[cb + 2 * t];
          }
        }
        acc[mi][ni][0] = addC ? c0 : -c0;
        acc[mi][ni][1] = addC ? c1 : -c1;
      }
    }
    for (int kc = kfirst(tm, tn); kc < nkc; ++kc, ++it) {
      const int st = it % ST2;
      if (threadIdx.x == 0 && it >= 1 && ctile < ntiles) {
        mbar_wait(&sy->empty[(it - 1) % ST2], ((it - 1) / ST2) & 1);
        load_next();
      }
      mbar_wait(&sy->full[st], (it / ST2) & 1);
      const int krem = min(BK2, K - kc * BK2);
      const uint32_t sa = smem0 + st * STAGE2, sb = sa + A2_BYTES;
      auto step = [&](const int k8, const bool partial) {
        double af[MI2][2], bf[NI2][2];
#pragma unroll
        for (int mi = 0; mi < MI2; ++mi) {
          if (A_KC) {
            lds128(af[mi][0], af[mi][1], sa + (k8 >> 1) * (BM2 * 128) + aoff[mi][k8 & 1]);
          } else {
            af[mi][0] = lds64(sa + k8 * 1024 + aoff[mi][0]);
            af[mi][1] = lds64(sa + k8 * 1024 + aoff[mi][1]);
          }
        }
#pragma unroll
        for (int ni = 0; ni < NI2; ++ni) {
          if (B_KC) {
            lds128(bf[ni][0], bf[ni][1], sb + (k8 >> 1) * (BN2 * 128) + boff[ni][k8 & 1]);
          } else {
            bf[ni][0] = lds64(sb + k8 * 1024 + boff[ni][0]);
            bf[ni][1] = lds64(sb + k8 * 1024 + boff[ni][1]);
          }
        }
        if (partial) {
          const int k = k8 * 8 + 2 * t;
          const bool v0 = k < krem, v1 = k + 1 < krem;
#pragma unroll
          for (int mi = 0; mi < MI2; ++mi) {
            af[mi][0] = v0 ? af[mi][0] : 0.0;
            af[mi][1] = v1 ? af[mi][1] : 0.0;
          }
#pragma unroll
          for (int ni = 0; ni < NI2; ++ni) {
            bf[ni][0] = v0 ? bf[ni][0] : 0.0;
            bf[ni][1] = v1 ? bf[ni][1] : 0.0;
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int mi = 0; mi < MI2; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI2; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi][h], bf[ni][h]);
      };
      if (krem == BK2) {
#pragma unroll
        for (int k8 = 0; k8 < BK2 / 8; ++k8) step(k8, false);
      } else {
#pragma unroll 1
        for (int k8 = 0; k8 * 8 < krem; ++k8) step(k8, true);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sy->empty[st]);
    }
    // epilogue: one branch per tile; interior tiles (no edge, no diagonal term) store unconditionally
    const bool interior = (tm + 1) * BM2 <= M && (tn + 1) * BN2 <= N && !ga.trans_c &&
                          (readC || ga.diag_add == 0.0 || tm * BM2 >= (tn + 1) * BN2 || tn * BN2 >= (tm + 1) * BM2);
    if (interior) {
      const double sgn = (readC && !addC) ? -1.0 : 1.0;
#pragma unroll
      for (int mi = 0; mi < MI2; ++mi) {
        const int r = tm * BM2 + wm * WTM2 + mi * 8 + arow;
        double *crow = ga.C + static_cast<int64_t>(r) * ga.ldc + tn * BN2 + wn * WTN2;
#pragma unroll
        for (int ni = 0; ni < NI2; ++ni) {
          if (B_KC) {
            crow[ni * 8 + t] = sgn * acc[mi][ni][0];
            crow[ni * 8 + t + 4] = sgn * acc[mi][ni][1];
          } else {
            *reinterpret_cast<double2 *>(crow + ni * 8 + 2 * t) = make_double2(sgn * acc[mi][ni][0], sgn * acc[mi][ni][1]);
          }
        }
      }
    } else {
#pragma unroll
      for (int mi = 0; mi < MI2; ++mi) {
        const int r = tm * BM2 + wm * WTM2 + mi * 8 + arow;
        if (r >= M) continue;
        double *crow = ga.C + static_cast<int64_t>(r) * ga.ldc;
#pragma unroll
        for (int ni = 0; ni < NI2; ++ni)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int c = tn * BN2 + wn * WTN2 + ni * 8 + (B_KC ? t + 4 * h : 2 * t + h);
            if (c >= N) continue;
            if (readC)
              crow[c] = addC ? acc[mi][ni][h] : -acc[mi][ni][h];
            else if (ga.trans_c)
              ga.C[static_cast<int64_t>(c) * ga.ldc + r] = acc[mi][ni][h];
            else
              crow[c] = acc[mi][ni][h] + (r == c ? ga.diag_add : 0.0);
          }
      }
    }
    ++tn;
  }
  __syncthreads();
}
template <bool A_KC, bool B_KC>
static __device__ __noinline__ void gemm3_call(const la::GemmArgs &ga, uint8_t *smem_al, Sync2 *sy) {
  gemm3<A_KC, B_KC>(ga, smem_al, sy);
}

}  // namespace proto
}  // namespace rmx
