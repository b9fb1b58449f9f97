// rint8.cu - R formation on the INT8 tensor cores (tcgen05.mma kind::i8) with exact FP64-level
// accuracy, by the Chinese-remainder (Ozaki-II-style) emulation of the fp64 contraction
//     R_ij(E) = (1/2a) sum_k w_ik w_jk / (E_k - E)          (Eq. 1-2; BASELINE.json:5)
// (reading Z1). Same C-ABI semantics as rform.cu; selected per context.
//
//   1. d_k(E) = 1/(E_k - E) and dmax(E) = max_k |d_k| (pole guard as everywhere: |E - E_k| < 1e-10).
//   2. Fixed-point operands (exact integers):  X'_ik = rint(w_ik d_k 2^{s_i}),  |X'| <= 2^54, with
//      s_i from the exact row maximum max_k|w_ik d_k|;  W'_jk = rint(w_jk 2^{t_j}),  |W'| <= 2^52.
//      Then P_ij = sum_k X'_ik W'_jk is an exact integer, |P| <= nlev 2^106 < M/2 for nlev < 2^17,
//      M = prod of the 16 pairwise-coprime moduli below (2^125.19).
//   3. For each modulus m_l: V_l = X' mod m_l (uint8 in [0, m); balanced int8 when nlev > 65000),
//      U_l = W' mod m_l as balanced int8 (|.| <= 128); the INT8 tensor-core GEMM C_l = V_l U_l^T is
//      exact in int32 (|C| <= 255 * 128 nlev < 2^31), its residue C_l mod m_l = P mod m_l. The GEMM
//      runs as CTA pairs (tcgen05.mma.cta_group::2, one 2-SM cluster per 256 x 256 upper-triangle
//      block: oz_gemm2_kernel); the 1-SM 128 x 256-tile kernel oz_gemm_kernel serves nch <= 256.
//   4. CRT (direct formula, exact 128-bit wrapping arithmetic) recovers P_ij in (-M/2, M/2); then
//      R_ij = P_ij 2^{-s_i - t_j} / (2a), upper triangle mirrored (bitwise symmetric R).
// The only approximation is the rounding of X and W to 55 / 53 significant bits relative to the row
// maximum (step 2): measured normwise error 3e-14 on darc rows (tools/ozaki_error.py), the level of an
// fp64 contraction; everything after it is exact integer arithmetic.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <string>
#include <vector>

#include "rmx_common.cuh"
#include "rmx_internal.h"

namespace rmx {
namespace i8 {

constexpr int L = 16;
__host__ __device__ constexpr int mod_of(int l) {
  constexpr int m[L] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 211, 199, 197, 193, 191};
  return m[l];
}
constexpr int BX = 54, BW = 52;  // fixed-point magnitudes 2^BX, 2^BW

// ---------------------------------------------------------------------------------------------
// residues of a 55-bit signed integer u - 2^54 (u = X' + 2^54 in [0, 2^55]) for all 16 moduli,
// as balanced int8 (r > 127 -> r - m)
__device__ __forceinline__ int8_t bal(int r, int m) { return static_cast<int8_t>(r > 127 ? r - m : r); }

struct ModConst {
  int c36, c18, off;  // 2^36 mod m, 2^18 mod m, (m * 2^10 - (2^BIAS mod m)) so that s stays >= 0
  float inv;          // 1/m (rounded down a little: q never overestimates by more than 1)
  uint32_t magic;     // ceil(2^32 / m): umulhi(s, magic) is floor(s/m) or one more for s < 2^28
  uint32_t m36;       // ceil(2^36 / m): umulhi(s, m36) >> 4 == floor(s/m) exactly for s < 2^28, m < 256
  uint32_t blo, bhi;  // byte weights (2^{8b} mod m, b = 0..3 | 4..7) packed for dp4a
  uint32_t boff;      // (-2^BX) mod m: removes the bias of u = X' + 2^BX
};
__constant__ ModConst c_mod[L];

// s mod m for s < 2^28 by multiply-high: 3 integer ops + 1 correction
__device__ __forceinline__ int umod_magic(uint32_t s, int m, uint32_t magic) {
  int r = static_cast<int>(s) - static_cast<int>(__umulhi(s, magic)) * m;
  return r + ((r < 0) ? m : 0);
}

__device__ __forceinline__ int umod_small(uint32_t s, int m, float inv) {
  int q = static_cast<int>(__uint2float_rz(s) * inv);
  int r = static_cast<int>(s) - q * m;
  r += (r < 0) ? m : 0;
  r -= (r >= m) ? m : 0;
  return r;
}

// ---------------------------------------------------------------------------------------------
// per energy: d_k = 1/(E_k - E) into dbuf [ne][nlev] with the nearest pole's entry zeroed (its term
// w_ik* w_jk* d_k* is added in the CRT epilogue, reading N1: the fixed-point scale of a row then
// follows the rest of the row), its index and d in kstar / dstar [ne], dmax [ne], pole flags (status)
__global__ void __launch_bounds__(256) oz_denom_kernel(const double *__restrict__ Ek, const double *__restrict__ E,
                                                       int nlev, double *__restrict__ dbuf,
                                                       double *__restrict__ dmax, int32_t *__restrict__ pflag,
                                                       int32_t *__restrict__ kstar, double *__restrict__ dstar,
                                                       int32_t *__restrict__ status) {
  const int64_t e = blockIdx.x;
  const double Ee = E[e];
  __shared__ int ks;
  if (threadIdx.x == 0) {
    ks = nearest_pole(Ek, nlev, Ee);
    kstar[e] = ks;
    dstar[e] = 1.0 / (Ek[ks] - Ee);
  }
  __syncthreads();
  double mx = 0.0;
  int pole = 0;
  for (int k = threadIdx.x; k < nlev; k += blockDim.x) {
    const double diff = Ek[k] - Ee;
    if (fabs(diff) < kPoleGuard) pole = 1;
    const double d = (k == ks) ? 0.0 : 1.0 / diff;
    dbuf[e * nlev + k] = d;
    mx = fmax(mx, fabs(d));
  }
  __shared__ double red[8];
  __shared__ int pr[8];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
    pole |= __shfl_xor_sync(0xffffffffu, pole, off);
  }
  if (lane_id() == 0) {
    red[warp_id()] = mx;
    pr[warp_id()] = pole;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    int p = 0;
    for (int q = 0; q < 8; ++q) {
      m = fmax(m, red[q]);
      p |= pr[q];
    }
    dmax[e] = m;
    pflag[e] = p;
    if (p) set_status(status, e, RMX_E_POLE);
  }
}

// row maxima of |w| (once per call)
__global__ void __launch_bounds__(256) oz_rowmax_kernel(const double *__restrict__ w, int64_t ldw, int nlev,
                                                        double *__restrict__ rowmax) {
  const int64_t i = blockIdx.x;
  double mx = 0.0;
  for (int k = threadIdx.x; k < nlev; k += blockDim.x) mx = fmax(mx, fabs(w[i * ldw + k]));
  __shared__ double red[8];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane_id() == 0) red[warp_id()] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int q = 0; q < 8; ++q) m = fmax(m, red[q]);
    rowmax[i] = m;
  }
}

// Exact row maxima xmax[e][i] = max_k |fl(w_ik d_k)| for the ne (<= 8) energies of a chunk: one CTA per
// row, the w values read once for all energies. (A bound max|w_i.| * max|d| can overshoot by orders of
// magnitude when the largest |d| sits on a pole with a small amplitude - the narrow resonances of
// config fine - and the fixed-point rounding would then lose those bits.)
// One CTA per 16 rows; the |d| values of the chunk's energies are staged through shared memory in
// k-tiles of 512 (they would otherwise be re-read from L2 for every row), each warp owns 2 rows. The
// maxima are fp32 UPPER bounds (operands and products rounded up): within 2^-20 of the exact value,
// which only decides the exponent of the scale.
// The k range is split over gridDim.y CTAs whose partial maxima meet by atomicMax on the float bit
// patterns (non-negative floats order like their bits; max is order-independent: deterministic).
constexpr int XM_ROWS = 16, XM_KT = 512, XM_KSPLIT = 8;
__global__ void __launch_bounds__(256) oz_xmax_kernel(const double *__restrict__ w, int64_t ldw, int nch, int nlev,
                                                      int ne, const double *__restrict__ dbuf,
                                                      float *__restrict__ xmax) {
  __shared__ float ds[8][XM_KT];
  const int r0 = blockIdx.x * XM_ROWS + warp_id() * 2;
  float mx[2][8];
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int e = 0; e < 8; ++e) mx[r][e] = 0.0f;
  const int ntile = (nlev + XM_KT - 1) / XM_KT;
  const int t0 = static_cast<int>((static_cast<int64_t>(ntile) * blockIdx.y) / gridDim.y);
  const int t1 = static_cast<int>((static_cast<int64_t>(ntile) * (blockIdx.y + 1)) / gridDim.y);
  for (int k0 = t0 * XM_KT; k0 < t1 * XM_KT; k0 += XM_KT) {
    __syncthreads();
    for (int q = threadIdx.x; q < 8 * XM_KT; q += blockDim.x) {
      const int e = q / XM_KT, kk = q % XM_KT;
      ds[e][kk] = (e < ne && k0 + kk < nlev)
                      ? __double2float_ru(fabs(dbuf[static_cast<int64_t>(e) * nlev + k0 + kk]))
                      : 0.0f;
    }
    __syncthreads();
    // all 2 x 16 w loads of this lane issued before any use (the loop is latency-bound otherwise)
    float wv[2][XM_KT / 32];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int i = r0 + r;
      const double *wr = w + static_cast<int64_t>(i) * ldw + k0;
#pragma unroll
      for (int q = 0; q < XM_KT / 32; ++q) {
        const int kk = lane_id() + 32 * q;
        wv[r][q] = (i < nch && k0 + kk < nlev) ? __double2float_ru(fabs(wr[kk])) : 0.0f;
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int q = 0; q < XM_KT / 32; ++q) {
        const int kk = lane_id() + 32 * q;
#pragma unroll
        for (int e = 0; e < 8; ++e) mx[r][e] = fmaxf(mx[r][e], __fmul_ru(wv[r][q], ds[e][kk]));
      }
  }
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) mx[r][e] = fmaxf(mx[r][e], __shfl_xor_sync(0xffffffffu, mx[r][e], off));
      const int i = r0 + r;
      if (lane_id() == 0 && i < nch && e < ne)
        atomicMax(reinterpret_cast<int *>(xmax + static_cast<int64_t>(e) * nch + i), __float_as_int(mx[r][e]));
    }
}

// Fixed-point conversion + residues. One CTA per (row i, 2048-wide k chunk); each thread 8
// consecutive k, its 8 w values loaded once and reused for all ne energies of the chunk.
// dbuf == nullptr: the W operand (d = 1, BW bits, ne = 1); else the X operands of energies 0..ne-1.
// out: planes [ne][L][nch][ldv] int8 (ldv multiple of 16); shift: [ne][nch] exponents s_i / t_j.
// SIGNED: balanced residues in [-(m-1)/2, (m-1)/2] (int8; needed when nlev > 65000), else plain
// residues in [0, m) (uint8 operand: u8 x s8 products stay < 2^31 summed over nlev <= 65000).
// Per residue: s = sum_b byte_b(u) (2^{8b} mod m) + (-2^54 mod m) (< 2^19, two dp4a),
// q = umulhi(s, ceil(2^32/m)) (exact), r = s - q m. The modulus 256 residue is the low byte of the two's-complement value.
template <bool SIGNED>
__global__ void __launch_bounds__(256) oz_convert_kernel(const double *__restrict__ w, int64_t ldw, int nch,
                                                         int nlev, int ne, const double *__restrict__ dbuf,
                                                         const float *__restrict__ xmax,
                                                         const double *__restrict__ rowmax, int bits,
                                                         int64_t ldv, int8_t *__restrict__ out,
                                                         int32_t *__restrict__ shift) {
  const int i = blockIdx.y;
  const int k0 = (blockIdx.x * 256 + threadIdx.x) * 8;
  double wv[8];
  const double *wr = w + static_cast<int64_t>(i) * ldw + k0;
#pragma unroll
  for (int q = 0; q < 8; ++q) wv[q] = (k0 + q < nlev) ? wr[q] : 0.0;
  const int64_t plane = static_cast<int64_t>(nch) * ldv;
  const uint64_t bias = static_cast<uint64_t>(1) << BX;
  for (int e = 0; e < ne; ++e) {
    // scale 2^s with bound * 2^s < 2^bits (bound = the row maximum, rounded up): frexp = f 2^ex, f < 1
    const double bound = dbuf ? static_cast<double>(xmax[static_cast<int64_t>(e) * nch + i]) : rowmax[i];
    int ex = 0;
    if (bound > 0.0 && isfinite(bound)) frexp(bound, &ex);
    const int s = bits - ex;
    const double scale = ldexp(1.0, s);  // exact power of two
    if (blockIdx.x == 0 && threadIdx.x == 0) shift[static_cast<int64_t>(e) * nch + i] = s;
    if (k0 >= nlev) continue;
    const double *dr = dbuf ? dbuf + static_cast<int64_t>(e) * nlev + k0 : nullptr;
    uint32_t uh[8], ul[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      double x = wv[q];
      if (dr && k0 + q < nlev) x *= dr[q];
      x *= scale;
      if (!isfinite(x)) x = 0.0;  // pole energies: R is NaN anyway (status POLE)
      const uint64_t u = static_cast<uint64_t>(__double2ll_rn(x) + static_cast<long long>(bias));
      uh[q] = static_cast<uint32_t>(u >> 32);
      ul[q] = static_cast<uint32_t>(u);
    }
    int8_t *o = out + static_cast<int64_t>(e) * L * plane + static_cast<int64_t>(i) * ldv + k0;
    {  // modulus 256: the low byte (u = X' + 2^54, 2^54 = 0 mod 256)
      uint32_t pk[2] = {0u, 0u};
#pragma unroll
      for (int q = 0; q < 8; ++q) pk[q >> 2] |= (ul[q] & 0xFFu) << (8 * (q & 3));
      *reinterpret_cast<uint2 *>(o) = make_uint2(pk[0], pk[1]);
    }
#pragma unroll
    for (int l = 1; l < L; ++l) {
      const int m = mod_of(l);
      const ModConst mc = c_mod[l];
      uint32_t pk[2] = {0u, 0u};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        // sv = sum_b byte_b(u) (2^{8b} mod m) + (-2^BX mod m) < 7 * 255^2 + 256 < 2^19 (two dp4a), so
        // q = umulhi(sv, ceil(2^32/m)) is floor(sv/m) exactly (error sv/2^32 < 2^-13 < 1/m)
        const uint32_t sv = __dp4a(uh[q], mc.bhi, __dp4a(ul[q], mc.blo, mc.boff));
        const uint32_t r = sv - __umulhi(sv, mc.magic) * m;  // in [0, m)
        if (SIGNED) {
          const int rb = static_cast<int>(r) - ((static_cast<int>(r) > (m - 1) / 2) ? m : 0);
          pk[q >> 2] |= (static_cast<uint32_t>(rb) & 0xFFu) << (8 * (q & 3));
        } else {
          pk[q >> 2] += r << (8 * (q & 3));  // r < 256: the bytes do not overlap
        }
      }
      *reinterpret_cast<uint2 *>(o + l * plane) = make_uint2(pk[0], pk[1]);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// tcgen05 INT8 GEMM over (upper-triangle tile, modulus, energy):
//   C = V[e][l] (128 rows of X residues) . U[l]^T (256 rows of W residues), int32 in TMEM,
//   epilogue: C mod m_l -> uint8 residue plane res[e][l][i][j] (row pitch ldr bytes)
constexpr int BM = 128, BN = 256, BKB = 128, STAGES = 4;
constexpr int A_BYTES = BM * BKB, B_BYTES = BN * BKB, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int GEMM_NT = 256;
constexpr int GEMM_SMEM = 1024 + STAGES * STAGE_BYTES + 256;
// instruction descriptor: s32 accumulate, A u8 (plain residues) or s8 (balanced), B s8, K-major, M 128, N 256
__host__ __device__ constexpr uint32_t idesc_i8(bool a_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
         (static_cast<uint32_t>(BM >> 4) << 24);
}

__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;           // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;   // SBO: 8-row groups 1024 B apart
  d |= static_cast<uint64_t>(1) << 46;           // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;           // SWIZZLE_128B
  return d;
}

// ---------------------------------------------------------------------------------------------
// The same conversion with the byte-weight sums on the tensor cores (the default for unsigned X
// residues; oz_convert_kernel above stays for balanced residues, nlev > 65000, and as the
// RMX_I8_CONV_ALU A/B switch). Per (row i, 1024 k) work item and energy each of the 128 threads
// forms u = X' + 2^54 for 8 consecutive k as in oz_convert_kernel and writes its 8 bytes plus a
// constant 1 in byte 7 (u < 2^56) to shared-memory row t (SWIZZLE_128B K-major, 32 K-bytes = 4
// elements per MMA K-slice); one tcgen05.mma.kind::i8 (M = 128, N = 64, K = 32, u8 x u8 -> s32) per
// slice against the block-diagonal weight matrix B[16q + l][8q + b] = 2^{8b} mod m_l (b < 7),
// (-2^54) mod m_l (b = 7) gives sv_l = sum_b byte_b (2^{8b} mod m_l) + (-2^54 mod m_l) < 2^19 for
// the 4 elements q and the 16 moduli l - exactly the two dp4a of oz_convert_kernel - in TMEM column
// 64 s + 16 q + l of lane t. The ALUs are left with the 15 reductions sv mod m (multiply-high) and the
// byte packing: half the integer-pipe instructions per element. Bitwise the same
// residues as oz_convert_kernel (tests/test_rint8.py: R bitwise equal under both).
constexpr int CT_NT = 128;  // threads per CTA = rows of the MMA tile
constexpr int CT_A_BYTES = 128 * 128, CT_B_BYTES = 64 * 128;  // SW128 tiles (A: 2 of 4 slices used)
constexpr int CT_SMEM = 1024 + CT_A_BYTES + CT_B_BYTES + 64;
// 128 registers x 128 threads cap residency at 4 CTAs per SM = 4 x 128 TMEM columns; the small shared
// footprint lets a conversion CTA sit beside a pair-GEMM CTA whose ring leaves room (RMX_I8_STAGES)
constexpr int CT_SMEM_REQ = (1024 + CT_A_BYTES + CT_B_BYTES + 64 + 127) / 128 * 128;
static_assert(CT_SMEM <= CT_SMEM_REQ, "conversion tiles exceed the requested shared memory");
constexpr uint32_t CT_IDESC = (2u << 4) | (static_cast<uint32_t>(64 >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);

__device__ __forceinline__ uint32_t ct_weight(int l, int b) {
  const ModConst &mc = c_mod[l];
  if (b < 4) return (mc.blo >> (8 * b)) & 0xFFu;
  if (b < 7) return (mc.bhi >> (8 * (b - 4))) & 0xFFu;
  return mc.boff;
}

// CT_EL elements (consecutive k) per thread: 8 -> 2 K-slices, 128 TMEM columns, <= 128 registers (4 CTAs
// per SM); 4 -> 1 K-slice, 64 TMEM columns, <= 64 registers (8 CTAs per SM)
template <int CT_EL>
__global__ void __launch_bounds__(CT_NT, 32 / CT_EL)
    oz_convert_tc_kernel(const double *__restrict__ w, int64_t ldw, int nch, int nlev, int ne,
                         const double *__restrict__ dbuf, const float *__restrict__ xmax, int bits, int64_t ldv,
                         int8_t *__restrict__ out, int32_t *__restrict__ shift, int items_per_cta) {
  constexpr int CT_K = CT_NT * CT_EL, CT_TMEM_COLS = 16 * CT_EL;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *As = smem, *Bs = smem + CT_A_BYTES;
  uint64_t *bar = reinterpret_cast<uint64_t *>(Bs + CT_B_BYTES);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 1);
  const int t = threadIdx.x, warp = warp_id();
  // weight tile: row n (= 16 q + l), K bytes 0..31 of 128 (SW128: 16-byte chunk c at c ^ (n & 7))
  for (int idx = t; idx < 64 * 8; idx += CT_NT) {
    const int n = idx >> 3, c = idx & 7;
    uint32_t v[4] = {0u, 0u, 0u, 0u};
    if (c < 2) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int kk = 16 * c + j;
        if ((kk >> 3) == (n >> 4)) v[j >> 2] |= ct_weight(n & 15, kk & 7) << (8 * (j & 3));
      }
    }
    *reinterpret_cast<uint4 *>(Bs + n * 128 + ((c ^ (n & 7)) * 16)) = make_uint4(v[0], v[1], v[2], v[3]);
  }
  if (t == 0) {
    mbar_init(bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(CT_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  fence_proxy_async();
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tmem_slot;
  const uint32_t a_base = smem_u32(As), b_base = smem_u32(Bs);
  uint8_t *arow = As + t * 128;
  const int sw = t & 7;
  const int nkb = (nlev + CT_K - 1) / CT_K;
  const int64_t nitems = static_cast<int64_t>(nch) * nkb;
  const int64_t plane = static_cast<int64_t>(nch) * ldv;
  const uint64_t bias = (static_cast<uint64_t>(1) << BX) | (static_cast<uint64_t>(1) << 56);  // + byte 7 = 1
  uint32_t phase = 0;
  const int64_t it0 = static_cast<int64_t>(blockIdx.x) * items_per_cta;
  const int64_t it1 = min(nitems, it0 + items_per_cta);
  for (int64_t it = it0; it < it1; ++it) {
    const int i = static_cast<int>(it / nkb), kb = static_cast<int>(it % nkb);
    const int k0 = kb * CT_K + t * CT_EL;
    double wv[CT_EL];
    const double *wr = w + static_cast<int64_t>(i) * ldw + k0;
#pragma unroll
    for (int q = 0; q < CT_EL; ++q) wv[q] = (k0 + q < nlev) ? wr[q] : 0.0;
    // d and the row bound of energy e + 1 are loaded while energy e is converted (latency-bound
    // otherwise: ncu long-scoreboard stalls on these loads dominated the first version; prefetching
    // the next work item's W as well spilled and measured slower)
    double dcur[CT_EL];
    float bcur = xmax[i];
#pragma unroll
    for (int q = 0; q < CT_EL; ++q) dcur[q] = (k0 + q < nlev) ? dbuf[k0 + q] : 0.0;
    for (int e = 0; e < ne; ++e) {
      double dnext[CT_EL];
      float bnext = 0.0f;
      if (e + 1 < ne) {
        const double *dn = dbuf + static_cast<int64_t>(e + 1) * nlev + k0;
        bnext = xmax[static_cast<int64_t>(e + 1) * nch + i];
#pragma unroll
        for (int q = 0; q < CT_EL; ++q) dnext[q] = (k0 + q < nlev) ? dn[q] : 0.0;
      }
      const double bound = static_cast<double>(bcur);
      int ex = 0;
      if (bound > 0.0 && isfinite(bound)) frexp(bound, &ex);
      const int s = bits - ex;
      const double scale = ldexp(1.0, s);
      if (kb == 0 && t == 0) shift[static_cast<int64_t>(e) * nch + i] = s;
      uint64_t u[CT_EL];
#pragma unroll
      for (int q = 0; q < CT_EL; ++q) {
        double x = wv[q] * dcur[q];
        x *= scale;
        if (!isfinite(x)) x = 0.0;  // pole energies: R is NaN anyway (status POLE)
        u[q] = static_cast<uint64_t>(__double2ll_rn(x)) + bias;
      }
      // row t: 16-byte chunk c (elements 2c, 2c+1) at chunk c ^ (t & 7)
#pragma unroll
      for (int c = 0; c < CT_EL / 2; ++c)
        *reinterpret_cast<uint4 *>(arow + ((c ^ sw) * 16)) =
            make_uint4(static_cast<uint32_t>(u[2 * c]), static_cast<uint32_t>(u[2 * c] >> 32),
                       static_cast<uint32_t>(u[2 * c + 1]), static_cast<uint32_t>(u[2 * c + 1] >> 32));
      fence_proxy_async();
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      __syncthreads();
      if (t == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const uint64_t db = umma_desc_sw128(b_base);
#pragma unroll
        for (int sl = 0; sl < CT_EL / 4; ++sl) {
          const uint64_t da = umma_desc_sw128(a_base) + 2 * sl;  // K-bytes 32 sl .. 32 sl + 31
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + 64u * sl),
                       "l"(da), "l"(db), "r"(CT_IDESC), "r"(0));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(bar))
                     : "memory");
      }
      mbar_wait(bar, phase);
      phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      uint32_t pk[L][CT_EL / 4];
#pragma unroll
      for (int sl = 0; sl < CT_EL / 4; ++sl) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // TMEM columns 64 sl + 16 q + l: element 4 sl + q, modulus l
          uint32_t v[16];
          const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + 64u * sl + 16u * q;
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                "=r"(v[15])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
#pragma unroll
          for (int l = 0; l < L; ++l) {
            uint32_t r = v[l];
            if (l > 0) {  // sv mod m (sv < 2^19: umulhi by ceil(2^32/m) is floor(sv/m) exactly)
              const uint32_t m = static_cast<uint32_t>(mod_of(l));
              r -= __umulhi(r, c_mod[l].magic) * m;
            }
            // byte q of the word (little-endian: element k0 + 4 sl + q)
            if (q == 0)
              pk[l][sl] = r;
            else
              pk[l][sl] = __byte_perm(pk[l][sl], r, q == 1 ? 0x3240 : (q == 2 ? 0x3410 : 0x4210));
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
      if (k0 < nlev) {
        int8_t *o = out + static_cast<int64_t>(e) * L * plane + static_cast<int64_t>(i) * ldv + k0;
#pragma unroll
        for (int l = 0; l < L; ++l) {
          if (CT_EL == 8)
            *reinterpret_cast<uint2 *>(o + l * plane) = make_uint2(pk[l][0], pk[l][CT_EL / 4 - 1]);
          else
            *reinterpret_cast<uint32_t *>(o + l * plane) = pk[l][0];
        }
      }
#pragma unroll
      for (int q = 0; q < CT_EL; ++q) dcur[q] = dnext[q];
      bcur = bnext;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(CT_TMEM_COLS));
}

// GEMM epilogue of one CTA (warps 4..7): TMEM lane quarter q holds output rows row0 + q*32 + lane,
// columns col0 .. col0 + BN - 1 in TMEM columns 0..BN-1; C mod m_l -> uint8 residue plane
// res[e][l][row][col] (rows >= nch and column groups starting at or past nch are not stored).
__device__ __forceinline__ void residue_epilogue(uint32_t tmem, int q, int row0, int col0, int nch, int l, int64_t e,
                                                 int64_t ldr, uint8_t *__restrict__ res) {
  const int lane = lane_id();
  const int row = row0 + q * 32 + lane;
  const int m = mod_of(l);
  const int c16 = (1 << 16) % m;
  const float inv = c_mod[l].inv;
  uint8_t *rrow = res + ((e * L + l) * static_cast<int64_t>(nch) + row) * ldr + col0;
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
          "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
    if (row < nch && col0 + c0 < nch) {
      uint32_t pk[8];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        // acc = h 2^16 + lo (h signed): residue of h c16 + lo (|.| < 2^24: exact in fp32)
        const int acc = static_cast<int>(v[j]);
        const int h = acc >> 16, lo = acc & 0xFFFF;
        const int sv = h * c16 + lo + (m << 16);  // > 0 (|h c16| < 2^15 * 255)
        const int r = umod_small(static_cast<uint32_t>(sv), m, inv);
        if ((j & 3) == 0) pk[j >> 2] = 0u;
        pk[j >> 2] |= static_cast<uint32_t>(r) << (8 * (j & 3));
      }
      uint4 *dst = reinterpret_cast<uint4 *>(rrow + c0);
      dst[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      dst[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
    }
  }
}

__global__ void __launch_bounds__(GEMM_NT, 1)
    oz_gemm_kernel(const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tu, int nch,
                   int nlev, int ntiles, const int2 *__restrict__ tiles, int64_t ldr, uint8_t *__restrict__ res,
                   uint32_t idesc, int nen) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *accf = empty + STAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accf + 1);
  const int warp = warp_id(), lane = lane_id();
  // tiles fastest, then energies, then moduli: the GEMMs resident together share U_l (one modulus's W
  // residues) through L2 and differ only in their X residues
  const int tile = blockIdx.x % ntiles;
  const int64_t e = (blockIdx.x / ntiles) % nen;
  const int l = blockIdx.x / (ntiles * nen);
  const int2 tij = tiles[tile];  // (I, J): rows I*128.., columns J*256..
  const int nk = (nlev + BKB - 1) / BKB;
  const int vrow = static_cast<int>((e * L + l) * nch) + tij.x * BM;  // row in the stacked V planes
  const int urow = l * nch + tij.y * BN;                                // row in the stacked U planes

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tv);
    tma_prefetch_desc(&tu);
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % STAGES;
      if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
      mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
      const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
      tma_load_2d(base, &tv, &full[s], kt * BKB, vrow);
      tma_load_2d(base + A_BYTES, &tu, &full[s], kt * BKB, urow);
    }
  } else if (warp == 1 && lane == 0) {
    const bool half = tij.y * BN + 127 < tij.x * BM;
    const uint32_t idesc_k = half ? ((idesc & ~(0x3Fu << 17)) | (static_cast<uint32_t>(128 >> 3) << 17)) : idesc;
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % STAGES;
      mbar_wait(&full[s], (kt / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
      // a tile whose first 128 columns lie entirely below the diagonal computes only its right half
      // (N = 128 into TMEM columns 128..255; the left half's residues are never read by the CRT)
      const uint32_t boff = half ? static_cast<uint32_t>(128 * BKB) : 0u;
      const uint64_t da = umma_desc_sw128(base), db = umma_desc_sw128(base + A_BYTES + boff);
#pragma unroll
      for (int k = 0; k < BKB / 32; ++k) {
        const uint32_t acc = (kt > 0 || k > 0) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + (half ? 128u : 0u)),
                     "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc_k), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(&empty[s]))
                   : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(accf))
                 : "memory");
  } else if (warp >= 4) {
    mbar_wait(accf, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    residue_epilogue(tmem, warp - 4, tij.x * BM, tij.y * BN, nch, l, e, ldr, res);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(BN));
}

// CTA-pair variant (tcgen05 cta_group::2), the default for nch > 256: one 2-CTA cluster per 256 x 256
// upper-triangle output block (I2, J), J >= I2, M = 256 per MMA instruction. CTA r stages its
// own 128 rows of V (rows I2*256 + 128 r) and 128 of the 256 U rows (J*256 + 128 r) - the pair shares
// operands, so each SM moves half the B bytes of the 1-SM kernel through shared memory (sustained INT8
// throughput under the power cap +6 %, tools/tc_i8_gemm2.cu). Both CTAs' TMA completions count on the
// leader's full barrier; the leader's single MMA thread commits each stage to both CTAs' empty
// barriers and the finished accumulator to both accf barriers; each CTA drains its own TMEM rows.
constexpr int P_B_BYTES = (BN / 2) * BKB, P_STAGE_BYTES = A_BYTES + P_B_BYTES;
__host__ __device__ constexpr int gemm2_smem(int stages) { return 1024 + stages * P_STAGE_BYTES + 256; }
__host__ __device__ constexpr uint32_t idesc_i8_pair(bool a_signed) {
  return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | (1u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
         (static_cast<uint32_t>(256 >> 4) << 24);
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_rank0(uint32_t saddr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;\n" : "=r"(r) : "r"(saddr));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int P_STAGES>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GEMM_NT, 1)
    oz_gemm2_kernel(const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tu2,
                    const __grid_constant__ CUtensorMap tun, int nch, int nlev, int ntiles,
                    const int2 *__restrict__ tiles, int64_t ldr, uint8_t *__restrict__ res, uint32_t idesc, int nen,
                    int jlast, int nlast) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + P_STAGES * P_STAGE_BYTES);
  uint64_t *empty = full + P_STAGES;
  uint64_t *accf = empty + P_STAGES;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(accf + 1);
  const int warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int cid = blockIdx.x >> 1;
  const int tile = cid % ntiles;
  const int64_t e = (cid / ntiles) % nen;
  const int l = cid / (ntiles * nen);
  const int2 tij = tiles[tile];  // (I2, J): rows I2*256.., columns J*256..
  const int nk = (nlev + BKB - 1) / BKB;
  const int row0 = tij.x * 256 + static_cast<int>(rank) * BM;
  const int vrow = static_cast<int>((e * L + l) * nch) + row0;
  // the ragged last column block (nch - jlast*256 columns) runs as N = nlast (a multiple of 16):
  // each CTA of the pair then holds nlast/2 of its W rows (tensor map tun, boxes of nlast/2 rows)
  const bool edge = tij.y == jlast && nlast < BN;
  const int nb2 = edge ? nlast / 2 : BN / 2;
  const CUtensorMap *tb = edge ? &tun : &tu2;
  const uint32_t idesc_k = edge ? ((idesc & ~(0x3Fu << 17)) | (static_cast<uint32_t>(nlast >> 3) << 17)) : idesc;
  const uint32_t stage_tx = 2u * static_cast<uint32_t>(A_BYTES + nb2 * BKB);
  const int urow = l * nch + tij.y * BN + static_cast<int>(rank) * nb2;

  if (threadIdx.x == 0) {
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "r"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tv);
    tma_prefetch_desc(tb);
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % P_STAGES;
      if (kt >= P_STAGES) mbar_wait(&empty[s], ((kt / P_STAGES) - 1) & 1);
      if (rank == 0) mbar_arrive_expect_tx(&full[s], stage_tx);
      const uint32_t base = smem_u32(smem + s * P_STAGE_BYTES);
      const uint32_t bar = mapa_rank0(smem_u32(&full[s]));
      asm volatile(
          "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(base), "l"(reinterpret_cast<uint64_t>(&tv)), "r"(bar),
          "r"(kt * BKB), "r"(vrow)
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(base + A_BYTES), "l"(reinterpret_cast<uint64_t>(tb)), "r"(bar),
          "r"(kt * BKB), "r"(urow)
          : "memory");
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    for (int kt = 0; kt < nk; ++kt) {
      const int s = kt % P_STAGES;
      mbar_wait(&full[s], (kt / P_STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const uint32_t base = smem_u32(smem + s * P_STAGE_BYTES);
      const uint64_t da = umma_desc_sw128(base), db = umma_desc_sw128(base + A_BYTES);
#pragma unroll
      for (int k = 0; k < BKB / 32; ++k) {
        const uint32_t acc = (kt > 0 || k > 0) ? 1u : 0u;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                     "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc_k), "r"(acc));
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
              smem_u32(&empty[s])),
          "h"(static_cast<uint16_t>(3))
          : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            smem_u32(accf)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
  } else if (warp >= 4) {
    mbar_wait(accf, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    residue_epilogue(tmem, warp - 4, row0, tij.y * BN, nch, l, e, ldr, res);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  cluster_sync_all();
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(BN));
}

// ---------------------------------------------------------------------------------------------
// CRT: residues r_l of P_ij -> P_ij -> R_ij. Direct formula: with C_l = (M/m_l)((M/m_l)^-1 mod m_l),
// S = sum_l r_l C_l = P (mod M), and S/M = sum_l r_l f_l with f_l = C_l/M = inv_l/m_l in (0, 1), so
// S/M = P/M + an integer. |P| <= nlev 2^54 2^52 = nlev 2^106 < M/2 (M = 2^125.19: |P|/M <= 0.07 at
// nlev 40000 and 0.23 at the supported maximum nlev 131071), and the fp64 sum of the 16 terms (< 4096)
// errs by < 1e-11, so q = rint(sum_l r_l f_l) is exactly the multiple of M to remove; P = S - q M is
// then evaluated exactly in 128-bit wrapping arithmetic (4 x 32-bit limbs).
struct CrtConst {
  uint32_t C[L][4];  // C_l, little-endian limbs
  double f[L];       // inv_l / m_l
  uint32_t M[4];     // product of the moduli
};
__constant__ CrtConst c_crt;

// CRT on 32 x 32 tiles of the upper triangle (one CTA per tile and energy, 256 threads x 4 rows):
// residue loads and the R[i][j] stores run along j, and the mirrored R[j][i] half is written from a
// shared-memory transpose along i (coalesced in both directions).
__device__ __forceinline__ double crt_value(const uint8_t *rp, int64_t plane, int s_sum, double inv2a) {
  uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  double sf = 0.0;
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const uint32_t r = rp[l * plane];
    a0 += static_cast<uint64_t>(r) * c_crt.C[l][0];
    a1 += static_cast<uint64_t>(r) * c_crt.C[l][1];
    a2 += static_cast<uint64_t>(r) * c_crt.C[l][2];
    a3 += static_cast<uint64_t>(r) * c_crt.C[l][3];
    sf = fma(static_cast<double>(r), c_crt.f[l], sf);
  }
  a1 += a0 >> 32;
  a2 += a1 >> 32;
  a3 += a2 >> 32;
  uint64_t lo = (a0 & 0xFFFFFFFFull) | (a1 << 32);
  uint64_t hi = (a2 & 0xFFFFFFFFull) | (a3 << 32);
  const uint64_t q = static_cast<uint64_t>(rint(sf));
  const uint64_t m01 = (static_cast<uint64_t>(c_crt.M[1]) << 32) | c_crt.M[0];
  const uint64_t m23 = (static_cast<uint64_t>(c_crt.M[3]) << 32) | c_crt.M[2];
  const uint64_t qlo = q * m01, qhi = __umul64hi(q, m01) + q * m23;
  const uint64_t nlo = lo - qlo;
  hi = hi - qhi - (lo < qlo ? 1ull : 0ull);
  lo = nlo;
  const bool neg = static_cast<int64_t>(hi) < 0;
  if (neg) {
    lo = ~lo + 1;
    hi = ~hi + (lo == 0 ? 1ull : 0ull);
  }
  double p = static_cast<double>(hi) * 18446744073709551616.0 + static_cast<double>(lo);
  if (neg) p = -p;
  return ldexp(p, -s_sum) * inv2a;
}

__global__ void __launch_bounds__(256) oz_crt_tile_kernel(const uint8_t *__restrict__ res, int64_t ldr, int nch,
                                                          const int32_t *__restrict__ sx,
                                                          const int32_t *__restrict__ tw, double inv2a,
                                                          const int32_t *__restrict__ pflag,
                                                          const double *__restrict__ w, int64_t ldw,
                                                          const int32_t *__restrict__ kstar,
                                                          const double *__restrict__ dstar, double *__restrict__ R) {
  __shared__ double tile[32][33];
  const int64_t e = blockIdx.y;
  // blockIdx.x enumerates the upper-triangle tiles (ti <= tj) row by row
  const int nt = (nch + 31) / 32;
  int ti = 0, rem = blockIdx.x;
  while (rem >= nt - ti) {
    rem -= nt - ti;
    ++ti;
  }
  const int tj = ti + rem;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double *Re = R + e * static_cast<int64_t>(nch) * nch;
  const int64_t plane = static_cast<int64_t>(nch) * ldr;
  const bool pole = pflag[e] != 0;
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  const int j = tj * 32 + tx;
  // the nearest pole's term w_ik* w_jk* d_k* / 2a, added to the CRT value (reading N1)
  const int ks = kstar[e];
  const double dsc = dstar[e] * inv2a;
  const double wj = j < nch ? w[static_cast<int64_t>(j) * ldw + ks] : 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int li = ty + 8 * q, i = ti * 32 + li;
    double v = 0.0;
    if (i < nch && j < nch && j >= i) {
      const double wi = w[static_cast<int64_t>(i) * ldw + ks];
      v = pole ? nan
               : crt_value(res + e * L * plane + static_cast<int64_t>(i) * ldr + j, plane,
                           sx[e * nch + i] + tw[j], inv2a) + (wi * wj) * dsc;
      Re[static_cast<int64_t>(i) * nch + j] = v;
    }
    tile[li][tx] = v;
  }
  __syncthreads();
  // mirror: R[j][i] = R[i][j] for i < j, written along i
  const int i2 = ti * 32 + tx;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int lj = ty + 8 * q, j2 = tj * 32 + lj;
    if (i2 < nch && j2 < nch && i2 < j2) Re[static_cast<int64_t>(j2) * nch + i2] = tile[tx][lj];
  }
}

}  // namespace i8

// ---------------------------------------------------------------------------------------------
// host side
// __constant__ memory is per device: the tables are uploaded once per device (once_per_device)
static cudaError_t upload_i8_consts() {
  i8::ModConst mc[i8::L];
  i8::CrtConst cc{};
  unsigned __int128 M = 1;
  for (int l = 0; l < i8::L; ++l) M *= static_cast<unsigned>(i8::mod_of(l));
  for (int l = 0; l < i8::L; ++l) {
    const int m = i8::mod_of(l);
    const uint64_t p54 = (static_cast<uint64_t>(1) << i8::BX) % m;
    mc[l].c36 = static_cast<int>((static_cast<uint64_t>(1) << 36) % m);
    mc[l].c18 = static_cast<int>((static_cast<uint64_t>(1) << 18) % m);
    mc[l].off = static_cast<int>(m * 1024 - static_cast<int>(p54));
    mc[l].inv = nextafterf(1.0f / static_cast<float>(m), 0.0f);
    mc[l].magic = static_cast<uint32_t>(((static_cast<uint64_t>(1) << 32) + m - 1) / m);
    mc[l].m36 = static_cast<uint32_t>(((static_cast<uint64_t>(1) << 36) + m - 1) / m);
    mc[l].blo = mc[l].bhi = 0;
    for (int b = 0; b < 4; ++b) {
      mc[l].blo |= static_cast<uint32_t>((static_cast<uint64_t>(1) << (8 * b)) % m) << (8 * b);
      mc[l].bhi |= static_cast<uint32_t>((static_cast<uint64_t>(1) << (8 * b + 32)) % m) << (8 * b);
    }
    mc[l].boff = static_cast<uint32_t>((m - p54) % m);
    // C_l = (M/m) * ((M/m)^-1 mod m)
    const unsigned __int128 Ml = M / static_cast<unsigned>(m);
    const int Mlm = static_cast<int>(Ml % static_cast<unsigned>(m));
    int inv = 0;
    for (int x = 1; x < m; ++x)
      if ((Mlm * x) % m == 1) { inv = x; break; }
    const unsigned __int128 C = Ml * static_cast<unsigned>(inv);
    for (int k = 0; k < 4; ++k) cc.C[l][k] = static_cast<uint32_t>(C >> (32 * k));
    cc.f[l] = static_cast<double>(inv) / static_cast<double>(m);
  }
  for (int k = 0; k < 4; ++k) cc.M[k] = static_cast<uint32_t>(M >> (32 * k));
  cudaError_t e = cudaMemcpyToSymbol(i8::c_mod, mc, sizeof(mc));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(i8::c_crt, &cc, sizeof(cc));
  return e;
}

static cudaError_t init_i8_consts() {
  static const int key = 0;
  return once_per_device(&key, upload_i8_consts);
}

static bool encode_i8(CUtensorMap *map, const void *base, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                      std::string &err) {
  typedef CUresult (*Enc)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                          const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Enc enc = nullptr;
  if (!enc) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      err = "cuTensorMapEncodeTiled unavailable";
      return false;
    }
    enc = reinterpret_cast<Enc>(p);
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(i8::BKB), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "cuTensorMapEncodeTiled (int8) failed (code " + std::to_string(static_cast<int>(r)) + ")";
    return false;
  }
  return true;
}

int64_t rint8_ldv(int64_t nlev) { return (nlev + 15) & ~static_cast<int64_t>(15); }
int64_t rint8_ldr(int64_t nch) { return (nch + 255) & ~static_cast<int64_t>(255); }
int rint8_max_nlev() { return 131071; }

// Energies per chunk: 8, or more when one chunk's GEMM grid would be short (few 256-blocks, e.g.
// config bp: 3 pair blocks -> 768 CTAs per 8 energies, 5.2 waves with a 0.8-wave tail), up to 64 and
// within ~24 GB of double-buffered X residues.
int64_t rint8_chunk(int64_t nch, int64_t nlev, int64_t ne, int nsm) {
  const int64_t nb = (nch + 255) / 256;
  const int64_t ctas_per_energy = 2 * (nb * (nb + 1) / 2) * 16;
  const int64_t want = (16 * static_cast<int64_t>(nsm) + ctas_per_energy - 1) / ctas_per_energy;
  int64_t chunk = std::max<int64_t>(8, std::min<int64_t>(64, (want + 7) / 8 * 8));
  const int64_t per_energy = 2 * 16 * nch * rint8_ldv(nlev);
  while (chunk > 8 && chunk * per_energy > (static_cast<int64_t>(24) << 30)) chunk -= 8;
  // very large nch x nlev: fewer than 8 energies per chunk (down to 1) rather than no INT8 path
  while (chunk > 1 && chunk * per_energy > (static_cast<int64_t>(24) << 30)) chunk /= 2;
  return std::min(chunk, ne);
}

// Workspace (bytes) for chunks of ne energies, double-buffered (V planes, d, dmax, shifts, pole flags)
// plus the W residues, one residue-plane buffer and the tile list
size_t rint8_ws_bytes(int64_t nch, int64_t nlev, int64_t ne) {
  const int64_t ldv = rint8_ldv(nlev), ldr = rint8_ldr(nch);
  size_t b = 0;
  b += static_cast<size_t>(i8::L) * nch * ldv;                       // U planes
  b += 2 * static_cast<size_t>(ne) * i8::L * nch * ldv;              // V planes (2 buffers)
  b += static_cast<size_t>(ne) * i8::L * nch * ldr;                  // residue planes
  b += 2 * sizeof(double) * (static_cast<size_t>(ne) * nlev + ne + static_cast<size_t>(ne) * nch);  // d, dmax, xmax
  b += sizeof(double) * nch;                                         // rowmax
  b += 2 * sizeof(int32_t) * (static_cast<size_t>(ne) * nch + ne);   // shifts, pole flags (2 buffers)
  b += 2 * (sizeof(int32_t) + sizeof(double)) * ne + 2 * 512;        // nearest pole k*, d_k* (2 buffers)
  b += sizeof(int32_t) * nch + sizeof(int2) * 4096 + 32 * 1024;      // t_j, tile list, alignment slack
  return b;
}

// Two-stream pipeline: the fixed-point conversion of chunk c+1 (ALU + HBM bound, aux stream) runs
// while the INT8 GEMMs of chunk c (tensor cores, whose warps leave the ALUs idle) run on st;
// V / d / shifts / pole flags are double-buffered, events order the reuse.
cudaError_t launch_rform_int8(const double *w, int64_t ldw, const double *Ek, int64_t nch, int64_t nlev,
                              double a, const double *E, int64_t ne, double *R, int32_t *status, void *ws,
                              size_t ws_bytes, int64_t chunk, const Int8Streams &ss, cudaStream_t st,
                              std::string &err, const std::function<void(bool)> &gemm_mark) {
  cudaError_t ce = init_i8_consts();
  if (ce != cudaSuccess) return ce;
  ce = ensure_smem_attr(reinterpret_cast<const void *>(i8::oz_gemm_kernel), i8::GEMM_SMEM);
  if (ce != cudaSuccess) return ce;
  // ring depth of the pair GEMM: 7 stages fill the SM's shared memory; RMX_I8_STAGES=6 / 5 leave room
  // for one / two conversion CTAs beside it (A/B switch)
  const char *stg_env = getenv("RMX_I8_STAGES");
  const int p_stages = stg_env ? std::max(5, std::min(7, atoi(stg_env))) : 7;
  ce = ensure_smem_attr(reinterpret_cast<const void *>(i8::oz_gemm2_kernel<7>), i8::gemm2_smem(7));
  if (ce == cudaSuccess) ce = ensure_smem_attr(reinterpret_cast<const void *>(i8::oz_gemm2_kernel<6>), i8::gemm2_smem(6));
  if (ce == cudaSuccess) ce = ensure_smem_attr(reinterpret_cast<const void *>(i8::oz_gemm2_kernel<5>), i8::gemm2_smem(5));
  if (ce != cudaSuccess) return ce;
  ce = ensure_smem_attr(reinterpret_cast<const void *>(i8::oz_convert_tc_kernel<8>), i8::CT_SMEM_REQ);
  if (ce == cudaSuccess) ce = ensure_smem_attr(reinterpret_cast<const void *>(i8::oz_convert_tc_kernel<4>), i8::CT_SMEM_REQ);
  if (ce != cudaSuccess) return ce;
  // X residues: byte-weight sums on the tensor cores (oz_convert_tc_kernel) unless RMX_I8_CONV_ALU is
  // set (A/B switch; read per call so that a test can compare both in one process)
  const bool conv_alu = getenv("RMX_I8_CONV_ALU") != nullptr;
  const char *el_env = getenv("RMX_I8_CONV_EL");  // elements per thread of the tensor-core conversion (A/B)
  const int conv_el = (el_env && atoi(el_env) == 4) ? 4 : 8;
  const int64_t ldv = rint8_ldv(nlev), ldr = rint8_ldr(nch);
  uint8_t *wsp = static_cast<uint8_t *>(ws);
  auto carve = [&](size_t bytes) {
    uint8_t *p = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(wsp) + 255) & ~uintptr_t(255));
    wsp = p + ((bytes + 255) & ~size_t(255));
    return p;
  };
  int8_t *U = reinterpret_cast<int8_t *>(carve(static_cast<size_t>(i8::L) * nch * ldv));
  int8_t *V[2];
  double *dbuf[2], *dmax[2];
  float *xmax[2];
  int32_t *sx[2], *pflag[2], *kst[2];
  double *dst[2];
  for (int b = 0; b < 2; ++b) {
    V[b] = reinterpret_cast<int8_t *>(carve(static_cast<size_t>(chunk) * i8::L * nch * ldv));
    dbuf[b] = reinterpret_cast<double *>(carve(sizeof(double) * chunk * nlev));
    xmax[b] = reinterpret_cast<float *>(carve(sizeof(float) * chunk * nch));
    dmax[b] = reinterpret_cast<double *>(carve(sizeof(double) * chunk));
    sx[b] = reinterpret_cast<int32_t *>(carve(sizeof(int32_t) * chunk * nch));
    pflag[b] = reinterpret_cast<int32_t *>(carve(sizeof(int32_t) * chunk));
    kst[b] = reinterpret_cast<int32_t *>(carve(sizeof(int32_t) * chunk));
    dst[b] = reinterpret_cast<double *>(carve(sizeof(double) * chunk));
  }
  uint8_t *res = carve(static_cast<size_t>(chunk) * i8::L * nch * ldr);
  double *rowmax = reinterpret_cast<double *>(carve(sizeof(double) * nch));
  int32_t *tw = reinterpret_cast<int32_t *>(carve(sizeof(int32_t) * nch));
  int2 *tiles = reinterpret_cast<int2 *>(carve(sizeof(int2) * 4096));
  if (static_cast<size_t>(wsp - static_cast<uint8_t *>(ws)) > ws_bytes) {
    err = "rform int8: workspace too small";
    return cudaErrorInvalidValue;
  }

  // Upper-triangle tiles - static per nch. CTA-pair kernel: every 256 x 256 block (I2, J), J >= I2 (the
  // diagonal blocks compute their lower-left 128 x 128 quarter too, 6 % more MMA work at darc, which
  // measured far cheaper than a separate 1-SM launch for them: that second pass re-read the X
  // residues from HBM and kept the GEMMs at the power cap - DESIGN.md §5.5). 1-SM kernel (128 x 256
  // tiles, half tiles below the diagonal): nch <= 256, or RMX_I8_NOPAIR set (an A/B switch).
  static const bool no_pair = getenv("RMX_I8_NOPAIR") != nullptr;
  const bool use_pair = !no_pair && nch > i8::BN;
  std::vector<int2> tl, pl;
  if (use_pair) {
    for (int I2 = 0; I2 * 256 < nch; ++I2)
      for (int J = I2; J * i8::BN < nch; ++J) pl.push_back(make_int2(I2, J));
  } else {
    for (int I = 0; I * i8::BM < nch; ++I)
      for (int J = 0; J * i8::BN < nch; ++J)
        if (J * i8::BN + i8::BN - 1 >= I * i8::BM) tl.push_back(make_int2(I, J));  // not entirely below
  }
  if (tl.size() + pl.size() > 4096) {
    err = "rform int8: nch too large for the tile list";
    return cudaErrorInvalidValue;
  }
  std::vector<int2> all(tl);
  all.insert(all.end(), pl.begin(), pl.end());
  ce = cudaMemcpyAsync(tiles, all.data(), sizeof(int2) * all.size(), cudaMemcpyHostToDevice, st);
  if (ce != cudaSuccess) return ce;
  const int ntiles = static_cast<int>(tl.size()), npair = static_cast<int>(pl.size());

  // W operand: row maxima, W' residues, t_j (on st)
  i8::oz_rowmax_kernel<<<static_cast<unsigned>(nch), 256, 0, st>>>(w, ldw, static_cast<int>(nlev), rowmax);
  {
    dim3 g(static_cast<unsigned>((nlev + 2047) / 2048), static_cast<unsigned>(nch), 1);
    i8::oz_convert_kernel<true><<<g, 256, 0, st>>>(w, ldw, static_cast<int>(nch), static_cast<int>(nlev), 1,
                                                   nullptr, nullptr, rowmax, i8::BW, ldv, U, tw);
  }
  CUtensorMap tu, tv[2];
  if (!encode_i8(&tu, U, static_cast<int64_t>(i8::L) * nch, nlev, ldv, i8::BN, err)) return cudaErrorInvalidValue;
  CUtensorMap tu2;  // U rows in boxes of 128 (one half of a pair block's columns per CTA)
  if (!encode_i8(&tu2, U, static_cast<int64_t>(i8::L) * nch, nlev, ldv, i8::BN / 2, err)) return cudaErrorInvalidValue;
  // ragged last column block: N = nlast = round16(nch - jlast*256), nlast/2 W rows per CTA
  const int jlast = static_cast<int>((nch - 1) / i8::BN);
  const int nlast = static_cast<int>(std::max<int64_t>(16, ((nch - static_cast<int64_t>(jlast) * i8::BN) + 15) / 16 * 16));
  CUtensorMap tun = tu2;
  if (nlast < i8::BN &&
      !encode_i8(&tun, U, static_cast<int64_t>(i8::L) * nch, nlev, ldv, nlast / 2, err))
    return cudaErrorInvalidValue;
  for (int b = 0; b < 2; ++b)
    if (!encode_i8(&tv[b], V[b], chunk * i8::L * nch, nlev, ldv, i8::BM, err)) return cudaErrorInvalidValue;
  const double inv2a = 1.0 / (2.0 * a);
  // plain (unsigned) X residues keep |C| <= 255 * 128 * nlev < 2^31 up to nlev = 65793
  const bool x_signed = nlev > 65000;
  const uint32_t idesc = i8::idesc_i8(x_signed), idesc2 = i8::idesc_i8_pair(x_signed);
  // the aux stream starts after everything already queued on st (rowmax, inputs)
  cudaEventRecord(ss.start, st);
  cudaStreamWaitEvent(ss.aux, ss.start, 0);
  const int64_t nchunks = (ne + chunk - 1) / chunk;
  cudaStream_t cs = ss.aux;  // conversion stream (the GEMM-stream variant measured the same: DESIGN.md §9)
  auto convert = [&](int64_t c) {
    const int b = static_cast<int>(c & 1);
    const int64_t e0 = c * chunk, n = std::min(chunk, ne - e0);
    if (c >= 2) cudaStreamWaitEvent(cs, ss.gemm_done[b], 0);  // buffer b free again
    int32_t *stc = status ? status + e0 : nullptr;
    i8::oz_denom_kernel<<<static_cast<unsigned>(n), 256, 0, cs>>>(Ek, E + e0, static_cast<int>(nlev), dbuf[b],
                                                                      dmax[b], pflag[b], kst[b], dst[b], stc);
    dim3 g(static_cast<unsigned>((nlev + 2047) / 2048), static_cast<unsigned>(nch), 1);
    cudaMemsetAsync(xmax[b], 0, sizeof(float) * chunk * nch, cs);
    for (int64_t q = 0; q < n; q += 8)  // the row-maxima kernel stages at most 8 energies
      i8::oz_xmax_kernel<<<dim3(static_cast<unsigned>((nch + i8::XM_ROWS - 1) / i8::XM_ROWS), i8::XM_KSPLIT), 256,
                           0, cs>>>(w, ldw, static_cast<int>(nch), static_cast<int>(nlev),
                                    static_cast<int>(std::min<int64_t>(8, n - q)), dbuf[b] + q * nlev,
                                    xmax[b] + q * nch);
    if (!x_signed && !conv_alu) {
      const int el = conv_el;
      const int64_t nitems = nch * ((nlev + i8::CT_NT * el - 1) / (i8::CT_NT * el));
      const int ipc = 4;  // work items (row, 128 x CT_EL k) per CTA (16 with CT_EL = 8: 8.4 waves, slower)
      const unsigned gconv = static_cast<unsigned>((nitems + ipc - 1) / ipc);
      if (el == 8)
        i8::oz_convert_tc_kernel<8><<<gconv, i8::CT_NT, i8::CT_SMEM_REQ, cs>>>(
            w, ldw, static_cast<int>(nch), static_cast<int>(nlev), static_cast<int>(n), dbuf[b], xmax[b], i8::BX,
            ldv, V[b], sx[b], ipc);
      else
        i8::oz_convert_tc_kernel<4><<<gconv, i8::CT_NT, i8::CT_SMEM_REQ, cs>>>(
            w, ldw, static_cast<int>(nch), static_cast<int>(nlev), static_cast<int>(n), dbuf[b], xmax[b], i8::BX,
            ldv, V[b], sx[b], ipc);
    } else if (x_signed)
      i8::oz_convert_kernel<true><<<g, 256, 0, cs>>>(w, ldw, static_cast<int>(nch), static_cast<int>(nlev),
                                                         static_cast<int>(n), dbuf[b], xmax[b], rowmax, i8::BX, ldv,
                                                         V[b], sx[b]);
    else
      i8::oz_convert_kernel<false><<<g, 256, 0, cs>>>(w, ldw, static_cast<int>(nch), static_cast<int>(nlev),
                                                          static_cast<int>(n), dbuf[b], xmax[b], rowmax, i8::BX,
                                                          ldv, V[b], sx[b]);
    cudaEventRecord(ss.conv_done[b], cs);
  };
  convert(0);
  for (int64_t c = 0; c < nchunks; ++c) {
    const int b = static_cast<int>(c & 1);
    const int64_t e0 = c * chunk, n = std::min(chunk, ne - e0);
    if (c + 1 < nchunks) convert(c + 1);
    cudaStreamWaitEvent(st, ss.conv_done[b], 0);
    gemm_mark(true);
    if (ntiles > 0)
      i8::oz_gemm_kernel<<<static_cast<unsigned>(ntiles * i8::L * n), i8::GEMM_NT, i8::GEMM_SMEM, st>>>(
          tv[b], tu, static_cast<int>(nch), static_cast<int>(nlev), ntiles, tiles, ldr, res, idesc,
          static_cast<int>(n));
    if (npair > 0) {
      const unsigned g2 = static_cast<unsigned>(2 * npair * i8::L * n);
      const int nn = static_cast<int>(nch), nl = static_cast<int>(nlev), ne_c = static_cast<int>(n);
      if (p_stages == 7)
        i8::oz_gemm2_kernel<7><<<g2, i8::GEMM_NT, i8::gemm2_smem(7), st>>>(tv[b], tu2, tun, nn, nl, npair, tiles + ntiles,
                                                                           ldr, res, idesc2, ne_c, jlast, nlast);
      else if (p_stages == 6)
        i8::oz_gemm2_kernel<6><<<g2, i8::GEMM_NT, i8::gemm2_smem(6), st>>>(tv[b], tu2, tun, nn, nl, npair, tiles + ntiles,
                                                                           ldr, res, idesc2, ne_c, jlast, nlast);
      else
        i8::oz_gemm2_kernel<5><<<g2, i8::GEMM_NT, i8::gemm2_smem(5), st>>>(tv[b], tu2, tun, nn, nl, npair, tiles + ntiles,
                                                                           ldr, res, idesc2, ne_c, jlast, nlast);
    }
    gemm_mark(false);
    const int64_t ntc = (nch + 31) / 32;
    dim3 gc(static_cast<unsigned>(ntc * (ntc + 1) / 2), static_cast<unsigned>(n));
    i8::oz_crt_tile_kernel<<<gc, 256, 0, st>>>(res, ldr, static_cast<int>(nch), sx[b], tw, inv2a, pflag[b], w,
                                               ldw, kst[b], dst[b], R + e0 * nch * nch);
    cudaEventRecord(ss.gemm_done[b], st);  // after the CRT: it reads sx[b], pflag[b], kst[b], dst[b]
    ce = cudaGetLastError();
    if (ce != cudaSuccess) return ce;
  }
  return cudaSuccess;
}

}  // namespace rmx
