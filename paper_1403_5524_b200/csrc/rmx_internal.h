// rmx_internal.h - launcher declarations shared by the librmx translation units (not installed).
#pragma once
#include <cstdint>
#include <functional>
#include <string>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../include/rmx.h"

namespace rmx {

// A matrix inside one workspace slot that the per-energy kernels read with TMA:
// offset (doubles from the slot start), rows, tensor width (columns), leading dimension.
struct MatSpec {
  int64_t off, rows, cols, ld;
};

// Per-slot workspace layouts (doubles) of the matching and T kernels; every matrix start is
// 16-byte aligned and followed by 32 doubles of padding (bulk copies round rows up to 16 bytes).
struct MatchLayout {
  int64_t npad, ldm, m_off, tg_off, sp_off, slot;
};
struct TepiLayout {
  int64_t ldo, ar_off, ai_off, yr_off, yi_off, p_off, d_off, slot;
};
__host__ __device__ inline MatchLayout match_layout(int64_t nch) {
  MatchLayout L;
  L.npad = (nch + 1) & ~1LL;
  L.ldm = 2 * L.npad;  // [A | pad | B_open]
  L.m_off = 0;
  L.tg_off = nch * L.ldm + 32;
  L.sp_off = L.tg_off + 128 * 128 + 32;  // Tg: inverse of a 128 x 128 diagonal block
  L.slot = L.sp_off + ((9 * nch + 1) & ~1LL) + 32;  // LU sub-panel (n x 9) beyond shared memory
  return L;
}
// T epilogue (tepi.cu): five planes [nch][ldo] (Ar, Ai, Yr, Yi, P) and the vectors d (re, im), v
__host__ __device__ inline TepiLayout tepi_layout(int64_t nch) {
  TepiLayout L;
  L.ldo = (nch + 1) & ~1LL;  // even pitch (TMA stride rule)
  const int64_t plane = nch * L.ldo + 32;
  L.ar_off = 0;
  L.ai_off = plane;
  L.yr_off = 2 * plane;
  L.yi_off = 3 * plane;
  L.p_off = 4 * plane;
  L.d_off = 5 * plane;
  L.slot = L.d_off + ((3 * nch + 1) & ~1LL) + 32;
  return L;
}

// One-time per-device initialisation (rmx_api.cu): runs init() once per (key, current device),
// serialised by a mutex; a failed init is retried on the next call. Kernel attributes and
// __constant__ tables are per device, so a process-wide flag would skip them on a second device.
cudaError_t once_per_device(const void *key, const std::function<cudaError_t()> &init);
// cudaFuncAttributeMaxDynamicSharedMemorySize of `func` on the current device, set once
inline cudaError_t ensure_smem_attr(const void *func, size_t bytes) {
  return once_per_device(func, [&] {
    return cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
  });
}

// rform.cu
int rform_tile_for(int64_t nch);
cudaError_t launch_rform(const double *w, int64_t ldw, const double *Ek, int64_t nch, int64_t nlev,
                         double a, const double *E, int64_t ne, double *R, int32_t *status,
                         cudaStream_t st, std::string &err);
// host helper shared with the view tables: encode a 2D FP64 tensor map (box {16, box_rows},
// SWIZZLE_128B, zero fill out of range)
bool encode_tmap_f64(CUtensorMap *map, const double *base, int64_t rows, int64_t cols, int64_t ld,
                     int box_rows, std::string &err);

// rint8.cu: R formation on the INT8 tensor cores by CRT (exact integer arithmetic after a 55/53-bit
// fixed-point rounding of X = W diag(d) and W); ws: rint8_ws_bytes(nch, nlev, chunk) bytes
constexpr int64_t kInt8Chunk = 8;  // minimum energies per INT8 chunk (rint8_chunk may take more)
// below this many channels the 128 x 256 INT8 tiles and the conversion pass do not pay off (measured:
// config small, nch 64: DMMA 3.2e5 E/s vs INT8 1.3e5 E/s; bp, nch 500: INT8 +30 %): R_INT8 falls back
// to the FP64 DMMA kernel
constexpr int64_t kInt8MinChannels = 256;
int64_t rint8_ldv(int64_t nlev);
int64_t rint8_ldr(int64_t nch);
int rint8_max_nlev();
size_t rint8_ws_bytes(int64_t nch, int64_t nlev, int64_t ne);
int64_t rint8_chunk(int64_t nch, int64_t nlev, int64_t ne, int nsm);
struct Int8Streams {  // auxiliary stream + events of the conversion / GEMM pipeline (owned by the ctx)
  cudaStream_t aux = nullptr;
  cudaEvent_t start = nullptr, conv_done[2] = {nullptr, nullptr}, gemm_done[2] = {nullptr, nullptr};
};
cudaError_t launch_rform_int8(const double *w, int64_t ldw, const double *Ek, int64_t nch, int64_t nlev,
                              double a, const double *E, int64_t ne, double *R, int32_t *status, void *ws,
                              size_t ws_bytes, int64_t chunk, const Int8Streams &ss, cudaStream_t st,
                              std::string &err, const std::function<void(bool)> &gemm_mark);

// match.cu
int64_t match_ws_doubles_per_slot(int64_t nch);
void match_view_specs(int64_t nch, std::vector<MatSpec> &specs);
cudaError_t launch_match(const double *R, const double *F, const double *G, const double *Fp,
                         const double *Gp, double a, int64_t nch, int64_t ne, const int32_t *n_open,
                         double *K, double *ws, int64_t ws_slot, const CUtensorMap *views, int64_t ws_slots,
                         int32_t *status, cudaStream_t st, int open_rows_only = 0);

// tepi.cu
// Optional level-pair output of the T epilogue (NEXT-2): omega [ne][nlevel][nlevel] accumulates
// g * sum_{i in a, j in b} |T_ij|^2 over the open levels; level a = channels
// [level_start[a], level_start[a+1]) (DEVICE int32 [nlevel + 1]). omega == nullptr: off.
struct LevelSums {
  const int32_t *level_start = nullptr;
  int nlevel = 0;
  double g = 0.0;
  double *omega = nullptr;
};
// Optional photoionisation output of the T epilogue (NEXT-1, photo.cu header): per energy
//   v_j = (1/2)(g_j F'_j + sum_i g_i G'_i K_ij) (j < o), M = (I - i K_oo)^{-1} v (with the inverse the
//   T route forms), mabs2_j = |M_j|^2, sigma = C (E - E0) sum_j |M_j|^2.
// g == nullptr: off. g, Fp, Gp [ne][nch]; E [ne]; sigma [ne]; mabs2 [ne][nch] or nullptr.
struct PhotoArgs {
  const double *g = nullptr, *Fp = nullptr, *Gp = nullptr, *E = nullptr;
  double E0 = 0.0, C = 0.0;
  double *sigma = nullptr, *mabs2 = nullptr;
};
int64_t tepi_ws_doubles_per_slot(int64_t nch);
void tepi_view_specs(int64_t nch, std::vector<MatSpec> &specs);
cudaError_t launch_tepi(const double *K, int64_t ldk, int64_t kstride, int64_t nch, int64_t ne,
                        const int32_t *n_open, double *T2, const int64_t *t2_slot, double *rowsum,
                        const LevelSums &lv, const PhotoArgs &pa, double *ws, int64_t ws_slot,
                        const CUtensorMap *views, int64_t ws_slots, int32_t *status, cudaStream_t st);
// photo.cu
// part: scratch of part_cap doubles for the split-K partial planes (splits are reduced to fit;
// nullptr: no K split)
int dipole_g_splits(int64_t nch, int64_t nlev, int64_t ne);
cudaError_t launch_dipole_g(const double *w, int64_t ldw, const double *Ek, const double *d,
                            int64_t nch, int64_t nlev, const double *E, int64_t ne, double *g,
                            int32_t *status, double *part, int64_t part_cap, cudaStream_t st);

// post.cu (NEXT-4); the Gaussian window x[i-M, i+256+M) and its weights live in shared memory
constexpr int kMaxConvHalfWidth = 9000;
int conv_window(double dE, double fwhm, double *sigma);
cudaError_t launch_convolve(const double *x, int64_t nspec, const double *mix, int64_t ne,
                            double dE, double fwhm, double *y, cudaStream_t st);  // mix: HOST, <= 64
int64_t maxwell_chunks(int64_t ne);
cudaError_t launch_maxwell(const double *omega, int64_t ne, int64_t npair, const double *E,
                           const double *Eth, const double *kT, int nT, double *part, double *ups,
                           cudaStream_t st);

// largest channel count of the per-energy kernels: up to 2944 channels the LU sub-panels (n x 9
// doubles) are staged in the ~216 KB shared-memory union of the matching kernel, beyond in the
// slot's sub-panel scratch in global memory (L2-resident, ~0.6 MB at 8192); the paper's targets
// reach "in excess of 4,000 channels"
constexpr int64_t kMaxMatchChannels = 8192;
constexpr int64_t kSmemPanelChannels = 2944;

// box rows of the NVIEW tensor-map variants used by the CTA GEMM (cta_la.cuh)
constexpr int kViewBoxRows[3] = {128, 64, 32};

}  // namespace rmx
