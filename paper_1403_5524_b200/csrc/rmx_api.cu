// rmx_api.cu - the C ABI of librmx (include/rmx.h): context, argument validation, workspace,
// the streaming sweep driver and launch instrumentation. All arithmetic of the method lives in
// rform.cu / match.cu / tepi.cu; this file only validates, allocates and launches.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include <cublas_v2.h>
#include <cusolverDn.h>

#include "rmx_internal.h"

using namespace rmx;

cudaError_t rmx::once_per_device(const void *key, const std::function<cudaError_t()> &init) {
  static std::mutex mu;
  static std::set<std::pair<const void *, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({key, dev})) return cudaSuccess;
  e = init();
  if (e == cudaSuccess) done.insert({key, dev});
  return e;
}

struct PendingTiming {
  int kid;
  cudaEvent_t a, b;
};

struct rmx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int nsm = 148;
  std::string err;
  cudaError_t sticky = cudaSuccess;
  // linear-algebra workspace (match / tepi slots)
  double *ws = nullptr;
  size_t ws_bytes = 0;
  // TMA descriptor tables of the workspace slots (device memory), rebuilt when ws / nch change
  CUtensorMap *match_views = nullptr, *tepi_views = nullptr;
  int64_t views_nch = -1, views_slots = -1;
  const double *views_ws = nullptr;
  // sweep batch buffer (R, then K in place)
  double *rbuf = nullptr;
  size_t rbuf_bytes = 0;
  // device mirrors for rmx_sweep_host
  struct Dev {
    void *p = nullptr;
    size_t bytes = 0;
  } dw, dEk, dE, dF, dG, dFp, dGp, dno, drs, dst;
  // post-processing scratch (NEXT-4): Maxwell partial sums
  Dev dpart;
  // inner-region eigensolve (NEXT-3): library handles (created on first use) and scratch
  cusolverDnHandle_t solver = nullptr;
  cublasHandle_t blas = nullptr;
  Dev dV, dwork, dinfo;
  // photoionisation amplitudes g of one sweep batch and the split-K partials (NEXT-1)
  Dev dg, dgpart;
  // R-formation algorithm (RMX_R_DMMA / RMX_R_INT8) and the INT8-CRT workspace
  int r_algo = RMX_R_DMMA;
  int64_t r_fallbacks = 0;  // INT8-CRT requests served by the DMMA kernel (workspace did not fit)
  Dev dz;
  Int8Streams i8s;
  // instrumentation
  bool timing = false;
  std::vector<cudaEvent_t> free_events;
  std::vector<PendingTiming> pending;
  double ms[RMX_NKID] = {0, 0, 0, 0, 0};
  int64_t cnt[RMX_NKID] = {0, 0, 0, 0, 0};
  int64_t launches = 0;
};

namespace {

rmx_rc fail(rmx_ctx *c, rmx_rc rc, const std::string &msg) {
  if (c) c->err = msg;
  return rc;
}

rmx_rc cuda_fail(rmx_ctx *c, cudaError_t e, const char *where) {
  if (c) {
    c->err = std::string(where) + ": " + cudaGetErrorString(e);
    c->sticky = e;
  }
  return RMX_ECUDA;
}

cudaEvent_t get_event(rmx_ctx *c) {
  if (!c->free_events.empty()) {
    cudaEvent_t e = c->free_events.back();
    c->free_events.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Brackets one launcher call with events when timing is on; counts kernel launches.
template <class F>
cudaError_t timed(rmx_ctx *c, int kid, int nlaunch, F &&f) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->timing) {
    a = get_event(c);
    b = get_event(c);
    cudaEventRecord(a, c->stream);
  }
  cudaError_t e = f();
  if (c->timing) {
    cudaEventRecord(b, c->stream);
    c->pending.push_back({kid, a, b});
  }
  c->launches += nlaunch;
  c->cnt[kid] += nlaunch;
  return e;
}

void drain_timing(rmx_ctx *c) {
  for (auto &p : c->pending) {
    float ms = 0.f;
    cudaEventSynchronize(p.b);
    cudaEventElapsedTime(&ms, p.a, p.b);
    c->ms[p.kid] += ms;
    c->free_events.push_back(p.a);
    c->free_events.push_back(p.b);
  }
  c->pending.clear();
}

rmx_rc grow(rmx_ctx *c, void **p, size_t *have, size_t need) {
  if (need <= *have) return RMX_OK;
  if (*p) {
    cudaStreamSynchronize(c->stream);
    cudaFree(*p);
    *p = nullptr;
    *have = 0;
  }
  need = std::max<size_t>(need, 256);
  cudaError_t e = cudaMalloc(p, need);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, RMX_ENOMEM, "cudaMalloc(" + std::to_string(need) + " B) failed");
  }
  *have = need;
  return RMX_OK;
}

rmx_rc grow(rmx_ctx *c, rmx_ctx::Dev &d, size_t need) { return grow(c, &d.p, &d.bytes, need); }

int64_t ws_slot_doubles(int64_t nch);
// One CTA per SM (the per-energy kernels use ~220 KB of shared memory): slots = #SMs, fewer when the
// slots would exceed a 48 GB budget (large nch: the T slot is 5 n^2 doubles, 2.7 GB at n = 8192); the
// persistent kernels then loop over more energies per CTA.
int64_t ws_slots_for(const rmx_ctx *c, int64_t nch, int64_t ne) {
  const int64_t budget = static_cast<int64_t>(48) << 30;
  const int64_t by_mem = std::max<int64_t>(1, budget / (ws_slot_doubles(nch) * 8));
  return std::min<int64_t>(std::min<int64_t>(ne, static_cast<int64_t>(c->nsm)), by_mem);
}

rmx_rc build_views(rmx_ctx *c, CUtensorMap **dst, int64_t nch, int64_t slots, int64_t per_slot,
                   const std::vector<MatSpec> &specs) {
  const int nview = 3;
  std::vector<CUtensorMap> h(static_cast<size_t>(slots * specs.size() * nview));
  std::string err;
  for (int64_t s = 0; s < slots; ++s)
    for (size_t m = 0; m < specs.size(); ++m)
      for (int v = 0; v < nview; ++v) {
        const MatSpec &sp = specs[m];
        const double *base = c->ws + s * per_slot + sp.off;
        if (!encode_tmap_f64(&h[(s * specs.size() + m) * nview + v], base, sp.rows, sp.cols, sp.ld,
                             kViewBoxRows[v], err))
          return fail(c, RMX_ECUDA, "tensor map: " + err);
      }
  if (*dst) {
    cudaStreamSynchronize(c->stream);
    cudaFree(*dst);
    *dst = nullptr;
  }
  cudaError_t e = cudaMalloc(dst, h.size() * sizeof(CUtensorMap));
  if (e != cudaSuccess) return fail(c, RMX_ENOMEM, "cudaMalloc(tensor maps) failed");
  e = cudaMemcpy(*dst, h.data(), h.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(c, e, "tensor map upload");
  return RMX_OK;
}

int64_t ws_slot_doubles(int64_t nch) {
  // whole 128-byte lines, so that every slot base keeps the 16-byte alignment TMA needs
  const int64_t d = std::max(match_ws_doubles_per_slot(nch), tepi_ws_doubles_per_slot(nch));
  return (d + 15) & ~15LL;
}

// Workspace for `slots` per-energy slots of the matching / T kernels, with their TMA views.
rmx_rc ensure_ws(rmx_ctx *c, int64_t nch, int64_t slots) {
  slots = std::max<int64_t>(slots, c->views_slots);  // never shrink below what views cover
  const int64_t per = ws_slot_doubles(nch);
  rmx_rc rc = grow(c, reinterpret_cast<void **>(&c->ws), &c->ws_bytes,
                   static_cast<size_t>(per * slots) * sizeof(double) + 4096);
  if (rc != RMX_OK) return rc;
  if (c->views_ws != c->ws || c->views_nch != nch || c->views_slots < slots) {
    std::vector<MatSpec> specs;
    match_view_specs(nch, specs);
    if ((rc = build_views(c, &c->match_views, nch, slots, per, specs)) != RMX_OK) return rc;
    tepi_view_specs(nch, specs);
    if ((rc = build_views(c, &c->tepi_views, nch, slots, per, specs)) != RMX_OK) return rc;
    c->views_ws = c->ws;
    c->views_nch = nch;
    c->views_slots = slots;
  }
  return RMX_OK;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

rmx_rc check_sticky(rmx_ctx *c) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(c, e, "pending CUDA error");
  return RMX_OK;
}

}  // namespace

extern "C" {

int rmx_version(void) { return 200; }
int rmx_sm_target(void) { return 100; }
int64_t rmx_workspace_doubles_per_energy(int64_t nch) {
  if (nch < 1 || nch > (1 << 16)) return -1;
  return ws_slot_doubles(nch);
}

rmx_rc rmx_create(rmx_ctx **ctx, int device, void *stream) {
  if (!ctx) return RMX_EINVAL;
  *ctx = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return RMX_EINVAL;
  }
  rmx_ctx *c = new rmx_ctx();
  c->device = device;
  c->stream = static_cast<cudaStream_t>(stream);
  cudaSetDevice(device);
  cudaDeviceGetAttribute(&c->nsm, cudaDevAttrMultiProcessorCount, device);
  *ctx = c;
  return RMX_OK;
}

rmx_rc rmx_destroy(rmx_ctx *c) {
  if (!c) return RMX_EINVAL;
  cudaStreamSynchronize(c->stream);
  drain_timing(c);
  for (auto e : c->free_events) cudaEventDestroy(e);
  cudaFree(c->ws);
  cudaFree(c->rbuf);
  cudaFree(c->match_views);
  cudaFree(c->tepi_views);
  for (auto *d : {&c->dw, &c->dEk, &c->dE, &c->dF, &c->dG, &c->dFp, &c->dGp, &c->dno, &c->drs,
                  &c->dst, &c->dpart, &c->dV, &c->dwork, &c->dinfo, &c->dg, &c->dgpart, &c->dz})
    cudaFree(d->p);
  if (c->solver) cusolverDnDestroy(c->solver);
  if (c->i8s.aux) {
    cudaStreamDestroy(c->i8s.aux);
    for (cudaEvent_t ev : {c->i8s.start, c->i8s.conv_done[0], c->i8s.conv_done[1], c->i8s.gemm_done[0],
                           c->i8s.gemm_done[1]})
      cudaEventDestroy(ev);
  }
  if (c->blas) cublasDestroy(c->blas);
  delete c;
  return RMX_OK;
}

rmx_rc rmx_set_stream(rmx_ctx *c, void *stream) {
  if (!c) return RMX_EINVAL;
  c->stream = static_cast<cudaStream_t>(stream);
  return RMX_OK;
}

const char *rmx_last_error(const rmx_ctx *c) { return c ? c->err.c_str() : "null ctx"; }

// R formation with the context's algorithm; returns the number of kernel launches in *nl
static cudaError_t form_R(rmx_ctx *c, const double *w, int64_t ldw, const double *Ek, int64_t nch,
                          int64_t nlev, double a, const double *E, int64_t ne, double *R, int32_t *status,
                          std::string &err, int *nl) {
  if (c->r_algo == RMX_R_INT8 && nlev <= rint8_max_nlev() && nch >= kInt8MinChannels) {
    const int64_t chunk = rint8_chunk(nch, nlev, ne, c->nsm);
    const size_t need = rint8_ws_bytes(nch, nlev, chunk);
    if (grow(c, c->dz, need) != RMX_OK) {
      // not enough device memory for the INT8-CRT workspace: the FP64 DMMA formation computes the
      // same R (counted in rmx_stats as an RMX_KID_RFORM launch like the INT8 path)
      c->err.clear();
      c->r_fallbacks += 1;
      *nl = 1;
      return launch_rform(w, ldw, Ek, nch, nlev, a, E, ne, R, status, c->stream, err);
    }
    if (!c->i8s.aux) {
      // default priority: a highest-priority conversion stream (to place conversion CTAs next to the
      // resident GEMM CTAs) made the darc bench stall for > 20 min (round 2) - not used
      cudaStreamCreateWithFlags(&c->i8s.aux, cudaStreamNonBlocking);
      for (cudaEvent_t *ev : {&c->i8s.start, &c->i8s.conv_done[0], &c->i8s.conv_done[1], &c->i8s.gemm_done[0],
                              &c->i8s.gemm_done[1]})
        cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    }
    *nl = 2 + 5 * static_cast<int>((ne + chunk - 1) / chunk);
    cudaEvent_t ga = nullptr;
    auto mark = [&](bool begin) {  // events around each INT8 GEMM launch (instrumentation only)
      if (!c->timing) return;
      cudaEvent_t ev = get_event(c);
      cudaEventRecord(ev, c->stream);
      if (begin) {
        ga = ev;
      } else {
        c->pending.push_back({RMX_KID_I8GEMM, ga, ev});
        c->cnt[RMX_KID_I8GEMM] += 1;
      }
    };
    return launch_rform_int8(w, ldw, Ek, nch, nlev, a, E, ne, R, status, c->dz.p, c->dz.bytes, chunk, c->i8s,
                             c->stream, err, mark);
  }
  *nl = 1;
  return launch_rform(w, ldw, Ek, nch, nlev, a, E, ne, R, status, c->stream, err);
}

rmx_rc rmx_build_R(rmx_ctx *c, const double *w, int64_t ldw, const double *Ek, int64_t nch,
                   int64_t nlev, double a, const double *E, int64_t ne, double *R,
                   int32_t *status) {
  if (!c) return RMX_EINVAL;
  if (!w || !Ek || !E || !R) return fail(c, RMX_EINVAL, "rmx_build_R: null pointer");
  if (nch < 1 || nlev < 1 || ne < 1) return fail(c, RMX_EINVAL, "rmx_build_R: sizes must be >= 1");
  if (nch > (1 << 20) || nlev > (1 << 30)) return fail(c, RMX_EINVAL, "rmx_build_R: size too large");
  if (!(a > 0.0)) return fail(c, RMX_EINVAL, "rmx_build_R: a must be > 0");
  if (ldw < nlev || (ldw & 1) || !aligned16(w))
    return fail(c, RMX_EINVAL, "rmx_build_R: ldw must be >= nlev and even, w 16-byte aligned");
  if (check_sticky(c) != RMX_OK) return RMX_ECUDA;
  cudaSetDevice(c->device);
  std::string err;
  int nl = 1;
  cudaError_t e = timed(c, RMX_KID_RFORM, 0, [&] {
    return form_R(c, w, ldw, Ek, nch, nlev, a, E, ne, R, status, err, &nl);
  });
  c->launches += nl;
  c->cnt[RMX_KID_RFORM] += nl;
  if (e != cudaSuccess) {
    if (!err.empty()) return fail(c, RMX_ECUDA, "rmx_build_R: " + err);
    return cuda_fail(c, e, "rmx_build_R");
  }
  return RMX_OK;
}

rmx_rc rmx_match_K(rmx_ctx *c, const double *R, const double *F, const double *G,
                   const double *Fp, const double *Gp, double a, int64_t nch, int64_t ne,
                   const int32_t *n_open, double *K, int32_t *status) {
  if (!c) return RMX_EINVAL;
  if (!R || !F || !G || !Fp || !Gp || !K) return fail(c, RMX_EINVAL, "rmx_match_K: null pointer");
  if (nch < 1 || ne < 1) return fail(c, RMX_EINVAL, "rmx_match_K: sizes must be >= 1");
  if (nch > kMaxMatchChannels)
    return fail(c, RMX_EINVAL, "rmx_match_K: nch > " + std::to_string(kMaxMatchChannels) +
                                   " (smem-staged LU sub-panels)");
  if (!(a > 0.0)) return fail(c, RMX_EINVAL, "rmx_match_K: a must be > 0");
  if (check_sticky(c) != RMX_OK) return RMX_ECUDA;
  cudaSetDevice(c->device);
  const int64_t slots = ws_slots_for(c, nch, ne);
  rmx_rc rc = ensure_ws(c, nch, slots);
  if (rc != RMX_OK) return rc;
  cudaError_t e = timed(c, RMX_KID_MATCH, 1, [&] {
    return launch_match(R, F, G, Fp, Gp, a, nch, ne, n_open, K, c->ws, ws_slot_doubles(nch), c->match_views, slots, status,
                        c->stream);
  });
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_match_K");
  return RMX_OK;
}

rmx_rc rmx_collision_strength(rmx_ctx *c, const double *K, int64_t nch, int64_t ne,
                              const int32_t *n_open, double *T2, double *rowsum,
                              int32_t *status) {
  if (!c) return RMX_EINVAL;
  if (!K) return fail(c, RMX_EINVAL, "rmx_collision_strength: null K");
  if (nch < 1 || ne < 1) return fail(c, RMX_EINVAL, "rmx_collision_strength: sizes must be >= 1");
  if (nch > (1 << 16)) return fail(c, RMX_EINVAL, "rmx_collision_strength: nch too large");
  if (check_sticky(c) != RMX_OK) return RMX_ECUDA;
  cudaSetDevice(c->device);
  const int64_t slots = ws_slots_for(c, nch, ne);
  rmx_rc rc = ensure_ws(c, nch, slots);
  if (rc != RMX_OK) return rc;
  cudaError_t e = timed(c, RMX_KID_TEPI, 1, [&] {
    return launch_tepi(K, nch, nch * nch, nch, ne, n_open, T2, nullptr, rowsum, LevelSums{}, PhotoArgs{}, c->ws,
                       ws_slot_doubles(nch), c->tepi_views, slots, status, c->stream);
  });
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_collision_strength");
  return RMX_OK;
}

// host-side validation of a level partition: 0 = level_start[0] < ... <= nch (the array itself is
// on the device; only nlevel and the pointer can be checked synchronously)
static rmx_rc check_levels(rmx_ctx *c, const char *who, const int32_t *level_start, int64_t nlevel,
                           const double *omega) {
  if (!level_start || !omega) return fail(c, RMX_EINVAL, std::string(who) + ": null level_start / omega");
  if (nlevel < 1 || nlevel > (1 << 16)) return fail(c, RMX_EINVAL, std::string(who) + ": bad nlevel");
  return RMX_OK;
}

rmx_rc rmx_collision_strength_levels(rmx_ctx *c, const double *K, int64_t nch, int64_t ne,
                                     const int32_t *n_open, const int32_t *level_start,
                                     int64_t nlevel, double g, double *omega, int32_t *status) {
  if (!c) return RMX_EINVAL;
  if (!K) return fail(c, RMX_EINVAL, "rmx_collision_strength_levels: null K");
  if (nch < 1 || ne < 1) return fail(c, RMX_EINVAL, "rmx_collision_strength_levels: sizes must be >= 1");
  if (nch > (1 << 16)) return fail(c, RMX_EINVAL, "rmx_collision_strength_levels: nch too large");
  rmx_rc rc = check_levels(c, "rmx_collision_strength_levels", level_start, nlevel, omega);
  if (rc != RMX_OK) return rc;
  if (check_sticky(c) != RMX_OK) return RMX_ECUDA;
  cudaSetDevice(c->device);
  const int64_t slots = ws_slots_for(c, nch, ne);
  rc = ensure_ws(c, nch, slots);
  if (rc != RMX_OK) return rc;
  LevelSums lv;
  lv.level_start = level_start;
  lv.nlevel = static_cast<int>(nlevel);
  lv.g = g;
  lv.omega = omega;
  cudaError_t e = timed(c, RMX_KID_TEPI, 1, [&] {
    return launch_tepi(K, nch, nch * nch, nch, ne, n_open, nullptr, nullptr, nullptr, lv, PhotoArgs{}, c->ws,
                       ws_slot_doubles(nch), c->tepi_views, slots, status, c->stream);
  });
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_collision_strength_levels");
  return RMX_OK;
}

static int64_t default_batch(const rmx_ctx *c, int64_t nch, int64_t ne) {
  const int64_t unit = 2 * static_cast<int64_t>(c->nsm);
  const int64_t budget = static_cast<int64_t>(8) << 30;  // bytes for the R/K batch buffer
  int64_t b = std::max<int64_t>(1, budget / (nch * nch * 8));
  if (b >= unit) b = (b / unit) * unit;  // whole waves of 2 energies per SM when the budget allows
  return std::min<int64_t>(b, ne);
}

// NEXT-1 inputs/outputs of the fused photoionisation sweep
struct PhotoIn {
  const double *d;
  double E0, C;
  double *sigma, *mabs2;
};

static rmx_rc sweep_impl(rmx_ctx *c, const double *w, int64_t ldw, const double *Ek, int64_t nch,
                         int64_t nlev, double a, const double *E, int64_t ne, const double *F,
                         const double *G, const double *Fp, const double *Gp,
                         const int32_t *n_open, int64_t batch, const int64_t *dump_idx,
                         int64_t n_dump, double *R_d, double *K_d, double *T2_d, double *rowsum,
                         const LevelSums &lv, int32_t *status, const PhotoIn *ph = nullptr) {
  if (!c) return RMX_EINVAL;
  if (!w || !Ek || !E || !F || !G || !Fp || !Gp || (!rowsum && !lv.omega && !ph))
    return fail(c, RMX_EINVAL, "rmx_sweep: null pointer");
  if (nch < 1 || nlev < 1 || ne < 1) return fail(c, RMX_EINVAL, "rmx_sweep: sizes must be >= 1");
  if (nch > kMaxMatchChannels)
    return fail(c, RMX_EINVAL, "rmx_sweep: nch > " + std::to_string(kMaxMatchChannels) +
                                   " (smem-staged LU sub-panels)");
  if (!(a > 0.0)) return fail(c, RMX_EINVAL, "rmx_sweep: a must be > 0");
  if (ldw < nlev || (ldw & 1) || !aligned16(w))
    return fail(c, RMX_EINVAL, "rmx_sweep: ldw must be >= nlev and even, w 16-byte aligned");
  if (n_dump < 0 || (n_dump > 0 && !dump_idx)) return fail(c, RMX_EINVAL, "rmx_sweep: bad dump list");
  for (int64_t d = 0; d < n_dump; ++d)
    if (dump_idx[d] < 0 || dump_idx[d] >= ne) return fail(c, RMX_EINVAL, "rmx_sweep: dump index out of range");
  if (check_sticky(c) != RMX_OK) return RMX_ECUDA;
  cudaSetDevice(c->device);
  if (batch <= 0) batch = default_batch(c, nch, ne);
  batch = std::min(batch, ne);
  const int64_t slots = ws_slots_for(c, nch, batch);
  rmx_rc rc = ensure_ws(c, nch, slots);
  if (rc != RMX_OK) return rc;
  const size_t mat = static_cast<size_t>(nch) * nch;
  rc = grow(c, reinterpret_cast<void **>(&c->rbuf), &c->rbuf_bytes,
            static_cast<size_t>(batch) * mat * sizeof(double));
  if (rc != RMX_OK) return rc;
  double *rb = c->rbuf;
  if (ph && ((rc = grow(c, c->dg, sizeof(double) * batch * nch)) ||
             (rc = grow(c, c->dgpart, sizeof(double) * dipole_g_splits(nch, nlev, batch) * batch * nch))))
    return rc;
  std::string err;
  for (int64_t b0 = 0; b0 < ne; b0 += batch) {
    const int64_t nb = std::min(batch, ne - b0);
    int32_t *stb = status ? status + b0 : nullptr;
    const int32_t *nob = n_open ? n_open + b0 : nullptr;
    int nl = 1;
    cudaError_t e = timed(c, RMX_KID_RFORM, 0, [&] {
      return form_R(c, w, ldw, Ek, nch, nlev, a, E + b0, nb, rb, stb, err, &nl);
    });
    c->launches += nl;
    c->cnt[RMX_KID_RFORM] += nl;
    if (e != cudaSuccess) return err.empty() ? cuda_fail(c, e, "rmx_sweep/R") : fail(c, RMX_ECUDA, err);
    for (int64_t d = 0; d < n_dump; ++d)
      if (R_d && dump_idx[d] >= b0 && dump_idx[d] < b0 + nb)
        cudaMemcpyAsync(R_d + d * mat, rb + (dump_idx[d] - b0) * mat, mat * sizeof(double),
                        cudaMemcpyDeviceToDevice, c->stream);
    // the T epilogue reads K_oo only: solve for the open unknowns alone unless this batch dumps a
    // full K or the photoionisation amplitudes need K's closed rows
    bool dumps = false;
    for (int64_t d = 0; d < n_dump; ++d) dumps |= dump_idx[d] >= b0 && dump_idx[d] < b0 + nb;
    const int open_only = (!dumps && !ph) ? 1 : 0;
    e = timed(c, RMX_KID_MATCH, 1, [&] {
      return launch_match(rb, F + b0 * nch, G + b0 * nch, Fp + b0 * nch, Gp + b0 * nch, a, nch, nb,
                          nob, rb, c->ws, ws_slot_doubles(nch), c->match_views, slots, stb, c->stream,
                          open_only);
    });
    if (e != cudaSuccess) return cuda_fail(c, e, "rmx_sweep/K");
    for (int64_t d = 0; d < n_dump; ++d) {
      const int64_t l = dump_idx[d] - b0;
      if (l < 0 || l >= nb) continue;
      if (K_d)
        cudaMemcpyAsync(K_d + d * mat, rb + l * mat, mat * sizeof(double),
                        cudaMemcpyDeviceToDevice, c->stream);
      if (T2_d) {
        e = timed(c, RMX_KID_TEPI, 1, [&] {
          return launch_tepi(rb + l * mat, nch, mat, nch, 1, nob ? nob + l : nullptr, T2_d + d * mat,
                             nullptr, nullptr, LevelSums{}, PhotoArgs{}, c->ws, ws_slot_doubles(nch), c->tepi_views, 1, nullptr, c->stream);
        });
        if (e != cudaSuccess) return cuda_fail(c, e, "rmx_sweep/T dump");
      }
    }
    LevelSums lvb = lv;
    if (lvb.omega) lvb.omega += b0 * static_cast<int64_t>(lv.nlevel) * lv.nlevel;
    PhotoArgs pab;
    if (ph) {
      // NEXT-1: g for this batch, then the amplitudes inside the T epilogue
      double *gb = static_cast<double *>(c->dg.p);
      e = timed(c, RMX_KID_OTHER, 3, [&] {
        return launch_dipole_g(w, ldw, Ek, ph->d, nch, nlev, E + b0, nb, gb, stb,
                               static_cast<double *>(c->dgpart.p),
                               static_cast<int64_t>(c->dgpart.bytes / sizeof(double)), c->stream);
      });
      if (e != cudaSuccess) return cuda_fail(c, e, "rmx_sweep_photo/g");
      pab.g = gb;
      pab.Fp = Fp + b0 * nch;
      pab.Gp = Gp + b0 * nch;
      pab.E = E + b0;
      pab.E0 = ph->E0;
      pab.C = ph->C;
      pab.sigma = ph->sigma + b0;
      pab.mabs2 = ph->mabs2 ? ph->mabs2 + b0 * nch : nullptr;
    }
    e = timed(c, RMX_KID_TEPI, 1, [&] {
      return launch_tepi(rb, nch, mat, nch, nb, nob, nullptr, nullptr,
                         rowsum ? rowsum + b0 * nch : nullptr, lvb, pab, c->ws, ws_slot_doubles(nch),
                         c->tepi_views, slots, stb, c->stream);
    });
    if (e != cudaSuccess) return cuda_fail(c, e, "rmx_sweep/T");
  }
  return RMX_OK;
}

rmx_rc rmx_sweep(rmx_ctx *c, const double *w, int64_t ldw, const double *Ek, int64_t nch,
                 int64_t nlev, double a, const double *E, int64_t ne, const double *F,
                 const double *G, const double *Fp, const double *Gp, const int32_t *n_open,
                 int64_t batch, const int64_t *dump_idx, int64_t n_dump, double *R_d,
                 double *K_d, double *T2_d, double *rowsum, int32_t *status) {
  if (c && !rowsum) return fail(c, RMX_EINVAL, "rmx_sweep: null rowsum");
  return sweep_impl(c, w, ldw, Ek, nch, nlev, a, E, ne, F, G, Fp, Gp, n_open, batch, dump_idx,
                    n_dump, R_d, K_d, T2_d, rowsum, LevelSums{}, status);
}

rmx_rc rmx_sweep_levels(rmx_ctx *c, const double *w, int64_t ldw, const double *Ek, int64_t nch,
                        int64_t nlev, double a, const double *E, int64_t ne, const double *F,
                        const double *G, const double *Fp, const double *Gp,
                        const int32_t *n_open, int64_t batch, const int32_t *level_start,
                        int64_t nlevel, double g, double *omega, double *rowsum,
                        int32_t *status) {
  if (!c) return RMX_EINVAL;
  rmx_rc rc = check_levels(c, "rmx_sweep_levels", level_start, nlevel, omega);
  if (rc != RMX_OK) return rc;
  LevelSums lv;
  lv.level_start = level_start;
  lv.nlevel = static_cast<int>(nlevel);
  lv.g = g;
  lv.omega = omega;
  return sweep_impl(c, w, ldw, Ek, nch, nlev, a, E, ne, F, G, Fp, Gp, n_open, batch, nullptr, 0,
                    nullptr, nullptr, nullptr, rowsum, lv, status);
}

rmx_rc rmx_dipole_amplitude(rmx_ctx *c, const double *w, int64_t ldw, const double *Ek,
                            const double *d, int64_t nch, int64_t nlev, const double *E, int64_t ne,
                            double *g, int32_t *status) {
  if (!c) return RMX_EINVAL;
  if (!w || !Ek || !d || !E || !g) return fail(c, RMX_EINVAL, "rmx_dipole_amplitude: null pointer");
  if (nch < 1 || nlev < 1 || ne < 1 || nch > (1 << 20) || nlev > (1 << 30))
    return fail(c, RMX_EINVAL, "rmx_dipole_amplitude: bad sizes");
  if (ldw < nlev) return fail(c, RMX_EINVAL, "rmx_dipole_amplitude: ldw < nlev");
  if (check_sticky(c) != RMX_OK) return RMX_ECUDA;
  cudaSetDevice(c->device);
  const int64_t ne1 = std::min<int64_t>(ne, static_cast<int64_t>(65535) * 64);
  rmx_rc rc = grow(c, c->dgpart, sizeof(double) * dipole_g_splits(nch, nlev, ne1) * ne1 * nch);
  if (rc != RMX_OK) return rc;
  cudaError_t e = timed(c, RMX_KID_OTHER, 3, [&] {  // contraction, split-K reduction, nearest-pole term
    return launch_dipole_g(w, ldw, Ek, d, nch, nlev, E, ne, g, status,
                           static_cast<double *>(c->dgpart.p),
                           static_cast<int64_t>(c->dgpart.bytes / sizeof(double)), c->stream);
  });
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_dipole_amplitude");
  return RMX_OK;
}

rmx_rc rmx_photoionization(rmx_ctx *c, const double *K, const double *g, const double *Fp,
                           const double *Gp, const double *E, int64_t nch, int64_t ne,
                           const int32_t *n_open, double E0, double C, double *sigma,
                           double *mabs2, int32_t *status) {
  if (!c) return RMX_EINVAL;
  if (!K || !g || !Fp || !Gp || !E || !sigma)
    return fail(c, RMX_EINVAL, "rmx_photoionization: null pointer");
  if (nch < 1 || ne < 1 || nch > kMaxMatchChannels)
    return fail(c, RMX_EINVAL, "rmx_photoionization: bad sizes");
  if (check_sticky(c) != RMX_OK) return RMX_ECUDA;
  cudaSetDevice(c->device);
  const int64_t slots = ws_slots_for(c, nch, ne);
  rmx_rc rc = ensure_ws(c, nch, slots);
  if (rc != RMX_OK) return rc;
  PhotoArgs pa;
  pa.g = g;
  pa.Fp = Fp;
  pa.Gp = Gp;
  pa.E = E;
  pa.E0 = E0;
  pa.C = C;
  pa.sigma = sigma;
  pa.mabs2 = mabs2;
  cudaError_t e = timed(c, RMX_KID_TEPI, 1, [&] {
    return launch_tepi(K, nch, nch * nch, nch, ne, n_open, nullptr, nullptr, nullptr, LevelSums{}, pa,
                       c->ws, ws_slot_doubles(nch), c->tepi_views, slots, status, c->stream);
  });
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_photoionization");
  return RMX_OK;
}

rmx_rc rmx_sweep_photo(rmx_ctx *c, const double *w, int64_t ldw, const double *Ek, const double *d,
                       int64_t nch, int64_t nlev, double a, const double *E, int64_t ne,
                       const double *F, const double *G, const double *Fp, const double *Gp,
                       const int32_t *n_open, int64_t batch, double E0, double C, double *sigma,
                       double *mabs2, int32_t *status) {
  if (!c) return RMX_EINVAL;
  if (!d || !sigma) return fail(c, RMX_EINVAL, "rmx_sweep_photo: null d / sigma");
  PhotoIn ph{d, E0, C, sigma, mabs2};
  return sweep_impl(c, w, ldw, Ek, nch, nlev, a, E, ne, F, G, Fp, Gp, n_open, batch, nullptr, 0,
                    nullptr, nullptr, nullptr, nullptr, LevelSums{}, status, &ph);
}

rmx_rc rmx_sweep_host(rmx_ctx *c, const double *w, int64_t ldw, const double *Ek, int64_t nch,
                      int64_t nlev, double a, const double *E, int64_t ne, const double *F,
                      const double *G, const double *Fp, const double *Gp, const int32_t *n_open,
                      int64_t batch, double *rowsum, int32_t *status, int64_t *h2d_bytes,
                      int64_t *d2h_bytes) {
  if (!c) return RMX_EINVAL;
  if (!w || !Ek || !E || !F || !G || !Fp || !Gp || !rowsum || !status)
    return fail(c, RMX_EINVAL, "rmx_sweep_host: null pointer");
  if (nch < 1 || nlev < 1 || ne < 1 || ldw < nlev || (ldw & 1))
    return fail(c, RMX_EINVAL, "rmx_sweep_host: bad sizes / ldw");
  cudaSetDevice(c->device);
  const size_t bw = sizeof(double) * nch * ldw, bek = sizeof(double) * nlev,
               be = sizeof(double) * ne, bf = sizeof(double) * ne * nch,
               bno = sizeof(int32_t) * ne;
  rmx_rc rc;
  if ((rc = grow(c, c->dw, bw)) || (rc = grow(c, c->dEk, bek)) || (rc = grow(c, c->dE, be)) ||
      (rc = grow(c, c->dF, bf)) || (rc = grow(c, c->dG, bf)) || (rc = grow(c, c->dFp, bf)) ||
      (rc = grow(c, c->dGp, bf)) || (rc = grow(c, c->dno, bno)) || (rc = grow(c, c->drs, bf)) ||
      (rc = grow(c, c->dst, bno)))
    return rc;
  auto h2d = [&](void *dst, const void *src, size_t n) {
    return cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, c->stream);
  };
  cudaError_t e = cudaSuccess;
  e = e ? e : h2d(c->dw.p, w, bw);
  e = e ? e : h2d(c->dEk.p, Ek, bek);
  e = e ? e : h2d(c->dE.p, E, be);
  e = e ? e : h2d(c->dF.p, F, bf);
  e = e ? e : h2d(c->dG.p, G, bf);
  e = e ? e : h2d(c->dFp.p, Fp, bf);
  e = e ? e : h2d(c->dGp.p, Gp, bf);
  if (n_open) e = e ? e : h2d(c->dno.p, n_open, bno);
  e = e ? e : cudaMemsetAsync(c->dst.p, 0, bno, c->stream);
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_sweep_host/h2d");
  rc = rmx_sweep(c, static_cast<double *>(c->dw.p), ldw, static_cast<double *>(c->dEk.p), nch, nlev,
                 a, static_cast<double *>(c->dE.p), ne, static_cast<double *>(c->dF.p),
                 static_cast<double *>(c->dG.p), static_cast<double *>(c->dFp.p),
                 static_cast<double *>(c->dGp.p),
                 n_open ? static_cast<int32_t *>(c->dno.p) : nullptr, batch, nullptr, 0, nullptr,
                 nullptr, nullptr, static_cast<double *>(c->drs.p),
                 static_cast<int32_t *>(c->dst.p));
  if (rc != RMX_OK) return rc;
  e = cudaMemcpyAsync(rowsum, c->drs.p, bf, cudaMemcpyDeviceToHost, c->stream);
  e = e ? e : cudaMemcpyAsync(status, c->dst.p, bno, cudaMemcpyDeviceToHost, c->stream);
  e = e ? e : cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_sweep_host/d2h");
  if (h2d_bytes) *h2d_bytes = static_cast<int64_t>(bw + bek + be + 4 * bf + (n_open ? bno : 0));
  if (d2h_bytes) *d2h_bytes = static_cast<int64_t>(bf + bno);
  return RMX_OK;
}

rmx_rc rmx_convolve_gaussian(rmx_ctx *c, const double *x, int64_t nspec, const double *mix,
                             int64_t ne, double dE, double fwhm, double *y) {
  if (!c) return RMX_EINVAL;
  if (!x || !y) return fail(c, RMX_EINVAL, "rmx_convolve_gaussian: null pointer");
  if (nspec < 1 || ne < 1 || nspec > 65535) return fail(c, RMX_EINVAL, "rmx_convolve_gaussian: bad sizes");
  if (mix && nspec > 64) return fail(c, RMX_EINVAL, "rmx_convolve_gaussian: at most 64 admixture components");
  if (!(dE > 0.0) || !(fwhm > 0.0)) return fail(c, RMX_EINVAL, "rmx_convolve_gaussian: dE, fwhm must be > 0");
  if (fwhm < 2.0 * dE) return fail(c, RMX_EINVAL, "rmx_convolve_gaussian: fwhm < 2 dE (under-resolved kernel)");
  const int M = conv_window(dE, fwhm, nullptr);
  if (M > kMaxConvHalfWidth)
    return fail(c, RMX_EINVAL, "rmx_convolve_gaussian: window 5 sigma / dE > " + std::to_string(kMaxConvHalfWidth));
  double msum = 0.0;
  if (mix)
    for (int64_t m = 0; m < nspec; ++m) {
      if (!(mix[m] >= 0.0)) return fail(c, RMX_EINVAL, "rmx_convolve_gaussian: negative admixture weight");
      msum += mix[m];
    }
  if (mix && !(msum > 0.0)) return fail(c, RMX_EINVAL, "rmx_convolve_gaussian: admixture weights sum to 0");
  if (check_sticky(c) != RMX_OK) return RMX_ECUDA;
  cudaSetDevice(c->device);
  cudaError_t e = timed(c, RMX_KID_OTHER, 1, [&] {
    return launch_convolve(x, nspec, mix, ne, dE, fwhm, y, c->stream);
  });
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_convolve_gaussian");
  return RMX_OK;
}

rmx_rc rmx_maxwell_average(rmx_ctx *c, const double *omega, int64_t ne, int64_t npair,
                           const double *E, const double *Eth, const double *kT, int64_t nT,
                           double *ups) {
  if (!c) return RMX_EINVAL;
  if (!omega || !E || !Eth || !kT || !ups) return fail(c, RMX_EINVAL, "rmx_maxwell_average: null pointer");
  if (ne < 1 || npair < 1) return fail(c, RMX_EINVAL, "rmx_maxwell_average: sizes must be >= 1");
  if (nT < 1 || nT > RMX_MAX_TEMPS)
    return fail(c, RMX_EINVAL, "rmx_maxwell_average: 1 <= nT <= RMX_MAX_TEMPS");
  for (int64_t t = 0; t < nT; ++t)
    if (!(kT[t] > 0.0)) return fail(c, RMX_EINVAL, "rmx_maxwell_average: kT must be > 0");
  if (check_sticky(c) != RMX_OK) return RMX_ECUDA;
  cudaSetDevice(c->device);
  rmx_rc rc = grow(c, c->dpart, sizeof(double) * maxwell_chunks(ne) * npair * nT);
  if (rc != RMX_OK) return rc;
  cudaError_t e = timed(c, RMX_KID_OTHER, 2, [&] {
    return launch_maxwell(omega, ne, npair, E, Eth, kT, static_cast<int>(nT),
                          static_cast<double *>(c->dpart.p), ups, c->stream);
  });
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_maxwell_average");
  return RMX_OK;
}

rmx_rc rmx_inner_region(rmx_ctx *c, const double *H, int64_t nlev, const double *P, int64_t nch,
                        double *Ek, double *w, int64_t ldw) {
  if (!c) return RMX_EINVAL;
  if (!H || !P || !Ek || !w) return fail(c, RMX_EINVAL, "rmx_inner_region: null pointer");
  if (nlev < 1 || nch < 1 || nlev > (1 << 17)) return fail(c, RMX_EINVAL, "rmx_inner_region: bad sizes");
  if (ldw < nlev) return fail(c, RMX_EINVAL, "rmx_inner_region: ldw < nlev");
  if (check_sticky(c) != RMX_OK) return RMX_ECUDA;
  cudaSetDevice(c->device);
  if (!c->solver && cusolverDnCreate(&c->solver) != CUSOLVER_STATUS_SUCCESS)
    return fail(c, RMX_ECUDA, "rmx_inner_region: cusolverDnCreate failed");
  if (!c->blas && cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS)
    return fail(c, RMX_ECUDA, "rmx_inner_region: cublasCreate failed");
  cusolverDnSetStream(c->solver, c->stream);
  cublasSetStream(c->blas, c->stream);
  const size_t nn = static_cast<size_t>(nlev) * nlev;
  rmx_rc rc;
  if ((rc = grow(c, c->dV, sizeof(double) * nn)) || (rc = grow(c, c->dinfo, sizeof(int))))
    return rc;
  double *V = static_cast<double *>(c->dV.p);
  cudaError_t e = cudaMemcpyAsync(V, H, sizeof(double) * nn, cudaMemcpyDeviceToDevice, c->stream);
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_inner_region/copy");
  // H is symmetric, so its row-major array is also its column-major array; after syevd the
  // column-major V holds eigenvector k in column k (= row k of the row-major view), E_k ascending.
  const int n = static_cast<int>(nlev);
  int lwork = 0;
  if (cusolverDnDsyevd_bufferSize(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, V, n,
                                  Ek, &lwork) != CUSOLVER_STATUS_SUCCESS)
    return fail(c, RMX_ECUDA, "rmx_inner_region: syevd_bufferSize failed");
  if ((rc = grow(c, c->dwork, sizeof(double) * static_cast<size_t>(lwork)))) return rc;
  int *info = static_cast<int *>(c->dinfo.p);
  cusolverStatus_t ss;
  e = timed(c, RMX_KID_OTHER, 1, [&] {
    ss = cusolverDnDsyevd(c->solver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, V, n, Ek,
                          static_cast<double *>(c->dwork.p), lwork, info);
    return cudaGetLastError();
  });
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_inner_region/syevd");
  if (ss != CUSOLVER_STATUS_SUCCESS) return fail(c, RMX_ECUDA, "rmx_inner_region: syevd failed");
  // w = P^T V, written row-major [nch][ldw]: as column-major that is w_cm (nlev x nch, ld ldw)
  // = V^T P, with P's row-major [nlev][nch] array being the column-major nch x nlev matrix P^T.
  const double one = 1.0, zero = 0.0;
  cublasStatus_t bs;
  e = timed(c, RMX_KID_OTHER, 1, [&] {
    bs = cublasDgemm(c->blas, CUBLAS_OP_T, CUBLAS_OP_T, n, static_cast<int>(nch), n, &one, V, n, P,
                     static_cast<int>(nch), &zero, w, static_cast<int>(ldw));
    return cudaGetLastError();
  });
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_inner_region/gemm");
  if (bs != CUBLAS_STATUS_SUCCESS) return fail(c, RMX_ECUDA, "rmx_inner_region: cublasDgemm failed");
  int hinfo = 0;
  e = cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, c->stream);
  e = e ? e : cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_inner_region/info");
  if (hinfo != 0)
    return fail(c, RMX_ECUDA, "rmx_inner_region: syevd info = " + std::to_string(hinfo));
  return RMX_OK;
}

rmx_rc rmx_sync(rmx_ctx *c, const int32_t *status, int64_t ne, int64_t *n_bad) {
  if (!c) return RMX_EINVAL;
  cudaSetDevice(c->device);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e != cudaSuccess) return cuda_fail(c, e, "rmx_sync");
  if (c->sticky != cudaSuccess) return RMX_ECUDA;
  if (n_bad) {
    *n_bad = 0;
    if (status && ne > 0) {
      std::vector<int32_t> h(static_cast<size_t>(ne));
      e = cudaMemcpy(h.data(), status, sizeof(int32_t) * ne, cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return cuda_fail(c, e, "rmx_sync/status");
      for (auto s : h) *n_bad += (s != 0);
    }
  }
  return RMX_OK;
}

rmx_rc rmx_set_r_algo(rmx_ctx *c, int algo) {
  if (!c) return RMX_EINVAL;
  if (algo != RMX_R_DMMA && algo != RMX_R_INT8) return fail(c, RMX_EINVAL, "rmx_set_r_algo: unknown algorithm");
  c->r_algo = algo;
  return RMX_OK;
}

rmx_rc rmx_set_timing(rmx_ctx *c, int enable) {
  if (!c) return RMX_EINVAL;
  c->timing = enable != 0;
  return RMX_OK;
}

rmx_rc rmx_reset_stats(rmx_ctx *c) {
  if (!c) return RMX_EINVAL;
  cudaStreamSynchronize(c->stream);
  drain_timing(c);
  for (int k = 0; k < RMX_NKID; ++k) {
    c->ms[k] = 0;
    c->cnt[k] = 0;
  }
  c->launches = 0;
  return RMX_OK;
}

rmx_rc rmx_stats(rmx_ctx *c, double *ms, int64_t *launches, int64_t *total) {
  if (!c) return RMX_EINVAL;
  cudaStreamSynchronize(c->stream);
  drain_timing(c);
  for (int k = 0; k < RMX_NKID; ++k) {
    if (ms) ms[k] = c->ms[k];
    if (launches) launches[k] = c->cnt[k];
  }
  if (total) *total = c->launches;
  return RMX_OK;
}

}  // extern "C"
