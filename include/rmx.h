/*
 * rmx.h - C ABI of librmx, the B200-native (sm_100a) outer-region energy sweep of the
 * R-matrix method (McLaughlin & Ballance, arxiv 1403.5524):
 *
 *     R(E)  = (1/2a) W diag(1/(E_k - E)) W^T                      (§6 Eq. 1-2,
 *                                                                  north_star convention, BASELINE.json:5)
 *     K(E)  = -(G - aR G')^{-1} (F - aR F')                       (BASELINE.json:5)
 *     T(E)  = 2i K_oo (I - i K_oo)^{-1},  |T_ij|^2                (BASELINE.json:5)
 *
 * Conventions shared by every call
 * --------------------------------
 *  - All floating-point arrays are IEEE fp64, row-major, C-contiguous unless a leading
 *    dimension is given. "DEVICE" pointers are CUDA device memory of the ctx's device;
 *    "HOST" pointers are ordinary (preferably pinned) host memory.
 *  - Ownership: the caller owns every buffer it passes; the library owns only the
 *    workspace inside rmx_ctx. No buffer is retained after a call returns.
 *  - Asynchrony: device-pointer calls are enqueued on the ctx's CUDA stream and return
 *    before the kernels finish; results are valid after the stream is synchronised
 *    (rmx_sync, cudaStreamSynchronize, or a later operation on the same stream).
 *    The only host allocation/cudaMalloc happens when the workspace must grow (first call
 *    at a larger shape); the hot loop of rmx_sweep allocates nothing.
 *  - Call-level errors (rmx_rc) are synchronous argument checks: a null pointer, a
 *    non-positive size, a <= 0, a bad leading dimension or alignment. (n_open lives on the
 *    device and cannot be checked synchronously: kernels clamp it to [0, nch].) On an
 *    error nothing is enqueued and
 *    rmx_last_error() describes it. RMX_ECUDA reports a CUDA launch/runtime error
 *    (sticky errors are also returned by the next call or by rmx_sync).
 *  - Per-energy problems never abort a batch. They are reported in the caller's int32
 *    status[ne] array, which the caller must initialise (e.g. to 0 = RMX_E_OK) before
 *    the first call of a pipeline. A call writes a code only into entries that are still
 *    RMX_E_OK (first error wins), so one status array can follow an energy through
 *    build_R -> match_K -> collision_strength. Outputs of a flagged energy are NaN (POLE)
 *    or undefined-but-finite-or-NaN (SINGULAR / NONFINITE).
 *  - Preconditions (not checked, documented; rmx_synth guarantees them): E_k ascending;
 *    channels sorted by threshold so the open set is the prefix [0, n_open); closed-
 *    channel entries of F,G,F',G' satisfy F=G, F'=G' (the e^{-kappa a} functions of
 *    BASELINE.json:9, reading M3), so the closed columns of K are exactly -e_j.
 */
#ifndef RMX_H
#define RMX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rmx_ctx rmx_ctx;

typedef enum {
  RMX_OK = 0,      /* success                                   */
  RMX_EINVAL = 1,  /* bad argument (synchronous; nothing launched) */
  RMX_ENOMEM = 2,  /* workspace / pinned staging allocation failed */
  RMX_ECUDA = 3    /* CUDA runtime / launch error                */
} rmx_rc;

/* per-energy status codes written into int32 status[ne] */
enum {
  RMX_E_OK = 0,
  RMX_E_POLE = 1,      /* |E - E_k| < 1e-10 Ry for some k; outputs NaN */
  RMX_E_SINGULAR = 2,  /* exact zero pivot in the matching LU (LAPACK info > 0 style) */
  RMX_E_NONFINITE = 3  /* a non-finite value reached K or |T|^2 */
};

/* Create a context on CUDA device `device`, enqueuing on `cuda_stream` (a cudaStream_t;
 * NULL = the legacy default stream). */
rmx_rc rmx_create(rmx_ctx **ctx, int device, void *cuda_stream);
rmx_rc rmx_destroy(rmx_ctx *ctx);
/* Change the stream subsequent calls enqueue on (e.g. torch's current stream). */
rmx_rc rmx_set_stream(rmx_ctx *ctx, void *cuda_stream);
/* Human-readable description of the last call-level error of this ctx ("" if none). */
const char *rmx_last_error(const rmx_ctx *ctx);

/*
 * rmx_build_R - S1+S2: R_ij(E_e) = (1/2a) sum_k w_ik w_jk / (E_k - E_e)   (Eq.1-2;
 * BASELINE.json:5). Upper triangle computed by an energy-batched FP64 DMMA contraction with
 * TMA-staged W tiles (or, after rmx_set_r_algo(RMX_R_INT8), exactly on the INT8 tensor cores);
 * the denominators 1/(E_k - E) are formed on chip, never stored. The term of the pole nearest to
 * E_e is summed apart and added last (reading N1: keeps the rest of the sum accurate next
 * to a pole). R is written full and BITWISE symmetric (upper triangle mirrored).
 *   w      DEVICE [nch][ldw]  amplitudes, k contiguous; ldw >= nlev, ldw even (ldw*8 % 16 == 0,
 *                             TMA stride rule) and w 16-byte aligned
 *   Ek     DEVICE [nlev]      poles, ascending
 *   E      DEVICE [ne]        energies
 *   R      DEVICE [ne][nch][nch]  output
 *   status DEVICE int32 [ne]  RMX_E_POLE where min_k |E - E_k| < 1e-10 (R is NaN there)
 * Errors: EINVAL on null pointers, nch/nlev/ne < 1, a <= 0 or a bad ldw/alignment.
 */
rmx_rc rmx_build_R(rmx_ctx *ctx, const double *w, int64_t ldw, const double *Ek, int64_t nch,
                   int64_t nlev, double a, const double *E, int64_t ne, double *R,
                   int32_t *status);

/*
 * rmx_match_K - S3+S4: K = -(G - aRG')^{-1}(F - aRF') per energy (BASELINE.json:5), with
 * A_ij = G_i d_ij - a R_ij G'_j, B_ij = F_i d_ij - a R_ij F'_j. One CTA per energy runs a
 * blocked right-looking LU with partial pivoting of A (FP64 DMMA trailing updates) on the
 * augmented matrix [A | B_open]; the n_open open columns are solved, the closed columns
 * are written as -e_j (precondition above).
 *   R              DEVICE [ne][nch][nch]
 *   F, G, Fp, Gp   DEVICE [ne][nch] asymptotic functions at r = a
 *   n_open         DEVICE int32 [ne] or NULL (= all nch open)
 *   K              DEVICE [ne][nch][nch] output
 *   status         DEVICE int32 [ne]: RMX_E_SINGULAR on an exact zero pivot,
 *                  RMX_E_NONFINITE if K_oo is not finite
 * Errors: EINVAL on null pointers, sizes < 1, a <= 0, or nch > 8192 (up to 2944 channels the LU
 * sub-panels live in shared memory, beyond in the workspace slot; the number of per-energy
 * workspace slots is capped at 48 GB, so very large nch runs fewer energies concurrently).
 */
rmx_rc rmx_match_K(rmx_ctx *ctx, const double *R, const double *F, const double *G,
                   const double *Fp, const double *Gp, double a, int64_t nch, int64_t ne,
                   const int32_t *n_open, double *K, int32_t *status);

/*
 * rmx_collision_strength - S5: T = 2i K_oo (I - i K_oo)^{-1}, o = n_open (BASELINE.json:5;
 * DESIGN.md reading T2): with A = I - i K_oo, T = 2(A^{-1} - I); A^{-1} from a complex-symmetric
 * LDL^T without pivoting (A's Hermitian part is I, so every pivot has Re d >= 1) per energy, FP64
 * DMMA GEMMs; |T_ij|^2 = 4 |(A^{-1})_ij - delta_ij|^2 (error ~u ||K_oo||, bitwise symmetric).
 *   K       DEVICE [ne][nch][nch] (only the open block is read)
 *   T2      DEVICE [ne][nch][nch] or NULL: |T|^2, open block top-left, 0 elsewhere
 *   rowsum  DEVICE [ne][nch] or NULL: sum_j |T_ij|^2 (0 for closed rows)
 *   status  DEVICE int32 [ne]: RMX_E_NONFINITE if a non-finite |T|^2 value arises
 */
rmx_rc rmx_collision_strength(rmx_ctx *ctx, const double *K, int64_t nch, int64_t ne,
                              const int32_t *n_open, double *T2, double *rowsum,
                              int32_t *status);

/*
 * rmx_collision_strength_levels - NEXT-2 of SURVEY.md §8(f) ("each block
 * represents a partial wave ... reduced to the time required for a single partial wave"):
 * level-pair collision strengths of one symmetry (partial wave), accumulated with weight g:
 *
 *     omega[e][a][b] += g * sum_{i in level a} sum_{j in level b} |T_ij(E_e)|^2
 *
 * for every pair of OPEN levels (a level is open when all its channels are < n_open[e]);
 * entries of closed levels are not touched. Summing calls over the symmetries of a sweep with
 * g_s = the symmetry's statistical weight gives Omega_ab(E) = sum_s g_s sum |T^s_ij|^2 (DESIGN.md
 * reading L1; the paper prints no formula). |T|^2 is formed as in rmx_collision_strength and
 * never stored.
 *   K            DEVICE [ne][nch][nch]
 *   n_open       DEVICE int32 [ne] or NULL (= all open)
 *   level_start  DEVICE int32 [nlevel + 1]: level a = channels [level_start[a], level_start[a+1]),
 *                0 = level_start[0] < level_start[1] < ... <= nch (channels sorted by threshold,
 *                the channels of a level contiguous; not checked on the host)
 *   omega        DEVICE [ne][nlevel][nlevel], caller-initialised (accumulated into)
 *   status       DEVICE int32 [ne] or NULL
 * Per (e, a, b) the sum runs i ascending then j ascending: deterministic, no atomics.
 * Errors: EINVAL on null K / level_start / omega, nlevel < 1, bad sizes.
 */
rmx_rc rmx_collision_strength_levels(rmx_ctx *ctx, const double *K, int64_t nch, int64_t ne,
                                     const int32_t *n_open, const int32_t *level_start,
                                     int64_t nlevel, double g, double *omega, int32_t *status);

/*
 * rmx_sweep - the fused streaming driver: for energies in batches of `batch`, runs
 * build_R -> match_K -> collision_strength on ctx workspace (R and K never leave the
 * device), writing only the per-energy summaries rowsum [ne][nch] and status [ne].
 * Per-energy arithmetic does not depend on the batch position or `batch`, so results are
 * bitwise identical for any batching / sharding.
 *   All array arguments DEVICE, shapes as above; F,G,Fp,Gp,n_open are per energy [ne].
 *   dump_idx  HOST int64 [n_dump] or NULL: energy indices (into [0, ne)) whose full R, K and
 *             |T|^2 are also written to R_d, K_d, T2_d (each DEVICE [n_dump][nch][nch] or NULL),
 *             in dump_idx order (the parity sample)
 *   batch <= 0 selects the default (a multiple of the SM count).
 */
rmx_rc rmx_sweep(rmx_ctx *ctx, const double *w, int64_t ldw, const double *Ek, int64_t nch,
                 int64_t nlev, double a, const double *E, int64_t ne, const double *F,
                 const double *G, const double *Fp, const double *Gp, const int32_t *n_open,
                 int64_t batch, const int64_t *dump_idx, int64_t n_dump, double *R_d,
                 double *K_d, double *T2_d, double *rowsum, int32_t *status);

/*
 * rmx_sweep_levels - rmx_sweep whose T epilogue also accumulates the level-pair collision
 * strengths of rmx_collision_strength_levels (omega [ne][nlevel][nlevel] += g * ...), fused:
 * |T|^2 never leaves the chip. One call per symmetry (partial wave) of a multi-symmetry sweep,
 * each with its own w, Ek, channels, F, G, F', G', n_open and level_start, the same E and omega.
 * rowsum [ne][nch] may be NULL. Same argument rules as rmx_sweep (no dump list).
 */
rmx_rc rmx_sweep_levels(rmx_ctx *ctx, const double *w, int64_t ldw, const double *Ek,
                        int64_t nch, int64_t nlev, double a, const double *E, int64_t ne,
                        const double *F, const double *G, const double *Fp, const double *Gp,
                        const int32_t *n_open, int64_t batch, const int32_t *level_start,
                        int64_t nlevel, double g, double *omega, double *rowsum,
                        int32_t *status);

/*
 * rmx_sweep_host - rmx_sweep with HOST inputs and outputs: copies w (as [nch][ldw]), Ek,
 * E, F, G, Fp, Gp, n_open host->device (staged through ctx pinned buffers), runs the sweep
 * and copies rowsum and status back, then synchronises the stream. status is fully
 * overwritten (initialised to RMX_E_OK internally). Used for the end-to-end measurement.
 * h2d_bytes / d2h_bytes (may be NULL) receive the bytes moved by this call.
 */
rmx_rc rmx_sweep_host(rmx_ctx *ctx, const double *w, int64_t ldw, const double *Ek,
                      int64_t nch, int64_t nlev, double a, const double *E, int64_t ne,
                      const double *F, const double *G, const double *Fp, const double *Gp,
                      const int32_t *n_open, int64_t batch, double *rowsum, int32_t *status,
                      int64_t *h2d_bytes, int64_t *d2h_bytes);

/* ---- NEXT-1 of SURVEY.md §8(f): the photoionisation variant of the sweep ------------------- *
 * PAPER.md:116-122, 148-156 (the bound-free dipole outer region PSTGBF0DAMP whose sweeps Tables 1-2
 * time). The paper prints no formula; readings P1-P4 give the R-matrix one used here:
 *   (9)  g_i(E) = sum_k w_ik d_k / (E_k - E)          d_k = <psi_k|D|Psi_0>, inner-region dipoles
 *   (10) v_j    = (1/2)(g_j F'_j + sum_i g_i G'_i K_ij), j < n_open   ((1/2) U'^T g, U = F + G K)
 *   (11) M      = (I - i K_oo)^{-1} v                  (ingoing-wave final states)
 *   (12) sigma  = C (E - E0) sum_j |M_j|^2            (C = 4 pi^2 alpha / 3 in atomic units)
 */

/*
 * rmx_dipole_amplitude - step (9) for ne energies: an energy-batched FP64 contraction with the
 * operand d_k/(E_k - E) generated on chip.
 *   w DEVICE [nch][ldw] (ldw >= nlev), Ek DEVICE [nlev], d DEVICE [nlev], E DEVICE [ne],
 *   g DEVICE [ne][nch] output, status DEVICE int32 [ne] or NULL (RMX_E_POLE, g = NaN, as build_R).
 */
rmx_rc rmx_dipole_amplitude(rmx_ctx *ctx, const double *w, int64_t ldw, const double *Ek,
                            const double *d, int64_t nch, int64_t nlev, const double *E, int64_t ne,
                            double *g, int32_t *status);

/*
 * rmx_photoionization - steps (10)-(12) from K (rmx_match_K output, all rows, closed columns -e_j)
 * and g: v, then M = (I - i K_oo)^{-1} v with the inverse of the T route (rmx_collision_strength),
 * per-channel |M_j|^2 and sigma.
 *   K DEVICE [ne][nch][nch]; g, Fp, Gp DEVICE [ne][nch]; E DEVICE [ne]; n_open DEVICE int32 [ne] or NULL
 *   E0     initial (bound) state energy: photon energy = E - E0
 *   C      cross-section prefactor (e.g. 4 pi^2 alpha / 3 = 0.0960769... in atomic units)
 *   sigma  DEVICE [ne] output;  mabs2 DEVICE [ne][nch] or NULL (|M_j|^2, 0 for closed channels)
 *   status DEVICE int32 [ne] or NULL: RMX_E_NONFINITE if |M|^2 is not finite
 */
rmx_rc rmx_photoionization(rmx_ctx *ctx, const double *K, const double *g, const double *Fp,
                           const double *Gp, const double *E, int64_t nch, int64_t ne,
                           const int32_t *n_open, double E0, double C, double *sigma,
                           double *mabs2, int32_t *status);

/*
 * rmx_sweep_photo - the fused photoionisation sweep: per batch R -> K (as rmx_sweep), g, then the
 * T-route inverse applied to v; only sigma [ne] (and optionally
 * mabs2 [ne][nch]) and status leave the device. Arguments as rmx_sweep plus d, E0, C.
 */
rmx_rc rmx_sweep_photo(rmx_ctx *ctx, const double *w, int64_t ldw, const double *Ek, const double *d,
                       int64_t nch, int64_t nlev, double a, const double *E, int64_t ne,
                       const double *F, const double *G, const double *Fp, const double *Gp,
                       const int32_t *n_open, int64_t batch, double E0, double C, double *sigma,
                       double *mabs2, int32_t *status);

/* ---- NEXT-3 of SURVEY.md §8(f): the inner-region step that feeds the sweep ------------------ */

/*
 * rmx_inner_region - full dense eigensolve of the (synthetic) inner-region Hamiltonian and the
 * boundary amplitudes of its eigenstates ("The diagonalization of each matrix,
 * from which every eigenvalue and every eigenvector is required ... pdsyevd"; SURVEY.md §8(f)
 * item 3): (E_k, V) = eigh(H) by cuSOLVER syevd (library, like the paper's ScaLAPACK pdsyevd),
 * then w = P^T V by one cuBLAS DGEMM, where P [nlev][nch] are the channel projections of the basis
 * at r = a. The outputs are exactly the (E_k, w) inputs of rmx_build_R / rmx_sweep:
 * (1/2a) W diag(1/(E_k - E)) W^T = (1/2a) P^T (H - E)^{-1} P.
 *   H    DEVICE [nlev][nlev]  symmetric (read only; the lower triangle is used)
 *   P    DEVICE [nlev][nch]
 *   Ek   DEVICE [nlev]        eigenvalues, ascending
 *   w    DEVICE [nch][ldw]    amplitudes (ldw >= nlev; columns nlev..ldw-1 untouched)
 * Eigenvector signs are those of the solver (R, K, T do not depend on them). Synchronous (waits
 * for the solver's info). Errors: EINVAL on null pointers / bad sizes; ECUDA if the solver fails.
 */
rmx_rc rmx_inner_region(rmx_ctx *ctx, const double *H, int64_t nlev, const double *P, int64_t nch,
                        double *Ek, double *w, int64_t ldw);

/* ---- NEXT-4 of SURVEY.md §8(f): post-processing on the energy mesh ------------------------ */

/* largest number of temperatures per rmx_maxwell_average call */
#define RMX_MAX_TEMPS 32

/*
 * rmx_convolve_gaussian - Gaussian convolution at a given FWHM with optional statistical
 * admixture (Fig. 1 caption "convoluted with a 60 meV FWHM Gaussian";
 * PAPER.md:370-373 Fig. 3 caption "appropriate Gaussian of FWHM and a statistical admixture of
 * 2/3 ground and 1/3 metastable states"; operational definition, C1):
 *     xbar = sum_m mix_m x_m / sum_m mix_m                  (mix == NULL: each spectrum alone)
 *     y_i  = sum_{|j-i|<=M, 0<=j<ne} g_{j-i} xbar_j / sum_{same j} g_{j-i}
 *     g_d  = exp(-(d dE)^2 / (2 s^2)), s = fwhm / (2 sqrt(2 ln 2)), M = floor(5 s / dE)
 * on a UNIFORM mesh of spacing dE (kernel truncated at +-5 s, renormalised at the mesh edges).
 *   x    DEVICE [nspec][ne]    spectra on the mesh (e.g. Omega_ab(E) or a row sum)
 *   mix  HOST [nspec] or NULL  admixture weights (>= 0, any scale: 2:1 == 2/3, 1/3)
 *   y    DEVICE [ne] if mix, else [nspec][ne]
 * Errors: EINVAL on null x/y, dE or fwhm <= 0, fwhm < 2 dE (SPEC.md:299 UnderResolvedKernel),
 * M > 9000, a negative weight or weights summing to 0, more than 64 admixture components.
 * Async on the ctx stream (mix is read on the host during the call).
 */
rmx_rc rmx_convolve_gaussian(rmx_ctx *ctx, const double *x, int64_t nspec, const double *mix,
                             int64_t ne, double dE, double fwhm, double *y);

/*
 * rmx_maxwell_average - Maxwellian-averaged (effective) collision strengths (SURVEY.md §8(f)
 * item 4; reading U1; the paper prints no formula):
 *     Ups_p(T) = int Omega_p(eps) exp(-eps/kT) d(eps/kT),  eps = E - Eth_p,
 * by the trapezoid rule over the mesh points with E_i > Eth_p (no extrapolation).
 *   omega  DEVICE [ne][npair]   Omega_p(E_i), row-major (pair fastest)
 *   E      DEVICE [ne]          ascending mesh (need not be uniform)
 *   Eth    DEVICE [npair]       excitation threshold of each pair (energy of the upper level)
 *   kT     HOST [nT]            temperatures (energy units of E), 1 <= nT <= RMX_MAX_TEMPS
 *   ups    DEVICE [npair][nT]   output
 * Deterministic (fixed-order chunked sums, no atomics). Errors: EINVAL on null pointers, sizes < 1,
 * nT out of range or kT <= 0.
 */
rmx_rc rmx_maxwell_average(rmx_ctx *ctx, const double *omega, int64_t ne, int64_t npair,
                           const double *E, const double *Eth, const double *kT, int64_t nT,
                           double *ups);

/* Synchronise ctx's stream; if n_bad_status/status given, counts nonzero entries of the
 * DEVICE int32 status[ne] (pass status=NULL to skip). Returns sticky CUDA errors. */
rmx_rc rmx_sync(rmx_ctx *ctx, const int32_t *status, int64_t ne, int64_t *n_bad);

/*
 * rmx_set_r_algo - choose how rmx_build_R / rmx_sweep* form R on this context:
 *   RMX_R_DMMA (default): the FP64 tensor-core (DMMA) contraction of rform.cu;
 *   RMX_R_INT8: the same R by exact integer arithmetic on the INT8 tensor cores (tcgen05 kind::i8):
 *     X = W diag(d) and W rounded to 55 / 53-bit fixed point per row, 16 modular INT8 GEMMs (CTA
 *     pairs, tcgen05.mma.cta_group::2, for nch > 256), CRT reconstruction (rint8.cu);
 *     R error at the level of an fp64 contraction (normwise ~1e-14). Applies for nch >= 256 and
 *     nlev <= 131071 (int32 accumulator bound); otherwise the DMMA contraction is used.
 *     Workspace ~ 2 x chunk x 16 x nch x nlev bytes (chunk = 8 energies, more for small nch).
 */
enum { RMX_R_DMMA = 0, RMX_R_INT8 = 1 };
rmx_rc rmx_set_r_algo(rmx_ctx *ctx, int algo);

/* ---- instrumentation (bench / roofline evidence; not needed for correctness) ----------
 * When enabled, every kernel launch is bracketed by cudaEvents on the ctx stream and its
 * duration accumulated per kernel id: 0 = R formation, 1 = matching, 2 = T epilogue,
 * 3 = other (post-processing, dipole amplitudes, eigensolve), 4 = the INT8 GEMM launches of the
 * RMX_R_INT8 R formation (a subset of 0's time). rmx_stats reads (total ms, launch count) per id and the
 * total number of kernel launches since the last reset (counted whether or not timing is
 * enabled). */
enum { RMX_KID_RFORM = 0, RMX_KID_MATCH = 1, RMX_KID_TEPI = 2, RMX_KID_OTHER = 3,
       RMX_KID_I8GEMM = 4 /* the INT8 tensor-core GEMMs inside R formation (RMX_R_INT8), also in RFORM */,
       RMX_NKID = 5 };
rmx_rc rmx_set_timing(rmx_ctx *ctx, int enable);
rmx_rc rmx_reset_stats(rmx_ctx *ctx);
rmx_rc rmx_stats(rmx_ctx *ctx, double *ms_per_kid /* [RMX_NKID] */,
                 int64_t *launches_per_kid /* [RMX_NKID] */, int64_t *total_launches);

/* Library version (major*10000 + minor*100 + patch) and the compiled SM target (100). */
int rmx_version(void);
int rmx_sm_target(void);

/* Host-only query (no GPU, no context): doubles of device workspace one in-flight energy of the
 * per-energy kernels (rmx_match_K, rmx_collision_strength*, rmx_photoionization) takes for nch
 * channels - the larger of the matching slot ([A | B_open] n x 2n_pad, a 128 x 128 block inverse, an
 * n x 9 LU sub-panel) and the T-epilogue slot (five n x ld_o planes and the d/v vectors), rounded up
 * to whole 128-byte lines so every slot base is 16-byte aligned for TMA. A context holds
 * min(#SMs, ne, 48 GB / slot) such slots. Returns -1 for nch < 1 or nch > 65536. */
int64_t rmx_workspace_doubles_per_energy(int64_t nch);

#ifdef __cplusplus
}
#endif
#endif /* RMX_H */
