/*
 * rmx_oracle.c - plain, slow, obviously-correct CPU oracle for the outer-region energy
 * sweep R(E) -> K(E) -> |T(E)|^2 of arxiv 1403.5524 (McLaughlin & Ballance).
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product path (paper_1403_5524_b200/, librmx)
 * may include, link or call this file. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg use it. It shares no code, header,
 * table or helper with the CUDA path.
 *
 * Arithmetic: long double (x87 80-bit) accumulation throughout; outputs are rounded to
 * double once at the end. Algorithms are deliberately the textbook ones, in the paper's
 * / north_star's order, with no blocking, fusion or reordering:
 *
 *   (1) pole guard     : status POLE if min_k |E - E_k| < 1e-10 Ry
 *   (2) R_ij(E)        = (1/2a) sum_k w_ik w_jk / (E_k - E), ALL i,j computed independently,
 *                        ascending k (BASELINE.json:5 north_star form of PAPER.md:471-474 §6 Eq.1;
 *                        reading §8(c) 1-3 in DESIGN.md)
 *   (3) A_ij           = G_i d_ij - a R_ij G'_j ;  B_ij = F_i d_ij - a R_ij F'_j     (BASELINE.json:5)
 *   (4) K              = -A^{-1} B by Gaussian elimination with partial pivoting on A
 *                        (pivot = max |a_rk|, ties -> lowest row), applied to ALL nch columns of B
 *   (5) K_oo           = K[0:n_o, 0:n_o], n_o = #{eps_i < E} (given)
 *   (6) (I - i K_oo) X = K_oo by complex long double GE with partial pivoting; T = 2 i X
 *                        (= 2iK(I - iK)^{-1} since K and (I-iK)^{-1} commute; BASELINE.json:5)
 *   (7) |T_ij|^2 = Re^2 + Im^2 on the open block, 0 elsewhere; rowsum_i = sum_j |T_ij|^2
 *   (8) diagnostics    : unitarity max|S S^H - I| with S = I + T; max|K_oo - K_oo^T|; cond_1(A)
 *
 * NEXT-1 (photoionisation variant; DESIGN.md
 * readings P1-P4), per energy, after (4):
 *   (9)  g_i(E)  = sum_k w_ik d_k / (E_k - E)    (dipole amplitude contraction, ascending k)
 *   (10) v_j     = (1/2) (g_j F'_j + sum_i g_i G'_i K_ij),  j < n_o   (v = (1/2) U'^T g with the
 *                  standing-wave solutions U = F + G K of (4), derivatives at r = a)
 *   (11) (I - i K_oo) M = v by complex long double GE (ingoing-wave normalisation U (I - iK_oo)^-1)
 *   (12) |M_j|^2; sigma(E) = C (E - E0) sum_j |M_j|^2 (in oracle/__init__.py)
 *
 * Parallelism (OpenMP) only splits independent rows / energies; each output element sees
 * the same operation sequence for any thread count, so results are thread-count invariant.
 *
 * Parity pins for every function: tests/test_oracle_pins.py (closed forms, brute-force
 * (1/2a) P^T (H-E)^{-1} P, pole residue, K continuity across poles, symmetry, unitarity,
 * decoupled channels, closed-channel invariance). No function here is "parity unpinned"
 * except the diagnostics in (8), which are themselves checks, not outputs.
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef long double ld;
typedef long double complex cld;

enum { ORC_OK = 0, ORC_POLE = 1, ORC_SINGULAR = 2, ORC_NONFINITE = 3 };

#define POLE_GUARD 1e-10L

/* ---- (1)+(2) R-matrix pole sum ------------------------------------------------------ */

/* Returns ORC_POLE if E is within the guard of a pole, else fills R (nch*nch, long double). */
static int r_matrix_ld(const double *w, int64_t ldw, const double *Ek, int64_t nch,
                       int64_t nlev, double a, double E, ld *R, int inner_threads) {
  ld *d = (ld *)malloc(sizeof(ld) * (size_t)(nlev > 0 ? nlev : 1));
  int pole = 0;
  for (int64_t k = 0; k < nlev; ++k) {
    ld diff = (ld)Ek[k] - (ld)E;
    if (fabsl(diff) < POLE_GUARD) pole = 1;
    d[k] = 1.0L / diff; /* 1/(E_k - E) */
  }
  if (pole) {
    free(d);
    return ORC_POLE;
  }
  const ld inv2a = 1.0L / (2.0L * (ld)a);
#pragma omp parallel for schedule(dynamic, 1) num_threads(inner_threads) if (inner_threads > 1)
  for (int64_t i = 0; i < nch; ++i) {
    const double *wi = w + i * ldw;
    for (int64_t j = 0; j < nch; ++j) {
      const double *wj = w + j * ldw;
      ld s = 0.0L;
      for (int64_t k = 0; k < nlev; ++k) s += (ld)wi[k] * (ld)wj[k] * d[k];
      R[i * nch + j] = s * inv2a;
    }
  }
  free(d);
  return ORC_OK;
}

/* ---- (3)+(4) matching: K = -A^{-1} B ------------------------------------------------- */

/* In place: A (n*n) and B (n*m) long double; on exit B holds A^{-1} B. Row-major.
 * Gaussian elimination with partial pivoting, ties -> lowest row index. */
static int ge_solve_ld(ld *A, ld *B, int64_t n, int64_t m, int inner_threads) {
  int status = ORC_OK;
  for (int64_t c = 0; c < n; ++c) {
    int64_t p = c;
    ld best = fabsl(A[c * n + c]);
    for (int64_t r = c + 1; r < n; ++r) {
      ld v = fabsl(A[r * n + c]);
      if (v > best) { best = v; p = r; }
    }
    if (best == 0.0L) { status = ORC_SINGULAR; continue; }
    if (p != c) {
      for (int64_t j = 0; j < n; ++j) { ld t = A[c * n + j]; A[c * n + j] = A[p * n + j]; A[p * n + j] = t; }
      for (int64_t j = 0; j < m; ++j) { ld t = B[c * m + j]; B[c * m + j] = B[p * m + j]; B[p * m + j] = t; }
    }
    const ld piv = A[c * n + c];
#pragma omp parallel for schedule(static) num_threads(inner_threads) if (inner_threads > 1 && (n - c) * (n + m) > 65536)
    for (int64_t r = c + 1; r < n; ++r) {
      ld f = A[r * n + c] / piv;
      A[r * n + c] = 0.0L;
      if (f == 0.0L) continue;
      for (int64_t j = c + 1; j < n; ++j) A[r * n + j] -= f * A[c * n + j];
      for (int64_t j = 0; j < m; ++j) B[r * m + j] -= f * B[c * m + j];
    }
  }
  if (status != ORC_OK) return status;
  /* back substitution, U X = B */
  for (int64_t c = n - 1; c >= 0; --c) {
    const ld piv = A[c * n + c];
    for (int64_t j = 0; j < m; ++j) B[c * m + j] /= piv;
#pragma omp parallel for schedule(static) num_threads(inner_threads) if (inner_threads > 1 && c * m > 65536)
    for (int64_t r = 0; r < c; ++r) {
      ld f = A[r * n + c];
      if (f == 0.0L) continue;
      for (int64_t j = 0; j < m; ++j) B[r * m + j] -= f * B[c * m + j];
    }
  }
  return ORC_OK;
}

static void build_AB(const ld *R, const double *F, const double *G, const double *Fp,
                     const double *Gp, int64_t n, double a, ld *A, ld *B) {
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      ld aR = (ld)a * R[i * n + j];
      A[i * n + j] = (i == j ? (ld)G[i] : 0.0L) - aR * (ld)Gp[j];
      B[i * n + j] = (i == j ? (ld)F[i] : 0.0L) - aR * (ld)Fp[j];
    }
}

/* 1-norm of a square long double matrix */
static ld norm1(const ld *A, int64_t n) {
  ld best = 0.0L;
  for (int64_t j = 0; j < n; ++j) {
    ld s = 0.0L;
    for (int64_t i = 0; i < n; ++i) s += fabsl(A[i * n + j]);
    if (s > best) best = s;
  }
  return best;
}

/* K (n*n long double) from R. Optionally cond_1(A) (extra O(n^3) inverse). */
static int k_matrix_ld(const ld *R, const double *F, const double *G, const double *Fp,
                       const double *Gp, int64_t n, double a, ld *K, double *cond1,
                       int inner_threads) {
  size_t nn = (size_t)n * (size_t)n;
  ld *A = (ld *)malloc(sizeof(ld) * nn);
  build_AB(R, F, G, Fp, Gp, n, a, A, K);
  ld anorm = 0.0L;
  if (cond1) anorm = norm1(A, n);
  ld *Acopy = NULL;
  if (cond1) { Acopy = (ld *)malloc(sizeof(ld) * nn); memcpy(Acopy, A, sizeof(ld) * nn); }
  int st = ge_solve_ld(A, K, n, n, inner_threads);
  for (size_t t = 0; t < nn; ++t) K[t] = -K[t];
  if (cond1) {
    if (st == ORC_OK) {
      ld *Ainv = (ld *)calloc(nn, sizeof(ld));
      for (int64_t i = 0; i < n; ++i) Ainv[i * n + i] = 1.0L;
      ge_solve_ld(Acopy, Ainv, n, n, inner_threads);
      *cond1 = (double)(anorm * norm1(Ainv, n));
      free(Ainv);
    } else {
      *cond1 = INFINITY;
    }
    free(Acopy);
  }
  free(A);
  return st;
}

/* ---- (6)+(7) T = 2iK(I - iK)^{-1}, |T|^2 -------------------------------------------- */

static int ge_solve_cld(cld *A, cld *B, int64_t n, int64_t m, int inner_threads) {
  for (int64_t c = 0; c < n; ++c) {
    int64_t p = c;
    ld best = cabsl(A[c * n + c]);
    for (int64_t r = c + 1; r < n; ++r) {
      ld v = cabsl(A[r * n + c]);
      if (v > best) { best = v; p = r; }
    }
    if (best == 0.0L) return ORC_SINGULAR;
    if (p != c) {
      for (int64_t j = 0; j < n; ++j) { cld t = A[c * n + j]; A[c * n + j] = A[p * n + j]; A[p * n + j] = t; }
      for (int64_t j = 0; j < m; ++j) { cld t = B[c * m + j]; B[c * m + j] = B[p * m + j]; B[p * m + j] = t; }
    }
    const cld piv = A[c * n + c];
#pragma omp parallel for schedule(static) num_threads(inner_threads) if (inner_threads > 1 && (n - c) * (n + m) > 16384)
    for (int64_t r = c + 1; r < n; ++r) {
      cld f = A[r * n + c] / piv;
      A[r * n + c] = 0.0L;
      for (int64_t j = c + 1; j < n; ++j) A[r * n + j] -= f * A[c * n + j];
      for (int64_t j = 0; j < m; ++j) B[r * m + j] -= f * B[c * m + j];
    }
  }
  for (int64_t c = n - 1; c >= 0; --c) {
    const cld piv = A[c * n + c];
    for (int64_t j = 0; j < m; ++j) B[c * m + j] /= piv;
#pragma omp parallel for schedule(static) num_threads(inner_threads) if (inner_threads > 1 && c * m > 16384)
    for (int64_t r = 0; r < c; ++r) {
      cld f = A[r * n + c];
      for (int64_t j = 0; j < m; ++j) B[r * m + j] -= f * B[c * m + j];
    }
  }
  return ORC_OK;
}

/* K: n*n (long double, full); T written as complex long double o*o; diag: unitarity. */
static int t_matrix_cld(const ld *K, int64_t n, int64_t o, cld *T, double *unitarity,
                        int inner_threads) {
  if (o == 0) { if (unitarity) *unitarity = 0.0; return ORC_OK; }
  size_t oo = (size_t)o * (size_t)o;
  cld *M = (cld *)malloc(sizeof(cld) * oo);
  for (int64_t i = 0; i < o; ++i)
    for (int64_t j = 0; j < o; ++j) {
      M[i * o + j] = (i == j ? 1.0L : 0.0L) - I * K[i * n + j]; /* I - iK_oo */
      T[i * o + j] = K[i * n + j];                              /* RHS K_oo   */
    }
  int st = ge_solve_cld(M, T, o, o, inner_threads);
  for (size_t t = 0; t < oo; ++t) T[t] = 2.0L * I * T[t]; /* T = 2 i X */
  if (unitarity) {
    ld worst = 0.0L;
    for (int64_t i = 0; i < o; ++i)
      for (int64_t j = 0; j < o; ++j) {
        cld s = 0.0L;
        for (int64_t l = 0; l < o; ++l) {
          cld sil = (i == l ? 1.0L : 0.0L) + T[i * o + l];
          cld sjl = (j == l ? 1.0L : 0.0L) + T[j * o + l];
          s += sil * conjl(sjl);
        }
        s -= (i == j ? 1.0L : 0.0L);
        if (cabsl(s) > worst) worst = cabsl(s);
      }
    *unitarity = (double)worst;
  }
  free(M);
  return st;
}

/* ---- (9)-(11) photoionisation amplitudes (NEXT-1) ------------------------------------ */

/* g[nch] = sum_k w_ik d_k / (E_k - E) in long double, ascending k. */
static int dipole_g_ld(const double *w, int64_t ldw, const double *Ek, const double *d, int64_t nch,
                       int64_t nlev, double E, ld *g) {
  for (int64_t k = 0; k < nlev; ++k)
    if (fabsl((ld)Ek[k] - (ld)E) < POLE_GUARD) return ORC_POLE;
  for (int64_t i = 0; i < nch; ++i) {
    ld s = 0.0L;
    for (int64_t k = 0; k < nlev; ++k) s += (ld)w[i * ldw + k] * ((ld)d[k] / ((ld)Ek[k] - (ld)E));
    g[i] = s;
  }
  return ORC_OK;
}

/* K: full nch*nch (double, row-major, closed columns -e_j); M (complex, o entries) and |M|^2. */
static int photo_amp_ld(const double *K, int64_t n, int64_t o, const ld *g, const double *Fp,
                        const double *Gp, cld *M) {
  if (o == 0) return ORC_OK;
  cld *A = (cld *)malloc(sizeof(cld) * (size_t)o * (size_t)o);
  for (int64_t j = 0; j < o; ++j) {
    ld s = g[j] * (ld)Fp[j];
    for (int64_t i = 0; i < n; ++i) s += g[i] * (ld)Gp[i] * (ld)K[i * n + j];
    M[j] = 0.5L * s;                                                   /* v_j */
    for (int64_t l = 0; l < o; ++l)
      A[j * o + l] = (j == l ? 1.0L : 0.0L) - I * (ld)K[j * n + l];    /* I - iK_oo */
  }
  int st = ge_solve_cld(A, M, o, 1, 1);
  free(A);
  return st;
}

int oracle_dipole_g(const double *w, int64_t ldw, const double *Ek, const double *d, int64_t nch,
                    int64_t nlev, double E, double *g) {
  ld *gl = (ld *)malloc(sizeof(ld) * (size_t)nch);
  int st = dipole_g_ld(w, ldw, Ek, d, nch, nlev, E, gl);
  for (int64_t i = 0; i < nch; ++i) g[i] = st == ORC_OK ? (double)gl[i] : NAN;
  free(gl);
  return st;
}

/* M_re/M_im [n_open], mabs2 [nch] (0 for closed channels). g is taken in double (as stored). */
int oracle_photo(const double *K, int64_t nch, int64_t n_open, const double *g, const double *Fp,
                 const double *Gp, double *M_re, double *M_im, double *mabs2) {
  ld *gl = (ld *)malloc(sizeof(ld) * (size_t)nch);
  cld *M = (cld *)malloc(sizeof(cld) * (size_t)(n_open > 0 ? n_open : 1));
  for (int64_t i = 0; i < nch; ++i) gl[i] = g[i];
  int st = photo_amp_ld(K, nch, n_open, gl, Fp, Gp, M);
  for (int64_t j = 0; j < nch; ++j) {
    if (j < n_open) {
      M_re[j] = (double)creall(M[j]);
      M_im[j] = (double)cimagl(M[j]);
      mabs2[j] = (double)(creall(M[j]) * creall(M[j]) + cimagl(M[j]) * cimagl(M[j]));
    } else {
      mabs2[j] = 0.0;
    }
  }
  free(gl);
  free(M);
  return st;
}

/* ---- exported API ------------------------------------------------------------------ */

int oracle_version(void) { return 1; }

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* R at one energy; R out: double nch*nch. NaN on pole. */
int oracle_R(const double *w, int64_t ldw, const double *Ek, int64_t nch, int64_t nlev,
             double a, double E, double *R, int threads) {
  size_t nn = (size_t)nch * (size_t)nch;
  ld *Rl = (ld *)malloc(sizeof(ld) * nn);
  int st = r_matrix_ld(w, ldw, Ek, nch, nlev, a, E, Rl, threads);
  for (size_t t = 0; t < nn; ++t) R[t] = st == ORC_OK ? (double)Rl[t] : NAN;
  free(Rl);
  return st;
}

/* Selected R entries R_{ij}(E) for pairs (ii[p], jj[p]), p < npairs (full-size sampling). */
int oracle_R_entries(const double *w, int64_t ldw, const double *Ek, int64_t nlev, double a,
                     double E, const int64_t *ii, const int64_t *jj, int64_t npairs,
                     double *out) {
  for (int64_t k = 0; k < nlev; ++k)
    if (fabsl((ld)Ek[k] - (ld)E) < POLE_GUARD) {
      for (int64_t p = 0; p < npairs; ++p) out[p] = NAN;
      return ORC_POLE;
    }
  const ld inv2a = 1.0L / (2.0L * (ld)a);
  for (int64_t p = 0; p < npairs; ++p) {
    const double *wi = w + ii[p] * ldw, *wj = w + jj[p] * ldw;
    ld s = 0.0L;
    for (int64_t k = 0; k < nlev; ++k) s += (ld)wi[k] * (ld)wj[k] * (1.0L / ((ld)Ek[k] - (ld)E));
    out[p] = (double)(s * inv2a);
  }
  return ORC_OK;
}

/* K from a given (double) R; K out: double nch*nch (all columns). */
int oracle_K(const double *R, const double *F, const double *G, const double *Fp,
             const double *Gp, int64_t nch, double a, double *K, double *cond1, int threads) {
  size_t nn = (size_t)nch * (size_t)nch;
  ld *Rl = (ld *)malloc(sizeof(ld) * nn), *Kl = (ld *)malloc(sizeof(ld) * nn);
  for (size_t t = 0; t < nn; ++t) Rl[t] = (ld)R[t];
  int st = k_matrix_ld(Rl, F, G, Fp, Gp, nch, a, Kl, cond1, threads);
  for (size_t t = 0; t < nn; ++t) K[t] = (double)Kl[t];
  free(Rl);
  free(Kl);
  return st;
}

/* |T|^2 (nch*nch, open block top-left, zeros elsewhere) and rowsum (nch) from a given K. */
int oracle_T2(const double *K, int64_t nch, int64_t n_open, double *T2, double *rowsum,
              double *Tre, double *Tim, double *unitarity, int threads) {
  size_t nn = (size_t)nch * (size_t)nch, oo = (size_t)n_open * (size_t)n_open;
  ld *Kl = (ld *)malloc(sizeof(ld) * nn);
  for (size_t t = 0; t < nn; ++t) Kl[t] = (ld)K[t];
  cld *T = (cld *)malloc(sizeof(cld) * (oo ? oo : 1));
  int st = t_matrix_cld(Kl, nch, n_open, T, unitarity, threads);
  for (int64_t i = 0; i < nch; ++i) {
    ld s = 0.0L;
    for (int64_t j = 0; j < nch; ++j) {
      ld v = 0.0L, re = 0.0L, im = 0.0L;
      if (i < n_open && j < n_open) {
        re = creall(T[i * n_open + j]);
        im = cimagl(T[i * n_open + j]);
        v = re * re + im * im;
      }
      if (T2) T2[i * nch + j] = (double)v;
      if (Tre) Tre[i * nch + j] = (double)re;
      if (Tim) Tim[i * nch + j] = (double)im;
      s += v;
    }
    if (rowsum) rowsum[i] = (double)s;
  }
  free(Kl);
  free(T);
  return st;
}

/* One energy end to end, long double throughout. Any of R, K, T2, rowsum may be NULL. */
static int sweep_one(const double *w, int64_t ldw, const double *Ek, int64_t nch, int64_t nlev,
                     double a, double E, const double *F, const double *G, const double *Fp,
                     const double *Gp, int64_t n_open, double *R, double *K, double *T2,
                     double *rowsum, double *diag, int threads) {
  size_t nn = (size_t)nch * (size_t)nch, oo = (size_t)n_open * (size_t)n_open;
  ld *Rl = (ld *)malloc(sizeof(ld) * nn), *Kl = (ld *)malloc(sizeof(ld) * nn);
  int st = r_matrix_ld(w, ldw, Ek, nch, nlev, a, E, Rl, threads);
  if (st == ORC_POLE) {
    for (size_t t = 0; t < nn; ++t) {
      if (R) R[t] = NAN;
      if (K) K[t] = NAN;
      if (T2) T2[t] = NAN;
    }
    if (rowsum) for (int64_t i = 0; i < nch; ++i) rowsum[i] = NAN;
    free(Rl); free(Kl);
    return st;
  }
  double cond1 = 0.0, *pcond = (diag ? &cond1 : NULL);
  st = k_matrix_ld(Rl, F, G, Fp, Gp, nch, a, Kl, pcond, threads);
  cld *T = (cld *)malloc(sizeof(cld) * (oo ? oo : 1));
  double unit = 0.0;
  int st2 = t_matrix_cld(Kl, nch, n_open, T, diag ? &unit : NULL, threads);
  if (st == ORC_OK) st = st2;
  ld kmax = 0.0L, asym = 0.0L;
  for (int64_t i = 0; i < n_open; ++i)
    for (int64_t j = 0; j < n_open; ++j) {
      if (fabsl(Kl[i * nch + j]) > kmax) kmax = fabsl(Kl[i * nch + j]);
      ld dd = fabsl(Kl[i * nch + j] - Kl[j * nch + i]);
      if (dd > asym) asym = dd;
    }
  int finite = 1;
  for (int64_t i = 0; i < nch; ++i) {
    ld s = 0.0L;
    for (int64_t j = 0; j < nch; ++j) {
      ld v = 0.0L;
      if (i < n_open && j < n_open) {
        ld re = creall(T[i * n_open + j]), im = cimagl(T[i * n_open + j]);
        v = re * re + im * im;
      }
      if (!isfinite((double)v)) finite = 0;
      if (T2) T2[i * nch + j] = (double)v;
      s += v;
      if (R) R[i * nch + j] = (double)Rl[i * nch + j];
      if (K) K[i * nch + j] = (double)Kl[i * nch + j];
    }
    if (rowsum) rowsum[i] = (double)s;
  }
  if (st == ORC_OK && !finite) st = ORC_NONFINITE;
  if (diag) {
    diag[0] = unit;
    diag[1] = kmax > 0 ? (double)(asym / kmax) : 0.0;
    diag[2] = cond1;
  }
  free(Rl); free(Kl); free(T);
  return st;
}

/*
 * Sweep over the selected energy indices idx[0..n_idx). Inputs are full-mesh arrays:
 *   E [ne], F/G/Fp/Gp [ne][nch], n_open [ne]. Outputs are per selected energy p:
 *   R/K/T2 [n_idx][nch][nch] (each may be NULL), rowsum [n_idx][nch] (may be NULL),
 *   status [n_idx], diag [n_idx][3] (may be NULL: unitarity, asym(K_oo), cond_1(A)).
 * threads: total OpenMP threads. Small problems parallelise over energies, large ones
 * over rows inside each energy (identical arithmetic either way).
 */
int oracle_sweep(const double *w, int64_t ldw, const double *Ek, int64_t nch, int64_t nlev,
                 double a, const double *E, const double *F, const double *G,
                 const double *Fp, const double *Gp, const int32_t *n_open,
                 const int64_t *idx, int64_t n_idx, double *R, double *K, double *T2,
                 double *rowsum, int32_t *status, double *diag, int threads) {
  if (threads < 1) threads = 1;
  size_t nn = (size_t)nch * (size_t)nch;
  int outer = (nch < 160 && n_idx > 1);
  if (outer) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(threads)
    for (int64_t p = 0; p < n_idx; ++p) {
      int64_t e = idx[p];
      status[p] = sweep_one(w, ldw, Ek, nch, nlev, a, E[e], F + e * nch, G + e * nch,
                            Fp + e * nch, Gp + e * nch, n_open ? n_open[e] : nch,
                            R ? R + p * nn : NULL, K ? K + p * nn : NULL,
                            T2 ? T2 + p * nn : NULL, rowsum ? rowsum + p * nch : NULL,
                            diag ? diag + 3 * p : NULL, 1);
    }
  } else {
    for (int64_t p = 0; p < n_idx; ++p) {
      int64_t e = idx[p];
      status[p] = sweep_one(w, ldw, Ek, nch, nlev, a, E[e], F + e * nch, G + e * nch,
                            Fp + e * nch, Gp + e * nch, n_open ? n_open[e] : nch,
                            R ? R + p * nn : NULL, K ? K + p * nn : NULL,
                            T2 ? T2 + p * nn : NULL, rowsum ? rowsum + p * nch : NULL,
                            diag ? diag + 3 * p : NULL, threads);
    }
  }
  return ORC_OK;
}
