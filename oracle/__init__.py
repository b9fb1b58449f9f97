"""CPU oracle for the outer-region sweep R(E) -> K(E) -> |T(E)|^2 (arxiv 1403.5524).

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The product path
(``paper_1403_5524_b200``) never imports it and shares no code with it.

The arithmetic lives in ``rmx_oracle.c`` (plain C, long double, OpenMP over independent
rows / energies); this module only compiles it with gcc and marshals numpy arrays.
Each function cites the passage it follows; see the C header comment for the steps.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rmx_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

STATUS = {0: "OK", 1: "POLE", 2: "SINGULAR", 3: "NONFINITE"}


def build(force: bool = False) -> str:
    """Compile rmx_oracle.c -> liboracle.so with gcc (-O2 -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=gnu11",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            d, i64, i32 = ctypes.c_double, ctypes.c_int64, ctypes.c_int
            P = ctypes.c_void_p
            lib.oracle_R.argtypes = [P, i64, P, i64, i64, d, d, P, i32]
            lib.oracle_R_entries.argtypes = [P, i64, P, i64, d, d, P, P, i64, P]
            lib.oracle_K.argtypes = [P, P, P, P, P, i64, d, P, P, i32]
            lib.oracle_T2.argtypes = [P, i64, i64, P, P, P, P, P, i32]
            lib.oracle_sweep.argtypes = [P, i64, P, i64, i64, d, P, P, P, P, P, P, P, i64,
                                         P, P, P, P, P, P, i32]
            lib.oracle_dipole_g.argtypes = [P, i64, P, P, i64, i64, d, P]
            lib.oracle_photo.argtypes = [P, i64, i64, P, P, P, P, P, P]
            for f in (lib.oracle_R, lib.oracle_R_entries, lib.oracle_K, lib.oracle_T2,
                      lib.oracle_sweep, lib.oracle_max_threads, lib.oracle_dipole_g, lib.oracle_photo):
                f.restype = ctypes.c_int
            _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


def R(w, Ek, a, E, threads: int = 1):
    """R_ij(E) = (1/2a) sum_k w_ik w_jk/(E_k - E) (BASELINE.json:5; Eq. 1).
    Returns (R [nch,nch] float64, status)."""
    w, Ek = _f64(w), _f64(Ek)
    nch, nlev = w.shape
    out = np.empty((nch, nch))
    st = _load().oracle_R(_p(w), nlev, _p(Ek), nch, nlev, float(a), float(E), _p(out), threads)
    return out, st


def R_entries(w, Ek, a, E, ii, jj):
    """Selected entries R_{ii[p], jj[p]}(E), for sampled parity at full size."""
    w, Ek = _f64(w), _f64(Ek)
    ii = np.ascontiguousarray(ii, dtype=np.int64)
    jj = np.ascontiguousarray(jj, dtype=np.int64)
    out = np.empty(len(ii))
    st = _load().oracle_R_entries(_p(w), w.shape[1], _p(Ek), w.shape[1], float(a), float(E),
                                  _p(ii), _p(jj), len(ii), _p(out))
    return out, st


def K(R_, F, G, Fp, Gp, a, want_cond: bool = False, threads: int = 1):
    """K = -(G - aRG')^{-1}(F - aRF') (BASELINE.json:5), all nch columns.
    Returns (K, status, cond_1(A) or None)."""
    R_ = _f64(R_)
    n = R_.shape[0]
    F, G, Fp, Gp = (_f64(x) for x in (F, G, Fp, Gp))
    out = np.empty((n, n))
    c = np.zeros(1)
    st = _load().oracle_K(_p(R_), _p(F), _p(G), _p(Fp), _p(Gp), n, float(a), _p(out),
                          _p(c) if want_cond else None, threads)
    return out, st, (float(c[0]) if want_cond else None)


def T2(K_, n_open: int, threads: int = 1):
    """T = 2iK_oo(I - iK_oo)^{-1} (BASELINE.json:5) -> (|T|^2 [nch,nch], rowsum [nch],
    ReT, ImT, unitarity max|SS^H - I|, status)."""
    K_ = _f64(K_)
    n = K_.shape[0]
    t2, rs, tre, tim = np.empty((n, n)), np.empty(n), np.empty((n, n)), np.empty((n, n))
    u = np.zeros(1)
    st = _load().oracle_T2(_p(K_), n, int(n_open), _p(t2), _p(rs), _p(tre), _p(tim), _p(u),
                           threads)
    return t2, rs, tre, tim, float(u[0]), st


def sweep(w, Ek, a, E, F, G, Fp, Gp, n_open, idx, want=("R", "K", "T2", "rowsum"),
          diag: bool = False, threads: int | None = None):
    """Oracle sweep over mesh indices ``idx`` (full-mesh input arrays, long double end to
    end). Returns dict with the requested outputs [n_idx, ...], 'status' and, if diag,
    'diag' [n_idx, 3] = (unitarity, asym(K_oo), cond_1(A))."""
    w, Ek, E = _f64(w), _f64(Ek), _f64(E)
    F, G, Fp, Gp = (_f64(x) for x in (F, G, Fp, Gp))
    nch, nlev = w.shape
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    n = len(idx)
    no = None if n_open is None else np.ascontiguousarray(n_open, dtype=np.int32)
    res = {}
    for k in ("R", "K", "T2"):
        res[k] = np.empty((n, nch, nch)) if k in want else None
    res["rowsum"] = np.empty((n, nch)) if "rowsum" in want else None
    res["status"] = np.empty(n, dtype=np.int32)
    res["diag"] = np.empty((n, 3)) if diag else None
    _load().oracle_sweep(_p(w), nlev, _p(Ek), nch, nlev, float(a), _p(E), _p(F), _p(G),
                         _p(Fp), _p(Gp), _p(no), _p(idx), n, _p(res["R"]), _p(res["K"]),
                         _p(res["T2"]), _p(res["rowsum"]), _p(res["status"]),
                         _p(res["diag"]), int(threads or default_threads()))
    return {k: v for k, v in res.items() if v is not None}


def level_omega(T2_, level_start, n_open: int, g: float = 1.0):
    """Level-pair collision strengths of one symmetry (
    DESIGN.md reading L1): Omega_ab = g * sum_{i in a} sum_{j in b} |T_ij|^2 for the open levels
    (all channels of the level < n_open), 0 for pairs involving a closed level. Plain loops over
    the definition with long-double accumulation; T2_ is the oracle's |T|^2 [nch, nch]."""
    ls = [int(x) for x in level_start]
    nlevel = len(ls) - 1
    om = np.zeros((nlevel, nlevel))
    T2l = np.asarray(T2_, dtype=np.longdouble)
    for la in range(nlevel):
        if ls[la + 1] > n_open:
            continue
        for lb in range(nlevel):
            if ls[lb + 1] > n_open:
                continue
            acc = T2l[ls[la]:ls[la + 1], ls[lb]:ls[lb + 1]].sum()  # the block's entries
            om[la, lb] = float(np.longdouble(g) * acc)
    return om


def convolve_gaussian(x, dE: float, fwhm: float, mix=None):
    """Gaussian convolution with statistical admixture (PAPER.md:298-300, 370-373 figure captions;
    operational definition; reading C1), written out per output point:
    s = fwhm/(2 sqrt(2 ln 2)), M = floor(5 s/dE), y_i = sum_j g(E_j - E_i) xbar_j / sum_j g(E_j - E_i)
    over 0 <= j < ne with |j - i| <= M, g(u) = exp(-u^2/(2 s^2)), xbar = sum_m c_m x_m / sum_m c_m.
    Long-double accumulation, j ascending. x: [nspec, ne] or [ne]."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    nspec, ne = x.shape
    if mix is not None:
        c = np.asarray(mix, dtype=np.longdouble)
        xs = [(c[:, None] * x.astype(np.longdouble)).sum(axis=0) / c.sum()]
    else:
        xs = [x[m].astype(np.longdouble) for m in range(nspec)]
    s = fwhm / (2.0 * np.sqrt(2.0 * np.log(2.0)))
    M = int(np.floor(5.0 * s / dE))
    d = np.arange(-M, M + 1)
    g = np.exp(-((d * dE) ** 2) / (2.0 * s * s)).astype(np.longdouble)
    out = np.empty((len(xs), ne))
    for m, xb in enumerate(xs):
        for i in range(ne):
            lo, hi = max(0, i - M), min(ne - 1, i + M)
            gw = g[lo - i + M:hi - i + M + 1]
            out[m, i] = float((gw * xb[lo:hi + 1]).sum() / gw.sum())
    return out[0] if mix is not None else out


def maxwell_average(omega, E, Eth, kT):
    """Maxwellian average Ups_p(T) = int Omega_p(eps) e^{-eps/kT} d(eps/kT), eps = E - Eth_p
    (reading U1), by the trapezoid rule over the mesh points with
    E_i > Eth_p: sum over intervals (E_{i+1} - E_i)(f_i + f_{i+1})/2, f = Omega e^{-eps/kT}/kT.
    omega: [ne, npair]; returns [npair, nT]."""
    omega = np.asarray(omega, dtype=np.float64)
    E = np.asarray(E, dtype=np.longdouble)
    ne, npair = omega.shape
    out = np.zeros((npair, len(kT)))
    for p in range(npair):
        first = int(np.searchsorted(np.asarray(E, dtype=np.float64), Eth[p], side="right"))
        for t, kt in enumerate(kT):
            kt = np.longdouble(kt)
            f = omega[first:, p].astype(np.longdouble) * np.exp(-(E[first:] - np.longdouble(Eth[p])) / kt) / kt
            Ei = E[first:]
            acc = ((Ei[1:] - Ei[:-1]) * (f[:-1] + f[1:]) / 2).sum()  # the trapezoids, summed
            out[p, t] = float(acc)
    return out


def inner_region(H, P):
    """Inner-region step feeding the sweep ('every eigenvalue and every
    eigenvector is required', ScaLAPACK pdsyevd): (E_k, V) = eigh(H)
    (LAPACK via numpy - a library primitive used as the step), w = P^T V. Returns (Ek, w [nch, nlev])."""
    Ek, V = np.linalg.eigh(np.asarray(H, dtype=np.float64))
    return Ek, np.ascontiguousarray(np.asarray(P, dtype=np.float64).T @ V)


FINE_STRUCTURE_ALPHA = 1.0 / 137.035999084  # CODATA 2018
SIGMA_PREFACTOR = 4.0 * np.pi ** 2 * FINE_STRUCTURE_ALPHA / 3.0  # DESIGN.md reading P4 (a.u.)


def dipole_g(w, Ek, d, E):
    """NEXT-1 step (9): g_i(E) = sum_k w_ik d_k/(E_k - E) (the outer-region dipole amplitude
    contraction of SURVEY.md §8(f) item 1). Returns (g [nch], status)."""
    w, Ek, d = _f64(w), _f64(Ek), _f64(d)
    nch, nlev = w.shape
    g = np.empty(nch)
    st = _load().oracle_dipole_g(_p(w), nlev, _p(Ek), _p(d), nch, nlev, float(E), _p(g))
    return g, st


def photo(K_, n_open: int, g, Fp, Gp):
    """NEXT-1 steps (10)-(11): v = (1/2) U'^T g over the open solutions, (I - iK_oo) M = v by
    complex GE. Returns (M complex [n_open], |M_j|^2 [nch] (0 on closed channels), status)."""
    K_ = _f64(K_)
    n = K_.shape[0]
    g, Fp, Gp = _f64(g), _f64(Fp), _f64(Gp)
    mr, mi, m2 = np.zeros(max(n_open, 1)), np.zeros(max(n_open, 1)), np.empty(n)
    st = _load().oracle_photo(_p(K_), n, int(n_open), _p(g), _p(Fp), _p(Gp), _p(mr), _p(mi), _p(m2))
    return (mr + 1j * mi)[:n_open], m2, st


def photo_sweep(w, Ek, d, a, E, F, G, Fp, Gp, n_open, E0, C=SIGMA_PREFACTOR, threads=None):
    """NEXT-1 end to end on each energy of E: R (2) -> K (4) -> g (9) -> M (10-11) ->
    sigma = C (E - E0) sum_j |M_j|^2 (12). Returns dict(sigma [ne], mabs2 [ne, nch], g [ne, nch],
    status [ne])."""
    E = _f64(E)
    ne = len(E)
    nch = np.asarray(w).shape[0]
    no = np.asarray(n_open, dtype=np.int32)
    ks = sweep(w, Ek, a, E, F, G, Fp, Gp, no, np.arange(ne), want=("K",), threads=threads)
    out = {"sigma": np.empty(ne), "mabs2": np.empty((ne, nch)), "g": np.empty((ne, nch)),
           "status": ks["status"].copy()}
    for e in range(ne):
        g, st = dipole_g(w, Ek, d, E[e])
        M, m2, st2 = photo(ks["K"][e], int(no[e]), g, Fp[e], Gp[e])
        out["g"][e], out["mabs2"][e] = g, m2
        out["sigma"][e] = float(np.longdouble(C) * (np.longdouble(E[e]) - np.longdouble(E0)) *
                                np.sum(m2.astype(np.longdouble)))
        if out["status"][e] == 0:
            out["status"][e] = st or st2
    return out
