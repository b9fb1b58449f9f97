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
            for f in (lib.oracle_R, lib.oracle_R_entries, lib.oracle_K, lib.oracle_T2,
                      lib.oracle_sweep, lib.oracle_max_threads):
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
