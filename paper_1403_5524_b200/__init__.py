"""paper_1403_5524_b200 - B200-native outer-region R-matrix energy sweep (arxiv 1403.5524).

Thin Python binding over the C-ABI library ``librmx.so`` (declared in ``include/rmx.h``):
argument marshalling only. Every step of R(E) -> K(E) -> |T(E)|^2 runs in the sm_100a CUDA
kernels of ``csrc/``; PyTorch supplies device memory, the current CUDA stream and (in
``paper_1403_5524_b200.dist``) process groups. There is no CPU or PyTorch fallback: if the
library is missing or no CUDA device is present the calls raise.

    import paper_1403_5524_b200 as rmx
    ctx = rmx.Context()                       # on torch.cuda.current_device()
    R, st = ctx.build_R(w, Ek, a, E)          # rmx_build_R
    K, st = ctx.match_K(R, F, G, Fp, Gp, a, n_open, status=st)       # rmx_match_K
    T2, rs, st = ctx.collision_strength(K, n_open, status=st)         # rmx_collision_strength
    out = ctx.sweep(w, Ek, a, E, F, G, Fp, Gp, n_open)                # rmx_sweep (fused driver)
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RMX_LIB", os.path.join(_PKG, "librmx.so"))

RMX_OK, RMX_EINVAL, RMX_ENOMEM, RMX_ECUDA = 0, 1, 2, 3
E_OK, E_POLE, E_SINGULAR, E_NONFINITE = 0, 1, 2, 3
KID_RFORM, KID_MATCH, KID_TEPI, KID_OTHER, KID_I8GEMM = 0, 1, 2, 3, 4
KID_NAMES = ("rform", "match", "tepi", "other", "i8gemm")
NKID = len(KID_NAMES)
R_DMMA, R_INT8 = 0, 1

# every symbol include/rmx.h declares (tests/test_abi.py checks the header and the .so agree)
EXPORTED = ("rmx_create", "rmx_destroy", "rmx_set_stream", "rmx_last_error", "rmx_build_R",
            "rmx_match_K", "rmx_collision_strength", "rmx_collision_strength_levels", "rmx_sweep",
            "rmx_sweep_levels", "rmx_sweep_host", "rmx_dipole_amplitude", "rmx_photoionization",
            "rmx_sweep_photo", "rmx_inner_region", "rmx_convolve_gaussian",
            "rmx_maxwell_average",
            "rmx_sync",
            "rmx_set_r_algo", "rmx_set_timing", "rmx_reset_stats", "rmx_stats", "rmx_version",
            "rmx_sm_target", "rmx_workspace_doubles_per_energy")


class RmxError(RuntimeError):
    pass


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """dlopen librmx.so and declare the C signatures (no CUDA call is made here)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"librmx.so not built at {path}: run `python -m paper_1403_5524_b200.build`"
                          " (no CPU fallback exists)")
    lib = ctypes.CDLL(path)
    P, i64, d, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    sig = {
        "rmx_create": [ctypes.POINTER(P), i32, P],
        "rmx_destroy": [P],
        "rmx_set_stream": [P, P],
        "rmx_build_R": [P, P, i64, P, i64, i64, d, P, i64, P, P],
        "rmx_match_K": [P, P, P, P, P, P, d, i64, i64, P, P, P],
        "rmx_collision_strength": [P, P, i64, i64, P, P, P, P],
        "rmx_collision_strength_levels": [P, P, i64, i64, P, P, i64, d, P, P],
        "rmx_sweep": [P, P, i64, P, i64, i64, d, P, i64, P, P, P, P, P, i64, P, i64, P, P, P, P, P],
        "rmx_sweep_levels": [P, P, i64, P, i64, i64, d, P, i64, P, P, P, P, P, i64, P, i64, d, P, P,
                             P],
        "rmx_sweep_host": [P, P, i64, P, i64, i64, d, P, i64, P, P, P, P, P, i64, P, P, P, P],
        "rmx_inner_region": [P, P, i64, P, i64, P, P, i64],
        "rmx_dipole_amplitude": [P, P, i64, P, P, i64, i64, P, i64, P, P],
        "rmx_photoionization": [P, P, P, P, P, P, i64, i64, P, d, d, P, P, P],
        "rmx_sweep_photo": [P, P, i64, P, P, i64, i64, d, P, i64, P, P, P, P, P, i64, d, d, P, P, P],
        "rmx_convolve_gaussian": [P, P, i64, P, i64, d, d, P],
        "rmx_maxwell_average": [P, P, i64, i64, P, P, P, i64, P],
        "rmx_sync": [P, P, i64, P],
        "rmx_set_timing": [P, i32],
        "rmx_set_r_algo": [P, i32],
        "rmx_reset_stats": [P],
        "rmx_stats": [P, P, P, P],
    }
    for name, args in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    lib.rmx_last_error.argtypes = [P]
    lib.rmx_last_error.restype = ctypes.c_char_p
    lib.rmx_version.restype = ctypes.c_int
    lib.rmx_sm_target.restype = ctypes.c_int
    lib.rmx_workspace_doubles_per_energy.argtypes = [ctypes.c_int64]
    lib.rmx_workspace_doubles_per_energy.restype = ctypes.c_int64
    _lib = lib
    return lib


def _torch():
    import torch
    return torch


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


class Context:
    """An rmx_ctx bound to one CUDA device; calls enqueue on torch's current stream."""

    def __init__(self, device: Optional[int] = None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RmxError("no CUDA device: librmx has no CPU fallback")
        self.lib = load_library()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self._h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            st = torch.cuda.current_stream().cuda_stream
        rc = self.lib.rmx_create(ctypes.byref(self._h), self.device, ctypes.c_void_p(st))
        if rc != RMX_OK:
            raise RmxError(f"rmx_create failed (rc={rc})")

    # ------------------------------------------------------------------ plumbing
    def close(self):
        if self._h:
            self.lib.rmx_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _bind_stream(self):
        torch = _torch()
        self.lib.rmx_set_stream(self._h, ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream))

    def _check(self, rc: int, what: str):
        if rc != RMX_OK:
            msg = self.lib.rmx_last_error(self._h)
            raise RmxError(f"{what}: rc={rc}: {msg.decode() if msg else ''}")

    def _dev(self, x, dtype):
        torch = _torch()
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x))
        t = x.to(device=f"cuda:{self.device}", dtype=dtype)
        return t.contiguous()

    def prepare_w(self, w):
        """Device copy of w with an even leading dimension (TMA stride rule, rmx.h)."""
        torch = _torch()
        w = self._dev(w, torch.float64)
        nch, nlev = w.shape
        ldw = nlev + (nlev & 1)
        if ldw != nlev or (w.data_ptr() % 16):
            buf = torch.zeros((nch, ldw), dtype=torch.float64, device=w.device)
            buf[:, :nlev] = w
            w = buf
        return w, nlev, ldw

    def _status(self, status, ne):
        torch = _torch()
        if status is None:
            return torch.zeros(ne, dtype=torch.int32, device=f"cuda:{self.device}")
        return status

    # ------------------------------------------------------------------ the three calls
    def build_R(self, w, Ek, a: float, E, status=None, out=None):
        """rmx_build_R: R[e] = (1/2a) W diag(1/(E_k - E_e)) W^T. Returns (R [ne,nch,nch], status)."""
        torch = _torch()
        self._bind_stream()
        w, nlev, ldw = self.prepare_w(w)
        Ek = self._dev(Ek, torch.float64)
        E = self._dev(E, torch.float64)
        nch, ne = w.shape[0], E.shape[0]
        R = out if out is not None else torch.empty((ne, nch, nch), dtype=torch.float64, device=w.device)
        status = self._status(status, ne)
        self._check(self.lib.rmx_build_R(self._h, _ptr(w), ldw, _ptr(Ek), nch, nlev, float(a), _ptr(E),
                                         ne, _ptr(R), _ptr(status)), "rmx_build_R")
        return R, status

    def match_K(self, R, F, G, Fp, Gp, a: float, n_open=None, status=None, out=None):
        """rmx_match_K: K[e] = -(G - aRG')^{-1}(F - aRF'). Returns (K [ne,nch,nch], status)."""
        torch = _torch()
        self._bind_stream()
        R = self._dev(R, torch.float64)
        F, G, Fp, Gp = (self._dev(x, torch.float64) for x in (F, G, Fp, Gp))
        ne, nch = R.shape[0], R.shape[1]
        no = None if n_open is None else self._dev(n_open, torch.int32)
        K = out if out is not None else torch.empty_like(R)
        status = self._status(status, ne)
        self._check(self.lib.rmx_match_K(self._h, _ptr(R), _ptr(F), _ptr(G), _ptr(Fp), _ptr(Gp),
                                         float(a), nch, ne, _ptr(no), _ptr(K), _ptr(status)),
                    "rmx_match_K")
        return K, status

    def collision_strength(self, K, n_open=None, status=None, want_T2: bool = True,
                           want_rowsum: bool = True):
        """rmx_collision_strength: |T|^2 with T = 2iK_oo(I - iK_oo)^{-1}.
        Returns (T2 [ne,nch,nch] or None, rowsum [ne,nch] or None, status)."""
        torch = _torch()
        self._bind_stream()
        K = self._dev(K, torch.float64)
        ne, nch = K.shape[0], K.shape[1]
        no = None if n_open is None else self._dev(n_open, torch.int32)
        T2 = torch.empty_like(K) if want_T2 else None
        rs = torch.empty((ne, nch), dtype=torch.float64, device=K.device) if want_rowsum else None
        status = self._status(status, ne)
        self._check(self.lib.rmx_collision_strength(self._h, _ptr(K), nch, ne, _ptr(no), _ptr(T2),
                                                    _ptr(rs), _ptr(status)),
                    "rmx_collision_strength")
        return T2, rs, status

    def collision_strength_levels(self, K, level_start, g: float = 1.0, n_open=None, omega=None,
                                  status=None):
        """rmx_collision_strength_levels: omega[e][a][b] += g sum_{i in a, j in b} |T_ij|^2 over
        the open levels. Returns (omega [ne,nlevel,nlevel], status)."""
        torch = _torch()
        self._bind_stream()
        K = self._dev(K, torch.float64)
        ne, nch = K.shape[0], K.shape[1]
        ls = self._dev(level_start, torch.int32)
        nlevel = ls.numel() - 1
        no = None if n_open is None else self._dev(n_open, torch.int32)
        if omega is None:
            omega = torch.zeros((ne, nlevel, nlevel), dtype=torch.float64, device=K.device)
        status = self._status(status, ne)
        self._check(self.lib.rmx_collision_strength_levels(
            self._h, _ptr(K), nch, ne, _ptr(no), _ptr(ls), nlevel, float(g), _ptr(omega),
            _ptr(status)), "rmx_collision_strength_levels")
        return omega, status

    # ------------------------------------------------------------------ fused drivers
    def sweep_levels(self, w, Ek, a: float, E, F, G, Fp, Gp, n_open, level_start, g: float = 1.0,
                     omega=None, rowsum=None, batch: int = 0, status=None, want_rowsum=False):
        """rmx_sweep_levels: the fused sweep of one symmetry accumulating
        omega[e][a][b] += g sum_{i in a, j in b} |T_ij(E_e)|^2. Returns dict(omega, rowsum, status)."""
        torch = _torch()
        self._bind_stream()
        w, nlev, ldw = self.prepare_w(w)
        Ek = self._dev(Ek, torch.float64)
        E = self._dev(E, torch.float64)
        F, G, Fp, Gp = (self._dev(x, torch.float64) for x in (F, G, Fp, Gp))
        n_open = None if n_open is None else self._dev(n_open, torch.int32)
        ls = self._dev(level_start, torch.int32)
        nlevel = ls.numel() - 1
        nch, ne = w.shape[0], E.shape[0]
        if omega is None:
            omega = torch.zeros((ne, nlevel, nlevel), dtype=torch.float64, device=w.device)
        if rowsum is None and want_rowsum:
            rowsum = torch.empty((ne, nch), dtype=torch.float64, device=w.device)
        status = self._status(status, ne)
        self._check(self.lib.rmx_sweep_levels(
            self._h, _ptr(w), ldw, _ptr(Ek), nch, nlev, float(a), _ptr(E), ne, _ptr(F), _ptr(G),
            _ptr(Fp), _ptr(Gp), _ptr(n_open), int(batch), _ptr(ls), nlevel, float(g), _ptr(omega),
            _ptr(rowsum), _ptr(status)), "rmx_sweep_levels")
        return {"omega": omega, "rowsum": rowsum, "status": status}

    def sweep(self, w, Ek, a: float, E, F, G, Fp, Gp, n_open=None, batch: int = 0,
              dump_idx: Optional[Sequence[int]] = None, status=None, rowsum=None, prepared=False):
        """rmx_sweep: R -> K -> |T|^2 for all energies; returns dict with rowsum [ne,nch], status
        [ne] and, for dump_idx, R/K/T2 [n_dump,nch,nch]."""
        torch = _torch()
        self._bind_stream()
        if prepared:
            nlev, ldw = int(prepared[0]), int(prepared[1])
        else:
            w, nlev, ldw = self.prepare_w(w)
            Ek = self._dev(Ek, torch.float64)
            E = self._dev(E, torch.float64)
            F, G, Fp, Gp = (self._dev(x, torch.float64) for x in (F, G, Fp, Gp))
            n_open = None if n_open is None else self._dev(n_open, torch.int32)
        nch, ne = w.shape[0], E.shape[0]
        dev = w.device
        rs = rowsum if rowsum is not None else torch.empty((ne, nch), dtype=torch.float64, device=dev)
        status = self._status(status, ne)
        nd = 0 if dump_idx is None else len(dump_idx)
        out = {"rowsum": rs, "status": status}
        didx = None
        Rd = Kd = T2d = None
        if nd:
            didx = np.ascontiguousarray(dump_idx, dtype=np.int64)
            Rd = torch.empty((nd, nch, nch), dtype=torch.float64, device=dev)
            Kd, T2d = torch.empty_like(Rd), torch.empty_like(Rd)
            out.update(R=Rd, K=Kd, T2=T2d)
        self._check(self.lib.rmx_sweep(
            self._h, _ptr(w), ldw, _ptr(Ek), nch, nlev, float(a), _ptr(E), ne, _ptr(F), _ptr(G),
            _ptr(Fp), _ptr(Gp), _ptr(n_open), int(batch),
            didx.ctypes.data_as(ctypes.c_void_p) if nd else None, nd, _ptr(Rd), _ptr(Kd), _ptr(T2d),
            _ptr(rs), _ptr(status)), "rmx_sweep")
        return out

    def sweep_host(self, w: np.ndarray, Ek: np.ndarray, a: float, E: np.ndarray, F: np.ndarray,
                   G: np.ndarray, Fp: np.ndarray, Gp: np.ndarray, n_open: Optional[np.ndarray],
                   batch: int = 0, rowsum: Optional[np.ndarray] = None,
                   status: Optional[np.ndarray] = None):
        """rmx_sweep_host: host arrays in, host rowsum/status out (copies inside the call).
        Arrays should be pinned (see pinned_empty) for asynchronous copies.
        Returns (rowsum, status, h2d_bytes, d2h_bytes)."""
        self._bind_stream()
        nch, ldw = w.shape
        nlev = Ek.shape[0]
        ne = E.shape[0]
        if rowsum is None:
            rowsum = np.empty((ne, nch))
        if status is None:
            status = np.empty(ne, dtype=np.int32)
        h2d, d2h = ctypes.c_int64(), ctypes.c_int64()
        P = lambda x: None if x is None else x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
        self._check(self.lib.rmx_sweep_host(
            self._h, P(w), ldw, P(Ek), nch, nlev, float(a), P(E), ne, P(F), P(G), P(Fp), P(Gp),
            P(n_open), int(batch), P(rowsum), P(status), ctypes.byref(h2d), ctypes.byref(d2h)),
            "rmx_sweep_host")
        return rowsum, status, h2d.value, d2h.value

    # ------------------------------------------------------------------ photoionisation (NEXT-1)
    SIGMA_PREFACTOR = 4.0 * np.pi ** 2 / 137.035999084 / 3.0  # 4 pi^2 alpha / 3 (atomic units)

    def dipole_amplitude(self, w, Ek, d, E, status=None):
        """rmx_dipole_amplitude: g[e][i] = sum_k w_ik d_k/(E_k - E_e). Returns (g [ne,nch], status)."""
        torch = _torch()
        self._bind_stream()
        w, nlev, ldw = self.prepare_w(w)
        Ek, d, E = (self._dev(x, torch.float64) for x in (Ek, d, E))
        nch, ne = w.shape[0], E.shape[0]
        g = torch.empty((ne, nch), dtype=torch.float64, device=w.device)
        status = self._status(status, ne)
        self._check(self.lib.rmx_dipole_amplitude(self._h, _ptr(w), ldw, _ptr(Ek), _ptr(d), nch, nlev,
                                                  _ptr(E), ne, _ptr(g), _ptr(status)),
                    "rmx_dipole_amplitude")
        return g, status

    def photoionization(self, K, g, Fp, Gp, E, E0: float, C: Optional[float] = None, n_open=None,
                        status=None, want_mabs2: bool = True):
        """rmx_photoionization: sigma(E) = C (E - E0) sum_j |M_j|^2, M = (I - iK_oo)^{-1} (1/2) U'^T g.
        Returns (sigma [ne], mabs2 [ne,nch] or None, status)."""
        torch = _torch()
        self._bind_stream()
        K = self._dev(K, torch.float64)
        g, Fp, Gp, E = (self._dev(x, torch.float64) for x in (g, Fp, Gp, E))
        ne, nch = K.shape[0], K.shape[1]
        no = None if n_open is None else self._dev(n_open, torch.int32)
        sigma = torch.empty(ne, dtype=torch.float64, device=K.device)
        m2 = torch.empty((ne, nch), dtype=torch.float64, device=K.device) if want_mabs2 else None
        status = self._status(status, ne)
        C = self.SIGMA_PREFACTOR if C is None else float(C)
        self._check(self.lib.rmx_photoionization(self._h, _ptr(K), _ptr(g), _ptr(Fp), _ptr(Gp), _ptr(E),
                                                 nch, ne, _ptr(no), float(E0), C, _ptr(sigma), _ptr(m2),
                                                 _ptr(status)), "rmx_photoionization")
        return sigma, m2, status

    def sweep_photo(self, w, Ek, d, a: float, E, F, G, Fp, Gp, n_open, E0: float,
                    C: Optional[float] = None, batch: int = 0, status=None, want_mabs2: bool = False):
        """rmx_sweep_photo: fused R -> K -> g -> sigma for all energies. Returns dict(sigma, mabs2, status)."""
        torch = _torch()
        self._bind_stream()
        w, nlev, ldw = self.prepare_w(w)
        Ek, d, E = (self._dev(x, torch.float64) for x in (Ek, d, E))
        F, G, Fp, Gp = (self._dev(x, torch.float64) for x in (F, G, Fp, Gp))
        n_open = None if n_open is None else self._dev(n_open, torch.int32)
        nch, ne = w.shape[0], E.shape[0]
        sigma = torch.empty(ne, dtype=torch.float64, device=w.device)
        m2 = torch.empty((ne, nch), dtype=torch.float64, device=w.device) if want_mabs2 else None
        status = self._status(status, ne)
        C = self.SIGMA_PREFACTOR if C is None else float(C)
        self._check(self.lib.rmx_sweep_photo(
            self._h, _ptr(w), ldw, _ptr(Ek), _ptr(d), nch, nlev, float(a), _ptr(E), ne, _ptr(F), _ptr(G),
            _ptr(Fp), _ptr(Gp), _ptr(n_open), int(batch), float(E0), C, _ptr(sigma), _ptr(m2),
            _ptr(status)), "rmx_sweep_photo")
        return {"sigma": sigma, "mabs2": m2, "status": status}

    # ------------------------------------------------------------------ inner region (NEXT-3)
    def inner_region(self, H, P):
        """rmx_inner_region: (E_k, V) = eigh(H), w = P^T V. Returns (Ek [nlev], w [nch, ldw], nlev,
        ldw) with ldw even (ready for build_R / sweep with prepared=(nlev, ldw))."""
        torch = _torch()
        self._bind_stream()
        H = self._dev(H, torch.float64)
        P = self._dev(P, torch.float64)
        nlev, nch = P.shape
        ldw = nlev + (nlev & 1)
        Ek = torch.empty(nlev, dtype=torch.float64, device=H.device)
        w = torch.zeros((nch, ldw), dtype=torch.float64, device=H.device)
        self._check(self.lib.rmx_inner_region(self._h, _ptr(H), nlev, _ptr(P), nch, _ptr(Ek), _ptr(w),
                                              ldw), "rmx_inner_region")
        return Ek, w, nlev, ldw

    # ------------------------------------------------------------------ post-processing
    def convolve_gaussian(self, x, dE: float, fwhm: float, mix=None):
        """rmx_convolve_gaussian: x [nspec, ne] (or [ne]) on a uniform mesh of spacing dE ->
        Gaussian-convolved spectra ([nspec, ne]) or, with admixture weights mix [nspec], one [ne]."""
        torch = _torch()
        self._bind_stream()
        x = self._dev(x, torch.float64)
        if x.dim() == 1:
            x = x[None, :]
        nspec, ne = x.shape
        mixh = None if mix is None else np.ascontiguousarray(mix, dtype=np.float64)
        y = torch.empty((ne,) if mixh is not None else (nspec, ne), dtype=torch.float64, device=x.device)
        self._check(self.lib.rmx_convolve_gaussian(
            self._h, _ptr(x), nspec, None if mixh is None else mixh.ctypes.data_as(ctypes.c_void_p),
            ne, float(dE), float(fwhm), _ptr(y)), "rmx_convolve_gaussian")
        return y

    def maxwell_average(self, omega, E, Eth, kT):
        """rmx_maxwell_average: omega [ne, npair] -> Upsilon [npair, nT]."""
        torch = _torch()
        self._bind_stream()
        omega = self._dev(omega, torch.float64)
        E = self._dev(E, torch.float64)
        Eth = self._dev(Eth, torch.float64)
        kTh = np.ascontiguousarray(kT, dtype=np.float64)
        ne, npair = omega.shape
        ups = torch.empty((npair, len(kTh)), dtype=torch.float64, device=omega.device)
        self._check(self.lib.rmx_maxwell_average(self._h, _ptr(omega), ne, npair, _ptr(E), _ptr(Eth),
                                                 kTh.ctypes.data_as(ctypes.c_void_p), len(kTh),
                                                 _ptr(ups)), "rmx_maxwell_average")
        return ups

    # ------------------------------------------------------------------ instrumentation
    def set_r_algo(self, algo: int):
        """rmx_set_r_algo: R_DMMA (FP64 tensor cores, default) or R_INT8 (exact CRT on INT8 tensor cores)."""
        self._check(self.lib.rmx_set_r_algo(self._h, int(algo)), "rmx_set_r_algo")

    def set_timing(self, on: bool = True):
        self._check(self.lib.rmx_set_timing(self._h, 1 if on else 0), "rmx_set_timing")

    def reset_stats(self):
        self._check(self.lib.rmx_reset_stats(self._h), "rmx_reset_stats")

    def stats(self):
        ms = (ctypes.c_double * NKID)()
        cnt = (ctypes.c_int64 * NKID)()
        tot = ctypes.c_int64()
        self._check(self.lib.rmx_stats(self._h, ms, cnt, ctypes.byref(tot)), "rmx_stats")
        return {KID_NAMES[k]: (ms[k], cnt[k]) for k in range(NKID)} | {"launches": tot.value}

    def sync(self, status=None):
        n_bad = ctypes.c_int64()
        ne = 0 if status is None else status.numel()
        self._check(self.lib.rmx_sync(self._h, _ptr(status), ne, ctypes.byref(n_bad)), "rmx_sync")
        return n_bad.value


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """A numpy array backed by pinned (page-locked) host memory via torch."""
    torch = _torch()
    tdt = {np.float64: torch.float64, np.int32: torch.int32, np.int64: torch.int64}[np.dtype(dtype).type]
    t = torch.empty(shape, dtype=tdt, pin_memory=True)
    _pinned_keepalive.append(t)  # the numpy view does not own the pinned storage
    return t.numpy()


_pinned_keepalive = []


_default_ctx = {}


def _ctx() -> Context:
    torch = _torch()
    dev = torch.cuda.current_device()
    if dev not in _default_ctx:
        _default_ctx[dev] = Context(dev)
    return _default_ctx[dev]


# module-level functions with the C-ABI names (argument marshalling only)
def rmx_build_R(w, Ek, a, E, status=None):
    return _ctx().build_R(w, Ek, a, E, status=status)


def rmx_match_K(R, F, G, Fp, Gp, a, n_open=None, status=None):
    return _ctx().match_K(R, F, G, Fp, Gp, a, n_open=n_open, status=status)


def rmx_collision_strength(K, n_open=None, status=None):
    return _ctx().collision_strength(K, n_open=n_open, status=status)


def rmx_sweep(w, Ek, a, E, F, G, Fp, Gp, n_open=None, batch=0, dump_idx=None):
    return _ctx().sweep(w, Ek, a, E, F, G, Fp, Gp, n_open=n_open, batch=batch, dump_idx=dump_idx)


def rmx_collision_strength_levels(K, level_start, g=1.0, n_open=None, omega=None, status=None):
    return _ctx().collision_strength_levels(K, level_start, g=g, n_open=n_open, omega=omega,
                                            status=status)


def rmx_dipole_amplitude(w, Ek, d, E, status=None):
    return _ctx().dipole_amplitude(w, Ek, d, E, status=status)


def rmx_photoionization(K, g, Fp, Gp, E, E0, C=None, n_open=None, status=None):
    return _ctx().photoionization(K, g, Fp, Gp, E, E0, C=C, n_open=n_open, status=status)


def rmx_sweep_photo(w, Ek, d, a, E, F, G, Fp, Gp, n_open, E0, C=None, batch=0):
    return _ctx().sweep_photo(w, Ek, d, a, E, F, G, Fp, Gp, n_open, E0, C=C, batch=batch)


def rmx_inner_region(H, P):
    return _ctx().inner_region(H, P)


def rmx_convolve_gaussian(x, dE, fwhm, mix=None):
    return _ctx().convolve_gaussian(x, dE, fwhm, mix=mix)


def rmx_maxwell_average(omega, E, Eth, kT):
    return _ctx().maxwell_average(omega, E, Eth, kT)


def rmx_sweep_levels(w, Ek, a, E, F, G, Fp, Gp, n_open, level_start, g=1.0, omega=None, batch=0):
    return _ctx().sweep_levels(w, Ek, a, E, F, G, Fp, Gp, n_open, level_start, g=g, omega=omega,
                               batch=batch)
