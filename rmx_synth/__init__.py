"""Seeded synthetic inputs for the outer-region energy sweep R(E) -> K(E) -> |T(E)|^2.

This module is shared by BOTH sides of the parity check (the CPU oracle under
``oracle/`` and the CUDA path under ``paper_1403_5524_b200/``) and therefore holds
NONE of the method's arithmetic: no R-matrix pole sum, no matching solve, no T.
It only draws the inputs the paper treats as given by the inner region
(poles E_k and boundary amplitudes w_ik, §6 Eq. 1-2), the energy
mesh (§3), the channel thresholds, and evaluates the
analytic asymptotic functions F, G, F', G' that BASELINE.json:7-11 prescribe as
inputs to ``rmx_match_K(R, F, G, F', G')``.

Readings of BASELINE.json / SURVEY.md §8(c) applied here (all listed in DESIGN.md §3):
  * item 4  : open-channel normalisation F = k^-1/2 sin(th), G = k^-1/2 cos(th),
              F' = k^1/2 cos(th), G' = -k^1/2 sin(th), th = k a + 0.3 i  (Wronskian -1)
  * item 5-7: F', G' are d/dr at r = a; channel index i is 0-based after sorting by
              threshold; k = sqrt(2(E - eps_i)) taken literally.
  * item 8  : channel i is open iff E > eps_i (strict).
  * item 9  : closed channels F = G = exp(-kappa a), F' = G' = -kappa exp(-kappa a),
              kappa = sqrt(2(eps_i - E)).
  * item 12 : the tiny mesh drops points within 1e-6 Ry of any pole.
  * item 14 : mesh E_i = lo + i (hi - lo)/(ne - 1); fine: E_i = 3.0 + i 5e-7.
  * item 15-19: numpy default_rng(seed) (PCG64), draw order exactly as coded below.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

__all__ = [
    "Case", "CONFIGS", "make_case", "asymptotic", "n_open", "mesh", "brute_force_case",
    "parity_sample", "level_start", "symmetry_cases",
]


@dataclasses.dataclass
class Case:
    """One synthetic sweep problem. Arrays are float64, C-contiguous.

    w      : [nch, nlev]  boundary amplitudes w_ik (k contiguous)
    Ek     : [nlev]       poles, ascending
    eps    : [nch]        channel thresholds, ascending (open set is a prefix)
    E      : [ne]         energy mesh
    a      : boundary radius
    H, P   : optional inner-region Hamiltonian / channel projections that generated
             (Ek, w) via w = P^T V, (Ek, V) = eigh(H) (configs 'small' and brute_force_case)
    """
    name: str
    w: np.ndarray
    Ek: np.ndarray
    eps: np.ndarray
    E: np.ndarray
    a: float
    H: Optional[np.ndarray] = None
    P: Optional[np.ndarray] = None
    dropped_mesh_points: int = 0

    @property
    def nch(self) -> int:
        return int(self.w.shape[0])

    @property
    def nlev(self) -> int:
        return int(self.w.shape[1])

    @property
    def ne(self) -> int:
        return int(self.E.shape[0])


# BASELINE.json:7-11, as (nch, nlev, ne, lo, hi, a)
CONFIGS = {
    "tiny": dict(nch=8, nlev=200, ne=1000, lo=0.05, hi=9.95, a=20.0),
    "small": dict(nch=64, nlev=3000, ne=20000, lo=0.1, hi=5.0, a=25.0),
    "bp": dict(nch=500, nlev=15000, ne=50000, lo=0.2, hi=20.0, a=18.0),
    "darc": dict(nch=2000, nlev=40000, ne=100000, lo=0.5, hi=60.0, a=12.0),
    "fine": dict(nch=1200, nlev=30000, ne=400000, lo=3.0, hi=3.2, a=15.0),
}


def mesh(lo: float, hi: float, ne: int) -> np.ndarray:
    """Uniform inclusive mesh, point i = lo + i*(hi-lo)/(ne-1)."""
    if ne == 1:
        return np.array([lo], dtype=np.float64)
    step = (hi - lo) / (ne - 1)
    return lo + np.arange(ne, dtype=np.float64) * step


def _drop_near_poles(E: np.ndarray, Ek: np.ndarray, guard: float = 1e-6):
    idx = np.searchsorted(Ek, E)
    lo = np.abs(E - Ek[np.clip(idx - 1, 0, len(Ek) - 1)])
    hi = np.abs(E - Ek[np.clip(idx, 0, len(Ek) - 1)])
    keep = np.minimum(lo, hi) >= guard
    return E[keep], int((~keep).sum())


def make_case(name: str, seed: int = 0, ne: Optional[int] = None) -> Case:
    """Generate one of the BASELINE.json configs (seed 0 by default).

    ``ne`` overrides the mesh length (the mesh keeps its end points) for reduced
    parity runs; the poles, amplitudes and thresholds are identical to the full config.
    """
    cfg = CONFIGS[name]
    nch, nlev, a = cfg["nch"], cfg["nlev"], cfg["a"]
    ne_full = cfg["ne"]
    rng = np.random.default_rng(seed)
    H = P = None
    dropped = 0
    if name == "tiny":
        # BASELINE.json:7 - E_k sorted uniform [0,10]; w ~ N(0, 0.1^2); eps_i = 0.01 i
        Ek = np.sort(rng.uniform(0.0, 10.0, nlev))
        w = rng.normal(0.0, 0.1, (nch, nlev))
        eps = 0.01 * np.arange(nch, dtype=np.float64)
        E = mesh(cfg["lo"], cfg["hi"], ne or ne_full)
        E, dropped = _drop_near_poles(E, Ek)
    elif name == "small":
        # BASELINE.json:8, SURVEY §8(c) 16
        H = np.zeros((nlev, nlev))
        iu = np.triu_indices(nlev, 1)
        diag = rng.uniform(0.0, 50.0, nlev)
        off = rng.normal(0.0, 0.05, len(iu[0]))
        H[iu] = off
        H = H + H.T
        H[np.diag_indices(nlev)] = diag
        Ek, V = np.linalg.eigh(H)
        P = rng.normal(0.0, 1.0, (nlev, nch))
        w = np.ascontiguousarray(P.T @ V)
        eps = np.sort(rng.uniform(0.0, 0.5, nch))
        E = mesh(cfg["lo"], cfg["hi"], ne or ne_full)
    elif name == "bp":
        # BASELINE.json:9, SURVEY §8(c) 17
        Ek = np.sort(rng.uniform(-2.0, 200.0, nlev))
        w = rng.normal(0.0, 0.05, (nch, nlev))
        rows = rng.choice(nch, int(round(0.05 * nch)), replace=False)
        w[rows] *= 10.0
        eps = np.sort(rng.uniform(0.0, 15.0, nch))
        E = mesh(cfg["lo"], cfg["hi"], ne or ne_full)
    elif name == "darc":
        # BASELINE.json:10, SURVEY §8(c) 18 - Wigner semicircle on [-5, 400]
        u1 = rng.uniform(0.0, 1.0, nlev)
        u2 = rng.uniform(0.0, 1.0, nlev)
        t = np.sqrt(u1) * np.cos(2.0 * np.pi * u2)
        Ek = np.sort(197.5 + 202.5 * t)
        w = rng.normal(0.0, 0.02, (nch, nlev))
        lev = rng.uniform(0.0, 50.0, 300)
        eps = np.sort(np.concatenate([np.repeat(lev[:200], 7), np.repeat(lev[200:], 6)]))
        E = mesh(cfg["lo"], cfg["hi"], ne or ne_full)
    elif name == "fine":
        # BASELINE.json:11, SURVEY §8(c) 19
        n_res = 200
        Ek_res = rng.uniform(3.0, 3.2, n_res)
        w_res = rng.normal(0.0, 1e-3, (nch, n_res))
        Ek_bg = rng.uniform(-3.0, 300.0, nlev - n_res)
        w_bg = rng.normal(0.0, 0.05, (nch, nlev - n_res))
        Ek_all = np.concatenate([Ek_res, Ek_bg])
        w_all = np.concatenate([w_res, w_bg], axis=1)
        order = np.argsort(Ek_all, kind="stable")
        Ek = Ek_all[order]
        w = np.ascontiguousarray(w_all[:, order])
        eps = np.sort(rng.uniform(0.0, 3.5, nch))
        n = ne or ne_full
        if ne is None:
            E = 3.0 + np.arange(n, dtype=np.float64) * 5e-7
        else:  # reduced mesh spanning the same window
            E = mesh(3.0, 3.0 + (ne_full - 1) * 5e-7, n)
    else:
        raise KeyError(name)
    return Case(name=name, w=np.ascontiguousarray(w, dtype=np.float64),
                Ek=np.ascontiguousarray(Ek, dtype=np.float64),
                eps=np.ascontiguousarray(eps, dtype=np.float64),
                E=np.ascontiguousarray(E, dtype=np.float64), a=float(a), H=H, P=P,
                dropped_mesh_points=dropped)


def brute_force_case(nch: int, nlev: int, seed: int, ne: int = 16, lo: float = -1.0,
                     hi: float = 12.0, a: float = 10.0, eps_hi: float = 0.0,
                     offdiag: float = 0.5) -> Case:
    """A small case generated from a seeded symmetric inner-region Hamiltonian H:
    (E_k, V) = eigh(H), w = P^T V with P ~ N(0,1)^{nlev x nch}. Then
    (1/2a) sum_k w_ik w_jk/(E_k - E) = (1/2a) [P^T (H - E)^-1 P]_ij exactly, which
    is the brute-force pin of the pole sum (BASELINE.json:5 north_star)."""
    rng = np.random.default_rng(seed)
    H = np.diag(rng.uniform(0.0, 10.0, nlev))
    iu = np.triu_indices(nlev, 1)
    H[iu] = rng.normal(0.0, offdiag, len(iu[0]))
    H = np.triu(H) + np.triu(H, 1).T
    Ek, V = np.linalg.eigh(H)
    P = rng.normal(0.0, 1.0, (nlev, nch))
    w = np.ascontiguousarray(P.T @ V)
    eps = np.sort(rng.uniform(0.0, eps_hi, nch)) if eps_hi > 0 else np.zeros(nch)
    E = mesh(lo, hi, ne)
    E, dropped = _drop_near_poles(E, Ek, 1e-3)
    return Case(name=f"bf{nch}x{nlev}s{seed}", w=w, Ek=Ek, eps=eps, E=E, a=a, H=H, P=P,
                dropped_mesh_points=dropped)


def n_open(eps: np.ndarray, E: np.ndarray) -> np.ndarray:
    """n_o(E) = #{i : eps_i < E} (strict); eps ascending. int32 [ne]."""
    return np.searchsorted(eps, np.asarray(E, dtype=np.float64), side="left").astype(np.int32)


def asymptotic(eps: np.ndarray, E: np.ndarray, a: float):
    """Asymptotic functions at r = a for every (energy, channel): returns F, G, Fp, Gp,
    each float64 [len(E), nch] (C-contiguous), per BASELINE.json:7,9 and SURVEY §8(c) 4-9.
    Channel index i is 0-based (phase 0.3 i)."""
    E = np.asarray(E, dtype=np.float64)[:, None]
    eps = np.asarray(eps, dtype=np.float64)[None, :]
    nch = eps.shape[1]
    i = np.arange(nch, dtype=np.float64)[None, :]
    is_open = E > eps
    diff = E - eps
    k = np.sqrt(np.where(is_open, 2.0 * diff, 1.0))
    th = k * a + 0.3 * i
    s, c = np.sin(th), np.cos(th)
    rk = np.sqrt(k)
    kappa = np.sqrt(np.where(is_open, 0.0, -2.0 * diff))
    ex = np.exp(-kappa * a)
    F = np.where(is_open, s / rk, ex)
    G = np.where(is_open, c / rk, ex)
    Fp = np.where(is_open, rk * c, -kappa * ex)
    Gp = np.where(is_open, -rk * s, -kappa * ex)
    return (np.ascontiguousarray(F), np.ascontiguousarray(G),
            np.ascontiguousarray(Fp), np.ascontiguousarray(Gp))


def parity_sample(case: Case, n_even: int, n_pole: int = 4, n_thresh: int = 4) -> np.ndarray:
    """Deterministic parity sample of mesh indices (SURVEY §8(d) oracle timing):
    evenly spaced indices, the mesh points nearest 4 isolated poles inside the mesh,
    and the mesh points just above 4 thresholds. Sorted unique int64."""
    ne = case.ne
    idx = set(np.linspace(0, ne - 1, n_even).round().astype(np.int64).tolist())
    E = case.E
    inside = case.Ek[(case.Ek > E[0]) & (case.Ek < E[-1])]
    if len(inside) and n_pole:
        for p in inside[np.linspace(0, len(inside) - 1, n_pole).round().astype(int)]:
            j = int(np.searchsorted(E, p))
            for jj in (j - 1, j):
                if 0 <= jj < ne:
                    idx.add(jj)
    th = case.eps[(case.eps > E[0]) & (case.eps < E[-1])]
    if len(th) and n_thresh:
        for t in th[np.linspace(0, len(th) - 1, n_thresh).round().astype(int)]:
            j = int(np.searchsorted(E, t, side="right"))
            if 0 <= j < ne:
                idx.add(j)
    return np.array(sorted(idx), dtype=np.int64)


def level_start(eps: np.ndarray) -> np.ndarray:
    """Level partition of the (threshold-sorted) channels: channels sharing one threshold belong to
    one target level (BASELINE.json:10 'each level spawning ~6-7 channels'). Returns int32
    [nlevel + 1] with level a = channels [ls[a], ls[a+1]). Pure input structure, no arithmetic of
    the method."""
    eps = np.asarray(eps, dtype=np.float64)
    cut = np.flatnonzero(np.diff(eps) != 0.0) + 1
    return np.concatenate([[0], cut, [len(eps)]]).astype(np.int32)


def symmetry_cases(nsym: int, nlevel: int, seed: int, nlev: int = 300, ne: int = 8,
                   lo: float = 0.5, hi: float = 6.0, a: float = 12.0, lev_hi: float = 4.0,
                   max_ch: int = 3):
    """Several symmetries (partial waves) over ONE set of target levels, for the level-pair
    collision strengths of SURVEY.md §8(f) item 2: the level energies
    (thresholds) ~ U[0, lev_hi] are shared; symmetry s couples level a through c_sa ~ U{1..max_ch}
    channels, has its own poles E_k ~ U[-1, 40] (sorted) and amplitudes w ~ N(0, 0.3^2). All
    symmetries share the energy mesh. Returns (levels [nlevel], E [ne], [(Case, level_start), ...])."""
    rng = np.random.default_rng(seed)
    lev = np.sort(rng.uniform(0.0, lev_hi, nlevel))
    E = mesh(lo, hi, ne)
    out = []
    for s in range(nsym):
        cnt = rng.integers(1, max_ch + 1, nlevel)
        eps = np.repeat(lev, cnt)
        nch = len(eps)
        Ek = np.sort(rng.uniform(-1.0, 40.0, nlev))
        w = rng.normal(0.0, 0.3, (nch, nlev))
        Es, _ = _drop_near_poles(E, Ek, 1e-6)
        assert len(Es) == len(E), "mesh point within 1e-6 of a pole: pick another seed"
        case = Case(name=f"sym{s}", w=np.ascontiguousarray(w), Ek=Ek, eps=eps, E=E.copy(), a=a)
        ls = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int32)
        out.append((case, ls))
    return lev, E, out


def isolated_poles(case: Case, n: int, lo: float, hi: float, min_gap: float) -> np.ndarray:
    """Up to n poles E_k inside [lo, hi] whose nearest neighbouring pole is >= min_gap away, spread
    evenly over the candidates (input structure only)."""
    Ek = case.Ek
    gaps = np.minimum(np.diff(Ek, prepend=-np.inf), np.diff(Ek, append=np.inf))
    cand = Ek[(Ek > lo) & (Ek < hi) & (gaps >= min_gap)]
    if len(cand) == 0:
        return cand
    return cand[np.unique(np.linspace(0, len(cand) - 1, min(n, len(cand))).round().astype(int))]


def survey_sample(case: Case):
    """The darc / fine parity samples of SURVEY.md §8(d) (the energies the oracle is timed and compared
    on), as energies with labels. darc (16): 4 isolated poles at offsets -1e-3, -1e-5, +1e-5; the
    three mesh points next to a pole of K found in round 1 (mesh 50106, 50169, 50228: ||K_oo|| up to
    3e5); one energy 1e-4 above a threshold. fine (32): 4 window resonances (narrow poles,
    |w| ~ 1e-3) at offsets +1.5e-6, -1e-5, +1e-4; 2 background poles inside the window at -1e-5, +1e-5;
    4 energies 1e-4 above a threshold; 12 evenly spaced mesh points. Returns (E [n], labels [n])."""
    E, lab = [], []
    if case.name == "darc":
        lo, hi = case.E[0], case.E[-1]
        for p in isolated_poles(case, 4, lo + 1.0, hi - 1.0, 3e-3):
            for off in (-1e-3, -1e-5, 1e-5):
                E.append(p + off)
                lab.append(f"pole {p:.6f} {off:+.0e}")
        for m in (50106, 50169, 50228):
            E.append(case.E[m])
            lab.append(f"mesh {m} (K pole)")
        th = np.unique(case.eps[(case.eps > lo) & (case.eps < hi)])
        t = th[len(th) // 2]
        E.append(t + 1e-4)
        lab.append(f"threshold {t:.6f} +1e-4")
    elif case.name == "fine":
        lo, hi = case.E[0], case.E[-1]
        win = isolated_poles(case, 10 ** 6, lo + 1e-3, hi - 1e-3, 2e-4)
        # resonance poles: the narrow ones (column norm ~ 1e-3 sqrt(nch)); background poles: wide
        cn = {float(p): float(np.linalg.norm(case.w[:, int(np.searchsorted(case.Ek, p))])) for p in win}
        res = np.array([p for p in win if cn[float(p)] < 0.2])
        bg = np.array([p for p in win if cn[float(p)] >= 0.2])
        for p in res[np.linspace(0, len(res) - 1, 4).round().astype(int)]:
            for off in (1.5e-6, -1e-5, 1e-4):
                E.append(p + off)
                lab.append(f"resonance {p:.7f} {off:+.1e}")
        for p in bg[np.linspace(0, len(bg) - 1, 2).round().astype(int)]:
            for off in (-1e-5, 1e-5):
                E.append(p + off)
                lab.append(f"background pole {p:.7f} {off:+.0e}")
        th = np.unique(case.eps[(case.eps > lo) & (case.eps < hi - 1e-3)])
        for t in th[np.linspace(0, len(th) - 1, 4).round().astype(int)]:
            E.append(t + 1e-4)
            lab.append(f"threshold {t:.7f} +1e-4")
        for m in np.linspace(0, case.ne - 1, 12).round().astype(int):
            E.append(case.E[m])
            lab.append(f"mesh {m}")
    else:
        raise KeyError(case.name)
    return np.array(E, dtype=np.float64), lab
