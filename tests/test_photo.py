"""NEXT-1 of SURVEY.md §8(f): the photoionisation variant of the sweep (PAPER.md:116-122, 148-156:
the bound-free dipole outer region PSTGBF0DAMP of Tables 1-2; readings P1-P4):

    g_i(E)  = sum_k w_ik d_k / (E_k - E)                       dipole amplitude contraction
    v_j     = (1/2) (g_j F'_j + sum_i g_i G'_i K_ij)            (1/2) U'^T g, U = F + G K, j open
    M       = (I - i K_oo)^{-1} v                               ingoing-wave final states
    sigma   = C (E - E0) sum_j |M_j|^2,  C = 4 pi^2 alpha / 3   (atomic units)

CPU (`-m "not gpu"`): the oracle pinned to a direct solve g = P^T (H - E)^{-1} delta (with
d = V^T delta), the single-channel closed form |M|^2 = v^2/(1 + K^2), an independent spectral route
for M (K_oo = Q L Q^T), invariance of |M|^2 under the arbitrary closed-channel normalisation, and
the scalings of sigma. GPU (`-m gpu`): rmx_dipole_amplitude, rmx_photoionization and the fused
rmx_sweep_photo against the oracle - g normwise 1e-10 (the R bar: same pole sum), |M|^2 and sigma
1e-8 (the |T|^2 bar), energies >= 1e-6 from poles and thresholds.
"""
import math

import numpy as np
import pytest

import oracle
import rmx_synth as syn

TOL_G, TOL_M = 1e-10, 1e-8


def nrel(x, ref):
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (den if den > 0 else 1.0))


def _case_with_dipole(nch, nlev, seed, **kw):
    c = syn.brute_force_case(nch, nlev, seed, **kw)
    Ek, V = np.linalg.eigh(c.H)
    delta = np.random.default_rng(seed + 1).normal(0.0, 1.0, nlev)
    return c, Ek, np.ascontiguousarray(c.P.T @ V), V.T @ delta, delta


# ----------------------------------------------------------------------------- oracle pins
def test_g_equals_direct_solve():
    c, Ek, w, d, delta = _case_with_dipole(5, 160, seed=31, ne=6)
    for E in c.E:
        g, st = oracle.dipole_g(w, Ek, d, E)
        ref = c.P.T @ np.linalg.solve(c.H - E * np.eye(c.nlev), delta)
        assert st == 0 and nrel(g, ref) < 1e-11


def test_single_channel_closed_form():
    rng = np.random.default_rng(2)
    for _ in range(5):
        K = np.array([[rng.normal()]])
        g, Fp, Gp = rng.normal(size=1), rng.normal(size=1), rng.normal(size=1)
        M, m2, st = oracle.photo(K, 1, g, Fp, Gp)
        v = 0.5 * (g[0] * Fp[0] + g[0] * Gp[0] * K[0, 0])
        assert math.isclose(m2[0], v * v / (1 + K[0, 0] ** 2), rel_tol=1e-14)
        assert abs(M[0] - v / (1 - 1j * K[0, 0])) < 1e-14 * abs(v)


def _k_for(c, E):
    F, G, Fp, Gp = syn.asymptotic(c.eps, np.array([E]), c.a)
    R, _ = oracle.R(c.w, c.Ek, c.a, E)
    K, _, _ = oracle.K(R, F[0], G[0], Fp[0], Gp[0], c.a)
    return K, F[0], G[0], Fp[0], Gp[0], int(syn.n_open(c.eps, np.array([E]))[0]), R


def test_spectral_and_spd_routes_agree():
    c, Ek, w, d, _ = _case_with_dipole(7, 200, seed=5, ne=5, lo=0.5, hi=9.0, eps_hi=3.0)
    for E in c.E:
        K, F, G, Fp, Gp, no, _ = _k_for(c, E)
        g, _ = oracle.dipole_g(w, Ek, d, E)
        M, m2, st = oracle.photo(K, no, g, Fp, Gp)
        v = 0.5 * (g[:no] * Fp[:no] + (g * Gp) @ K[:, :no])
        lam, Q = np.linalg.eigh(0.5 * (K[:no, :no] + K[:no, :no].T))
        M_spec = Q @ ((Q.T @ v) / (1 - 1j * lam))
        y = np.linalg.solve(np.eye(no) + K[:no, :no] @ K[:no, :no], v)
        M_spd = y + 1j * (K[:no, :no] @ y)
        assert nrel(M, M_spec) < 1e-11 and nrel(M, M_spd) < 1e-11
        assert np.all(m2[no:] == 0)


def test_closed_channel_normalisation_invariance():
    c, Ek, w, d, _ = _case_with_dipole(6, 180, seed=9, ne=4, lo=0.5, hi=4.0, eps_hi=3.0)
    for E in c.E:
        F, G, Fp, Gp = syn.asymptotic(c.eps, np.array([E]), c.a)
        no = int(syn.n_open(c.eps, np.array([E]))[0])
        if no == c.nch:
            continue
        R, _ = oracle.R(c.w, c.Ek, c.a, E)
        g, _ = oracle.dipole_g(w, Ek, d, E)
        out = []
        for scale in (1.0, 37.0):
            s = np.where(np.arange(c.nch) < no, 1.0, scale)
            K, _, _ = oracle.K(R, F[0] * s, G[0] * s, Fp[0] * s, Gp[0] * s, c.a)
            out.append(oracle.photo(K, no, g, Fp[0] * s, Gp[0] * s)[1])
        assert nrel(out[1], out[0]) < 1e-11


def test_sigma_scalings():
    c, Ek, w, d, _ = _case_with_dipole(4, 120, seed=12, ne=3, lo=1.0, hi=6.0, eps_hi=2.0)
    F, G, Fp, Gp = syn.asymptotic(c.eps, c.E, c.a)
    no = syn.n_open(c.eps, c.E)
    a1 = oracle.photo_sweep(w, Ek, d, c.a, c.E, F, G, Fp, Gp, no, E0=-1.5)
    a2 = oracle.photo_sweep(w, Ek, 3.0 * d, c.a, c.E, F, G, Fp, Gp, no, E0=-1.5, C=2.0)
    assert np.allclose(a2["sigma"], 9.0 * 2.0 / oracle.SIGMA_PREFACTOR * a1["sigma"], rtol=1e-12)
    assert np.all(a1["sigma"] > 0) and np.all(a1["status"] == 0)


# ----------------------------------------------------------------------------- GPU parity
@pytest.fixture(scope="module")
def ctx():
    import paper_1403_5524_b200 as rmx
    return rmx.Context()


def _excluded(c, E):
    return np.min(np.abs(E - c.Ek)) < 1e-6 or np.min(np.abs(E - c.eps)) < 1e-6


@pytest.mark.gpu
@pytest.mark.parametrize("nch,nlev,eps_hi", [(8, 200, 3.0), (70, 1000, 4.0), (150, 517, 4.0), (260, 900, 0.0)])
def test_gpu_photo(ctx, nch, nlev, eps_hi):
    import torch
    c, Ek, w, d, _ = _case_with_dipole(nch, nlev, seed=nch, ne=9, lo=0.5, hi=9.0, a=12.0,
                                       eps_hi=eps_hi)
    F, G, Fp, Gp = syn.asymptotic(c.eps, c.E, c.a)
    no = syn.n_open(c.eps, c.E)
    E0 = -2.0
    ref = oracle.photo_sweep(w, Ek, d, c.a, c.E, F, G, Fp, Gp, no, E0=E0)
    # three calls: g, K, then the amplitudes
    g, st = ctx.dipole_amplitude(w, Ek, d, c.E)
    R, st = ctx.build_R(w, Ek, c.a, c.E, status=st)
    K, st = ctx.match_K(R, F, G, Fp, Gp, c.a, no, status=st)
    sig, m2, st = ctx.photoionization(K, g, Fp, Gp, c.E, E0, n_open=no, status=st)
    fused = ctx.sweep_photo(w, Ek, d, c.a, c.E, F, G, Fp, Gp, no, E0, batch=4, want_mabs2=True)
    torch.cuda.synchronize()
    g, sig, m2 = g.cpu().numpy(), sig.cpu().numpy(), m2.cpu().numpy()
    assert int((st != 0).sum()) == 0 and int((fused["status"] != 0).sum()) == 0
    for e in range(c.ne):
        if _excluded(c, c.E[e]):
            continue
        assert nrel(g[e], ref["g"][e]) < TOL_G, e
        assert nrel(m2[e], ref["mabs2"][e]) < TOL_M, (e, nrel(m2[e], ref["mabs2"][e]))
        assert nrel(fused["mabs2"][e].cpu().numpy(), ref["mabs2"][e]) < TOL_M, e
    assert nrel(sig, ref["sigma"]) < TOL_M
    assert nrel(fused["sigma"].cpu().numpy(), ref["sigma"]) < TOL_M


@pytest.mark.gpu
def test_gpu_photo_near_poles(ctx):
    """NEXT-1 at energies 1e-5 and 1e-3 from poles (the nearest pole's term of g is summed apart and
    added last, reading N1, as in R formation): g, |M_j|^2 and sigma against the oracle."""
    import torch
    c, Ek, w, d, _ = _case_with_dipole(150, 517, seed=77, ne=4, lo=0.5, hi=9.0, a=12.0, eps_hi=4.0)
    inside = Ek[(Ek > 1.0) & (Ek < 8.5)]
    E = np.sort(np.concatenate([p + np.array([-1e-5, 1e-5, 1e-3]) for p in inside[[5, len(inside) // 2]]]))
    F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
    no = syn.n_open(c.eps, E)
    ref = oracle.photo_sweep(w, Ek, d, c.a, E, F, G, Fp, Gp, no, E0=-2.0)
    g, st = ctx.dipole_amplitude(w, Ek, d, E)
    fused = ctx.sweep_photo(w, Ek, d, c.a, E, F, G, Fp, Gp, no, -2.0, want_mabs2=True)
    torch.cuda.synchronize()
    g = g.cpu().numpy()
    assert int((st != 0).sum()) == 0 and int((fused["status"] != 0).sum()) == 0
    for e in range(len(E)):
        assert nrel(g[e], ref["g"][e]) < 1e-12, (E[e], nrel(g[e], ref["g"][e]))
        assert nrel(fused["mabs2"][e].cpu().numpy(), ref["mabs2"][e]) < TOL_M, e
    assert nrel(fused["sigma"].cpu().numpy(), ref["sigma"]) < TOL_M
