"""NEXT-3 of SURVEY.md §8(f): the inner-region eigensolve feeding the sweep.

CPU (`-m "not gpu"`): oracle.inner_region pinned to the closed-form spectrum of a tridiagonal
Toeplitz matrix (a + 2b cos(k pi/(n+1))), to a matrix built from a known spectrum, and to the
defining identity of its outputs: the pole sum of the returned (E_k, w) equals the direct solve
(1/2a) P^T (H - E)^{-1} P (BASELINE.json:5 north_star brute-force pin).
GPU (`-m gpu`): rmx_inner_region against the oracle - eigenvalues normwise 1e-12; w up to the
per-eigenvector sign (1e-9); and the sign-free R(E) built from the GPU outputs by rmx_build_R against
the oracle's R from its own outputs (1e-10, the R bar), energies midway between neighbouring poles.
"""
import math

import numpy as np
import pytest

import oracle
import rmx_synth as syn


def nrel(x, ref):
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (den if den > 0 else 1.0))


def test_tridiagonal_toeplitz_spectrum():
    n, a, b = 200, 2.0, -0.7
    H = np.diag(np.full(n, a)) + np.diag(np.full(n - 1, b), 1) + np.diag(np.full(n - 1, b), -1)
    Ek, w = oracle.inner_region(H, np.eye(n)[:, :3])
    ref = np.sort(a + 2 * b * np.cos(np.arange(1, n + 1) * math.pi / (n + 1)))
    assert np.max(np.abs(Ek - ref)) < 1e-13
    # w = P^T V with P = first 3 unit vectors: the first 3 components of each eigenvector,
    # |V_jk| = sqrt(2/(n+1)) |sin(j k pi/(n+1))| for the Toeplitz eigenvectors
    k = np.arange(1, n + 1)
    order = np.argsort(a + 2 * b * np.cos(k * math.pi / (n + 1)))
    for j in range(3):
        ref_abs = math.sqrt(2 / (n + 1)) * np.abs(np.sin((j + 1) * k[order] * math.pi / (n + 1)))
        assert np.max(np.abs(np.abs(w[j]) - ref_abs)) < 1e-12


def test_known_spectrum():
    rng = np.random.default_rng(1)
    lam = np.sort(rng.uniform(-3, 30, 120))
    Q, _ = np.linalg.qr(rng.normal(size=(120, 120)))
    Ek, w = oracle.inner_region((Q * lam) @ Q.T, Q)
    assert np.max(np.abs(Ek - lam)) < 1e-12
    assert np.allclose(np.abs(w), np.eye(120), atol=1e-12)  # P = Q: w = Q^T V = +-I


def test_pole_sum_equals_direct_solve():
    c = syn.brute_force_case(6, 150, seed=21, ne=5)
    Ek, w = oracle.inner_region(c.H, c.P)
    for E in c.E:
        R, st = oracle.R(w, Ek, c.a, E)
        ref = c.P.T @ np.linalg.solve(c.H - E * np.eye(c.nlev), c.P) / (2 * c.a)
        assert st == 0 and nrel(R, ref) < 1e-11


@pytest.fixture(scope="module")
def ctx():
    import paper_1403_5524_b200 as rmx
    return rmx.Context()


@pytest.mark.gpu
@pytest.mark.parametrize("nch,nlev", [(8, 200), (64, 1500), (130, 3000)])
def test_gpu_inner_region(ctx, nch, nlev):
    import torch
    c = syn.brute_force_case(nch, nlev, seed=nlev, ne=12, lo=0.5, hi=9.5)
    Ek_g, w_g, _, ldw = ctx.inner_region(c.H, c.P)
    torch.cuda.synchronize()
    Ek_o, w_o = oracle.inner_region(c.H, c.P)
    Ek_h, w_h = Ek_g.cpu().numpy(), w_g.cpu().numpy()[:, :nlev]
    assert nrel(Ek_h, Ek_o) < 1e-12
    # eigenvector signs are the solver's: align each GPU column to the oracle's (largest |entry|)
    piv = np.argmax(np.abs(w_o), axis=0)
    sgn = np.sign(w_o[piv, np.arange(nlev)] * w_h[piv, np.arange(nlev)])
    assert nrel(w_h * sgn[None, :], w_o) < 1e-9
    # the sign-free product the sweep consumes: R(E) from GPU outputs vs oracle R from oracle outputs,
    # at energies midway between neighbouring poles (eigenvalue rounding moves a pole term by
    # ~ delta_lambda / (E_k - E) relative)
    j = np.linspace(0, nlev - 2, 8).round().astype(int)
    E = 0.5 * (Ek_o[j] + Ek_o[j + 1])
    R_g, st = ctx.build_R(w_g[:, :nlev], Ek_g, c.a, E)
    torch.cuda.synchronize()
    R_g = R_g.cpu().numpy()
    for e, x in enumerate(E):
        R_o, _ = oracle.R(w_o, Ek_o, c.a, x)
        assert nrel(R_g[e], R_o) < 1e-10, (x, nrel(R_g[e], R_o))
