"""NEXT-4 of SURVEY.md §8(f): post-processing on the energy mesh - Gaussian convolution at a given
FWHM with statistical admixture (PAPER.md:298-300, 370-373 captions; DESIGN.md
reading C1) and the Maxwellian average (effective collision strength; reading U1).

CPU (`-m "not gpu"`): the oracle functions pinned to closed forms - a constant stays constant, an
interior delta becomes normalised Gaussian samples, a linear ramp is preserved in the interior (the
kernel is symmetric), SPEC.md:310's 2/3 + 1/3 admixture example, and the trapezoid sum of e^{-x}
(constant Omega) and of x e^{-x} (Omega linear in eps) in closed geometric-series form.
GPU (`-m gpu`): rmx_convolve_gaussian / rmx_maxwell_average against the oracle on seeded spectra,
normwise 1e-12 (fixed short sums; exp differs by an ulp between libm and CUDA).
"""
import math

import numpy as np
import pytest

import oracle

TOL = 1e-12


def nrel(x, ref):
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (den if den > 0 else 1.0))


# ----------------------------------------------------------------------------- convolution pins
def test_constant_stays_constant():
    y = oracle.convolve_gaussian(np.full(300, 2.5), dE=0.01, fwhm=0.2)
    assert np.allclose(y, 2.5, rtol=1e-15, atol=0)


def test_interior_delta_is_gaussian_samples():
    dE, fwhm, ne, c = 0.01, 0.1, 201, 100
    x = np.zeros(ne)
    x[c] = 1.0
    y = oracle.convolve_gaussian(x, dE, fwhm)[0]
    s = fwhm / (2 * math.sqrt(2 * math.log(2)))
    M = int(math.floor(5 * s / dE))
    d = np.arange(-M, M + 1)
    g = np.exp(-(d * dE) ** 2 / (2 * s * s))
    ref = np.zeros(ne)
    ref[c - M:c + M + 1] = g / g.sum()  # interior outputs all see the full window
    assert nrel(y, ref) < 1e-15
    assert math.isclose(y.max(), dE / (s * math.sqrt(2 * math.pi)), rel_tol=1e-3)


def test_linear_ramp_preserved_in_interior():
    dE, fwhm = 0.002, 0.03
    E = np.arange(500) * dE
    y = oracle.convolve_gaussian(3.0 * E - 1.0, dE, fwhm)[0]
    s = fwhm / (2 * math.sqrt(2 * math.log(2)))
    M = int(math.floor(5 * s / dE))
    assert np.allclose(y[M:-M], (3.0 * E - 1.0)[M:-M], rtol=0, atol=1e-13)
    assert not np.allclose(y[:M], (3.0 * E - 1.0)[:M], rtol=0, atol=1e-6)  # edges renormalised


def test_admixture_two_thirds_one_third():
    # SPEC.md:310 example ("2/3 ground and 1/3 metastable"): 3s and 0s, 2:1 -> 2.0
    x = np.stack([np.full(50, 3.0), np.zeros(50)])
    y = oracle.convolve_gaussian(x, dE=0.01, fwhm=0.05, mix=[2.0, 1.0])
    assert np.allclose(y, 2.0, rtol=1e-15, atol=0)


# ----------------------------------------------------------------------------- Maxwellian pins
def _trap_closed_form(h, x0, n, kind):
    """Trapezoid rule on x_i = x0 + i h, i = 0..n-1 of e^{-x} (kind 0) or x e^{-x} (kind 1), in
    closed form: geometric sums sum r^i, sum i r^i with r = e^{-h}."""
    r = math.exp(-h)
    m = n - 1
    S0 = (1 - r ** (m + 1)) / (1 - r)                                 # sum_{i=0}^{m} r^i
    S1 = r * (1 - (m + 1) * r ** m + m * r ** (m + 1)) / (1 - r) ** 2   # sum i r^i
    ends0 = 0.5 * (1 + r ** m)
    if kind == 0:
        return h * math.exp(-x0) * (S0 - ends0)
    ends1 = 0.5 * (x0 + (x0 + m * h) * r ** m)
    return h * math.exp(-x0) * (x0 * S0 + h * S1 - ends1)


def test_maxwell_constant_and_linear_closed_forms():
    E = 0.3 + np.arange(4000) * 0.005
    Eth = np.array([0.31234, 1.0])
    kT = [0.05, 0.4, 2.0]
    om = np.empty((len(E), 2))
    om[:, 0] = 1.7                                # constant Omega
    om[:, 1] = 0.8 * np.maximum(E - Eth[1], 0.0)  # Omega = 0.8 eps
    ups = oracle.maxwell_average(om, E, Eth, kT)
    for t, kt in enumerate(kT):
        f0 = int(np.searchsorted(E, Eth[0], side="right"))
        n = len(E) - f0
        ref0 = 1.7 * _trap_closed_form(0.005 / kt, (E[f0] - Eth[0]) / kt, n, 0)
        assert math.isclose(ups[0, t], ref0, rel_tol=1e-12)
        f1 = int(np.searchsorted(E, Eth[1], side="right"))
        n = len(E) - f1
        ref1 = 0.8 * kt * _trap_closed_form(0.005 / kt, (E[f1] - Eth[1]) / kt, n, 1)
        assert math.isclose(ups[1, t], ref1, rel_tol=1e-10)
    # and the integral itself: int_0^inf e^{-x} dx = 1, int x e^{-x} = 1 (trapezoid error O(h^2))
    assert math.isclose(ups[0, 1], 1.7 * math.exp(-(E[3] - Eth[0]) / 0.4), rel_tol=2e-4)


# ----------------------------------------------------------------------------- GPU parity
@pytest.fixture(scope="module")
def ctx():
    import paper_1403_5524_b200 as rmx
    return rmx.Context()


@pytest.mark.gpu
@pytest.mark.parametrize("ne,dE,fwhm", [(1000, 0.01, 0.06), (20011, 5e-7, 2.9e-4), (777, 0.01, 0.021)])
def test_gpu_convolve(ctx, ne, dE, fwhm):
    import torch
    rng = np.random.default_rng(ne)
    x = rng.uniform(0.0, 4.0, (3, ne)) + np.sin(np.arange(ne) * 0.01)[None, :]
    y = ctx.convolve_gaussian(x, dE, fwhm).cpu().numpy()
    ym = ctx.convolve_gaussian(x, dE, fwhm, mix=[2.0, 1.0, 0.5]).cpu().numpy()
    torch.cuda.synchronize()
    ref = oracle.convolve_gaussian(x, dE, fwhm)
    refm = oracle.convolve_gaussian(x, dE, fwhm, mix=[2.0, 1.0, 0.5])
    for m in range(3):
        assert nrel(y[m], ref[m]) < TOL
    assert nrel(ym, refm) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("nT,nan_below", [(1, False), (7, False), (16, False), (16, True), (20, False),
                                          (32, False)])
def test_gpu_maxwell(ctx, nT, nan_below):
    """Maxwell average against the oracle for every temperature bucket of the kernel (8 / 16 / 32);
    nan_below: Omega holds NaN at the points not above a pair's threshold, which reading U1 never
    integrates (the oracle starts at the first point above threshold) - the GPU must not read them
    into the sum either."""
    import torch
    rng = np.random.default_rng(4)
    ne, npair = 5000, 700
    E = 0.5 + np.arange(ne) * (59.5 / (ne - 1))
    Eth = np.sort(rng.uniform(0.0, 50.0, npair))
    om = rng.uniform(0.0, 3.0, (ne, npair)) * (E[:, None] > Eth[None, :])
    if nan_below:
        om[~(E[:, None] > Eth[None, :])] = np.nan
    kT = list(np.geomspace(0.03, 60.0, nT))
    ups = ctx.maxwell_average(om, E, Eth, kT).cpu().numpy()
    torch.cuda.synchronize()
    ref = oracle.maxwell_average(om, E, Eth, kT)
    for p in range(npair):
        assert nrel(ups[p], ref[p]) < TOL, p


@pytest.mark.gpu
def test_gpu_post_rejects_bad_args(ctx):
    import paper_1403_5524_b200 as rmx
    with pytest.raises(rmx.RmxError):
        ctx.convolve_gaussian(np.zeros(10), dE=0.1, fwhm=0.1)   # fwhm < 2 dE
    with pytest.raises(rmx.RmxError):
        ctx.maxwell_average(np.zeros((5, 2)), np.arange(5.0), np.zeros(2), [])
