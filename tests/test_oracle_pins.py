"""Pins for the CPU oracle (oracle/rmx_oracle.c) against what the paper and mathematics fix,
never against the oracle itself (task rule ③). Each test names the passage it checks.

The paper prints no R, K, T or collision-strength values, so the pins are
closed forms, brute force, invariants and physical identities, chosen so that a dropped
term, a wrong sign/index or a transposed operand anywhere in the oracle fails one:

  R : SPEC examples (golden), brute force (1/2a) P^T (H-E)^{-1} P, non-square/permuted w,
      pole residue, far field, pole guard.
  K : single-channel phase-shift closed form tan(arctan(k a R) - theta), independent
      symmetric-route formula, decoupled channels, continuity across R-poles,
      closed columns and closed-channel rescaling invariance, K_oo symmetry.
  T : |T|^2 = 4 sin^2(delta), spectral route via eigh(K), unitarity, row-sum identity,
      bounds; whole-sweep consistency and thread-count invariance.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
import rmx_synth as syn

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def nrel(x, ref):
    """Normwise relative error max|x - ref| / max|ref| (reading T1)."""
    x, ref = np.asarray(x), np.asarray(ref)
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (den if den > 0 else 1.0))


# ----------------------------------------------------------------------------- R pins

def test_R_golden_spec_examples():
    """SPEC.md:206-207 examples, converted to the north_star sign/prefactor."""
    g = json.load(open(os.path.join(GOLDEN, "spec_kernel_examples.json")))
    for c in g["cases"]:
        R, st = oracle.R(np.array(c["w"]), np.array(c["Ek"]), c["a"], c["E"])
        assert st == 0
        np.testing.assert_allclose(R, np.array(c["R_north"]), rtol=1e-15, atol=0)
        # and the paper-sign relation R_north = -R_paper/(2a) (reading R1)
        np.testing.assert_allclose(R, -np.array(c["R_paper"]) / (2 * c["a"]), rtol=1e-15)


def test_R_single_pole_closed_form():
    """Single pole: R = w^2 / (2a (E_k - E)) (BASELINE.json:5 with nlev = 1)."""
    for (w0, ek, E, a) in [(0.7, 1.3, 0.2, 20.0), (-2.0, -1.0, 3.5, 12.0), (1e-3, 3.1, 3.0999, 15.0)]:
        R, st = oracle.R(np.array([[w0]]), np.array([ek]), a, E)
        assert st == 0
        assert abs(R[0, 0] - w0 * w0 / (2 * a * (ek - E))) <= 1e-15 * abs(R[0, 0])


def test_R_nonsquare_permuted_amplitudes():
    """w with distinct rows and nlev != nch: R_ij = sum_k w_ik w_jk d_k / 2a; a transposed
    or mis-indexed operand changes individual entries. Hand-evaluated 2 x 3 case."""
    w = np.array([[1.0, 2.0, 0.0], [0.0, 3.0, -1.0]])
    Ek = np.array([0.0, 1.0, 4.0])
    E, a = 2.0, 0.5
    d = 1.0 / (Ek - E)  # [-1/2, -1, 1/2]
    expect = np.array([[1 * d[0] + 4 * d[1], 6 * d[1]],
                       [6 * d[1], 9 * d[1] + 1 * d[2]]]) / (2 * a)
    R, st = oracle.R(w, Ek, a, E)
    assert st == 0
    np.testing.assert_allclose(R, expect, rtol=1e-15, atol=1e-16)


@pytest.mark.parametrize("seed,nch,nlev", [(1, 6, 40), (2, 12, 150), (3, 20, 300)])
def test_R_brute_force_direct_solve(seed, nch, nlev):
    """north_star brute force: spectral sum == (1/2a) P^T (H - E)^{-1} P by a direct solve
    on the synthetic inner-region Hamiltonian whose eigenpairs generate E_k and w."""
    c = syn.brute_force_case(nch, nlev, seed, ne=7)
    for E in c.E:
        R, st = oracle.R(c.w, c.Ek, c.a, E)
        assert st == 0
        direct = c.P.T @ np.linalg.solve(c.H - E * np.eye(nlev), c.P) / (2 * c.a)
        # direct solve conditioning ~ 1/dist(E, spectrum); mesh keeps >= 1e-3 away
        assert nrel(R, direct) < 1e-9, (E, nrel(R, direct))


def test_R_entries_pinned():
    """oracle_R_entries (the reference of the full-size sampled R checks) against what fixes R
    independently of the oracle: the hand-evaluated 2 x 3 case (exact, both index orders), the
    brute force (1/2a) P^T (H - E)^{-1} P on sampled (i, j) pairs including diagonal, upper and
    lower entries (BASELINE.json:5; Eq. 1 in the north_star convention), and
    the pole guard. A scaled, transposed or mis-indexed sum fails one of these."""
    w = np.array([[1.0, 2.0, 0.0], [0.0, 3.0, -1.0]])
    Ek = np.array([0.0, 1.0, 4.0])
    E, a = 2.0, 0.5
    d = 1.0 / (Ek - E)
    expect = np.array([[1 * d[0] + 4 * d[1], 6 * d[1]],
                       [6 * d[1], 9 * d[1] + 1 * d[2]]]) / (2 * a)
    ii, jj = np.array([0, 0, 1, 1]), np.array([0, 1, 0, 1])
    vals, st = oracle.R_entries(w, Ek, a, E, ii, jj)
    assert st == 0
    np.testing.assert_allclose(vals, expect[ii, jj], rtol=1e-15, atol=1e-16)
    rng = np.random.default_rng(11)
    for seed, nch, nlev in [(4, 9, 60), (5, 17, 220)]:
        c = syn.brute_force_case(nch, nlev, seed, ne=5)
        ii = np.concatenate([np.arange(nch), rng.integers(0, nch, 40)])
        jj = np.concatenate([np.arange(nch), rng.integers(0, nch, 40)])
        for E in c.E:
            direct = c.P.T @ np.linalg.solve(c.H - E * np.eye(nlev), c.P) / (2 * c.a)
            vals, st = oracle.R_entries(c.w, c.Ek, c.a, E, ii, jj)
            assert st == 0
            err = np.max(np.abs(vals - direct[ii, jj])) / np.max(np.abs(direct))
            assert err < 1e-9, (seed, E, err)
    vals, st = oracle.R_entries(w, Ek, a, 1.0 + 1e-12, ii[:2], jj[:2])
    assert st == 1 and np.all(np.isnan(vals))


def test_R_small_config_is_its_own_brute_force():
    """Config 'small' (BASELINE.json:8) is generated as w = P^T V, so R(E) = (1/2a) P^T(H-E)^{-1}P
    holds for the config itself. Checked at 2 energies."""
    c = syn.make_case("small", ne=5)
    for E in c.E[[1, 3]]:
        R, st = oracle.R(c.w, c.Ek, c.a, E, threads=oracle.default_threads())
        direct = c.P.T @ np.linalg.solve(c.H - E * np.eye(c.nlev), c.P) / (2 * c.a)
        assert st == 0 and nrel(R, direct) < 1e-8


def test_R_pole_residue():
    """(E_k - E) R(E) -> w_k w_k^T / 2a as E -> E_k, error O(delta) (SURVEY pins)."""
    c = syn.brute_force_case(5, 30, 7, ne=3)
    k = 15
    target = np.outer(c.w[:, k], c.w[:, k]) / (2 * c.a)
    errs = []
    for delta in (1e-3, 1e-4, 1e-5, 1e-6):
        E = c.Ek[k] + delta
        R, st = oracle.R(c.w, c.Ek, c.a, E)
        errs.append(np.max(np.abs((c.Ek[k] - E) * R - target)))
    assert all(errs[i + 1] < errs[i] * 0.2 for i in range(3)), errs
    assert errs[-1] < 1e-4 * np.max(np.abs(target)) * 10


def test_R_far_field():
    """|E| >> max|E_k|: R(E) -> -W W^T / (2 a E) with error O(max|E_k|/|E|)."""
    c = syn.brute_force_case(4, 25, 9, ne=3)
    for E in (-1e6, 1e7):
        R, _ = oracle.R(c.w, c.Ek, c.a, E)
        ff = -(c.w @ c.w.T) / (2 * c.a * E)
        assert nrel(R, ff) < 3 * np.max(np.abs(c.Ek)) / abs(E)


def test_R_pole_guard_status():
    """|E - E_k| < 1e-10 -> status POLE and NaN outputs."""
    c = syn.brute_force_case(3, 10, 4, ne=3)
    R, st = oracle.R(c.w, c.Ek, c.a, c.Ek[4] + 5e-11)
    assert st == 1 and np.isnan(R).all()
    R, st = oracle.R(c.w, c.Ek, c.a, c.Ek[4] + 1e-9)
    assert st == 0 and np.isfinite(R).all()


# ----------------------------------------------------------------------------- K pins

def _one_channel(Rval, E, eps, a, i=0):
    F, G, Fp, Gp = syn.asymptotic(np.array([eps]), np.array([E]), a)
    k = math.sqrt(2 * (E - eps))
    th = k * a + 0.3 * i
    return F[0], G[0], Fp[0], Gp[0], k, th


@pytest.mark.parametrize("Rval,E,a", [(0.013, 1.7, 20.0), (-0.4, 0.33, 12.0), (2.5, 7.9, 25.0),
                                      (-1e-4, 0.05, 18.0)])
def test_K_single_channel_phase_shift(Rval, E, a):
    """nch = 1: K = tan(delta), delta = arctan(k a R) - theta (standard R-matrix phase shift;
    SURVEY §8(c) pins), and |T|^2 = 4 sin^2(delta) (S = exp(2 i delta), T = S - 1)."""
    F, G, Fp, Gp, k, th = _one_channel(Rval, E, 0.0, a)
    Kk, st, _ = oracle.K(np.array([[Rval]]), F, G, Fp, Gp, a)
    delta = math.atan(k * a * Rval) - th
    assert st == 0
    assert abs(Kk[0, 0] - math.tan(delta)) <= 1e-12 * max(1.0, abs(math.tan(delta)))
    t2, rs, tre, tim, unit, st = oracle.T2(Kk, 1)
    assert abs(t2[0, 0] - 4 * math.sin(delta) ** 2) < 1e-13
    # T = exp(2 i delta) - 1
    assert abs(tre[0, 0] - (math.cos(2 * delta) - 1)) < 1e-13
    assert abs(tim[0, 0] - math.sin(2 * delta)) < 1e-13
    assert unit < 1e-15 and abs(rs[0] - t2[0, 0]) < 1e-15


def _sym_route_K(R, F, G, Fp, Gp, a):
    """Independent route (needs all G' != 0, Wronskian FG' - F'G = -1):
    K = G'^-1 (D - aR)^-1 G'^-1 - diag(F'/G'), D = diag(G/G') (derivation in DESIGN.md §3)."""
    D = np.diag(G / Gp)
    M = np.linalg.solve(D - a * R, np.diag(1.0 / Gp))
    return np.diag(1.0 / Gp) @ M - np.diag(Fp / Gp)


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_K_independent_symmetric_route(seed):
    """All channels open: the LU route of the oracle equals the independently derived
    symmetric route (uses only the Wronskian normalisation)."""
    c = syn.brute_force_case(9, 80, seed, ne=5, lo=2.0, hi=8.0)
    for E in c.E:
        R, _ = oracle.R(c.w, c.Ek, c.a, E)
        F, G, Fp, Gp = (x[0] for x in syn.asymptotic(c.eps, np.array([E]), c.a))
        Kk, st, cond = oracle.K(R, F, G, Fp, Gp, c.a, want_cond=True)
        ref = _sym_route_K(R, F, G, Fp, Gp, c.a)
        assert st == 0
        assert nrel(Kk, ref) < 1e-10 * max(1.0, cond / 1e3)
        assert nrel(Kk, Kk.T) < 1e-11  # K symmetric iff Wronskian ∝ I


def test_K_decoupled_channels():
    """Block-diagonal w (channels {0,1,2} couple only to poles 0..19, {3,4} to 20..39):
    K is block diagonal and each block equals the solve of its own sub-problem."""
    rng = np.random.default_rng(5)
    w = np.zeros((5, 40))
    w[:3, :20] = rng.normal(0, 0.3, (3, 20))
    w[3:, 20:] = rng.normal(0, 0.3, (2, 20))
    Ek = np.sort(rng.uniform(0, 10, 40))
    a, E = 10.0, 4.321
    eps = np.zeros(5)
    F, G, Fp, Gp = (x[0] for x in syn.asymptotic(eps, np.array([E]), a))
    R, _ = oracle.R(w, Ek, a, E)
    Kk, _, _ = oracle.K(R, F, G, Fp, Gp, a)
    assert np.max(np.abs(Kk[:3, 3:])) < 1e-13 * np.max(np.abs(Kk))
    assert np.max(np.abs(Kk[3:, :3])) < 1e-13 * np.max(np.abs(Kk))
    # sub-problem 2 (channels 3,4): their phases use 0-based channel index i = 3,4 -> keep F,G
    R2, _ = oracle.R(w[3:, 20:], Ek[20:], a, E)
    K2, _, _ = oracle.K(R2, F[3:], G[3:], Fp[3:], Gp[3:], a)
    assert nrel(Kk[3:, 3:], K2) < 1e-12
    t2, rs, *_ = oracle.T2(Kk, 5)
    t2b, rsb, *_ = oracle.T2(K2, 2)
    assert nrel(t2[3:, 3:], t2b) < 1e-11 and np.max(np.abs(t2[:3, 3:])) < 1e-20


def test_K_continuous_across_R_pole():
    """R has a pole at E_k but K does not: K(E_k + d) - K(E_k - d) = O(d) (SURVEY pins)."""
    c = syn.brute_force_case(4, 30, 21, ne=3)
    k = 14
    jumps = []
    for d in (1e-3, 1e-4, 1e-5, 1e-6):
        Ks = []
        for E in (c.Ek[k] - d, c.Ek[k] + d):
            R, _ = oracle.R(c.w, c.Ek, c.a, E)
            F, G, Fp, Gp = (x[0] for x in syn.asymptotic(c.eps, np.array([E]), c.a))
            Ks.append(oracle.K(R, F, G, Fp, Gp, c.a)[0])
        jumps.append(np.max(np.abs(Ks[1] - Ks[0])))
    for i in range(3):
        assert jumps[i + 1] < 0.2 * jumps[i], jumps


def test_K_closed_columns_and_rescaling():
    """Closed channels (BASELINE.json:9 e^{-kappa a} functions): closed columns of K are
    exactly -e_j (B_{:,j} = A_{:,j}); K_oo is invariant when the closed-channel functions are
    rescaled to F = G = 1, F' = G' = -kappa."""
    c = syn.brute_force_case(8, 60, 31, ne=3, eps_hi=6.0)
    E = 3.0
    no = int(syn.n_open(c.eps, np.array([E]))[0])
    assert 0 < no < 8
    R, _ = oracle.R(c.w, c.Ek, c.a, E)
    F, G, Fp, Gp = (x[0].copy() for x in syn.asymptotic(c.eps, np.array([E]), c.a))
    Kk, st, _ = oracle.K(R, F, G, Fp, Gp, c.a)
    for j in range(no, 8):
        e = np.zeros(8)
        e[j] = -1.0
        assert np.max(np.abs(Kk[:, j] - e)) < 1e-9
    sc = np.exp(-np.sqrt(2 * (c.eps[no:] - E)) * c.a)
    F2, G2, Fp2, Gp2 = F.copy(), G.copy(), Fp.copy(), Gp.copy()
    for arr in (F2, G2, Fp2, Gp2):
        arr[no:] /= sc
    K2, _, _ = oracle.K(R, F2, G2, Fp2, Gp2, c.a)
    assert nrel(Kk[:no, :no], K2[:no, :no]) < 1e-11
    assert nrel(Kk[:no, :no], Kk[:no, :no].T) < 1e-11


# ----------------------------------------------------------------------------- T pins

def _rand_sym(n, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    X = rng.normal(0, scale, (n, n))
    return (X + X.T) / 2


@pytest.mark.parametrize("n,seed,scale", [(3, 1, 0.5), (10, 2, 2.0), (25, 3, 10.0)])
def test_T_spectral_route(n, seed, scale):
    """T = 2iK(I - iK)^{-1} = Q diag(2 i l/(1 - i l)) Q^T with K = Q diag(l) Q^T (eigh):
    a different algorithm for the same definition (BASELINE.json:5)."""
    Kk = _rand_sym(n, seed, scale)
    lam, Q = np.linalg.eigh(Kk)
    Tref = (Q * (2j * lam / (1 - 1j * lam))) @ Q.T
    t2, rs, tre, tim, unit, st = oracle.T2(Kk, n)
    assert st == 0
    assert nrel(tre + 1j * tim, Tref) < 1e-12
    assert nrel(t2, np.abs(Tref) ** 2) < 1e-11
    assert unit < 1e-13


def test_T_identities_and_open_block():
    """Row-sum identity sum_j |T_ij|^2 = -2 Re T_ii = 4(1 - [(I+K^2)^{-1}]_ii) (unitarity of
    S = I + T), 0 <= |T|^2 <= 4, symmetry, and zeros outside the open block."""
    n, no = 12, 7
    Kk = _rand_sym(n, 8, 3.0)
    t2, rs, tre, tim, unit, st = oracle.T2(Kk, no)
    Ko = Kk[:no, :no]
    Y = np.linalg.inv(np.eye(no) + Ko @ Ko)
    np.testing.assert_allclose(rs[:no], -2 * np.diag(tre)[:no], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(rs[:no], 4 * (1 - np.diag(Y)), rtol=1e-11, atol=1e-13)
    assert np.all(t2 >= 0) and np.all(t2 <= 4 + 1e-14)
    assert nrel(t2, t2.T) < 1e-12
    assert np.all(t2[no:, :] == 0) and np.all(t2[:, no:] == 0) and np.all(rs[no:] == 0)
    t2z, rsz, *_ = oracle.T2(Kk, 0)
    assert np.all(t2z == 0) and np.all(rsz == 0)


# ----------------------------------------------------------------------------- sweep pins

def _sweep_inputs(c, idx=None):
    F, G, Fp, Gp = syn.asymptotic(c.eps, c.E, c.a)
    no = syn.n_open(c.eps, c.E)
    idx = np.arange(c.ne) if idx is None else idx
    return F, G, Fp, Gp, no, idx


def test_sweep_matches_stepwise_and_threads_invariant():
    """oracle_sweep (long double end to end) == R -> K -> T2 step functions to rounding, and is
    bitwise identical for 1 and N threads (parallelism only splits independent work)."""
    c = syn.make_case("tiny", ne=40)
    F, G, Fp, Gp, no, idx = _sweep_inputs(c)
    s1 = oracle.sweep(c.w, c.Ek, c.a, c.E, F, G, Fp, Gp, no, idx, diag=True, threads=1)
    s4 = oracle.sweep(c.w, c.Ek, c.a, c.E, F, G, Fp, Gp, no, idx, diag=True, threads=4)
    for k in ("R", "K", "T2", "rowsum", "status"):
        assert np.array_equal(s1[k], s4[k]), k
    for p in (0, 5, 39):
        e = idx[p]
        R, _ = oracle.R(c.w, c.Ek, c.a, c.E[e])
        Kk, _, _ = oracle.K(R, F[e], G[e], Fp[e], Gp[e], c.a)
        t2, rs, *_ = oracle.T2(Kk, no[e])
        assert nrel(s1["R"][p], R) < 1e-15
        o = no[e]
        assert nrel(s1["K"][p][:o, :o], Kk[:o, :o]) < 1e-12
        assert nrel(s1["T2"][p], t2) < 1e-10
    assert np.all(s1["diag"][:, 0] < 1e-12)  # unitarity
    assert np.all(s1["diag"][:, 1] < 1e-11)  # asym(K_oo)
    assert np.all(s1["status"] == 0)


def test_tiny_config_open_channel_reading():
    """Tiny (BASELINE.json:7): E_0 = 0.05 == 0.01*5 in fp64, so with the strict open rule
     the first mesh points have n_o = 5, 6, 7 and then 8."""
    c = syn.make_case("tiny")
    no = syn.n_open(c.eps, c.E)
    assert c.E[0] == 0.05 and no[0] == 5
    assert no.min() == 5 and no.max() == 8 and (no < 8).sum() == 3
    assert c.ne + c.dropped_mesh_points == 1000


def test_wronskian_normalisation():
    """Open: F G' - F' G = -1 (reading §8(c) 4); closed: F = G, F' = G' = -kappa F."""
    eps = np.array([0.0, 0.3, 1.0, 2.5])
    E = np.array([0.7, 2.0])
    F, G, Fp, Gp = syn.asymptotic(eps, E, 12.0)
    no = syn.n_open(eps, E)
    for e in range(2):
        o = no[e]
        np.testing.assert_allclose((F * Gp - Fp * G)[e, :o], -1.0, rtol=1e-14)
        assert np.array_equal(F[e, o:], G[e, o:]) and np.array_equal(Fp[e, o:], Gp[e, o:])
