"""NEXT-2 of SURVEY.md §8(f): level-pair collision strengths over several symmetries (partial
waves), Omega_ab(E) = sum_s g_s sum_{i in a, j in b} |T^s_ij(E)|^2 (DESIGN.md
reading L1).

CPU (`-m "not gpu"`): the oracle's oracle.level_omega is pinned to what the definition and the
already-pinned |T|^2 fix - a hand-summed 3-channel example, the one-channel-per-level reduction to
|T|^2 itself, the single-channel closed form 4 sin^2(delta), symmetry, the row-sum identity
sum_b Omega_ab = sum_{i in a} 4(1 - [(I + K^2)^-1]_ii), and closed levels left at zero.
GPU (`-m gpu`): rmx_collision_strength_levels and the fused rmx_sweep_levels against the oracle on
seeded multi-symmetry inputs, normwise 1e-8 per energy (the |T|^2 bar, BASELINE.json:5).
"""
import math

import numpy as np
import pytest

import oracle
import rmx_synth as syn

TOL = 1e-8


def nrel(x, ref):
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (den if den > 0 else 1.0))


# ----------------------------------------------------------------------------- oracle pins
def test_hand_summed_example():
    T2 = np.array([[1.0, 2.0, 3.0], [2.0, 5.0, 7.0], [3.0, 7.0, 11.0]])
    om = oracle.level_omega(T2, [0, 1, 3], n_open=3, g=0.5)
    ref = 0.5 * np.array([[1.0, 2.0 + 3.0], [2.0 + 3.0, 5.0 + 7.0 + 7.0 + 11.0]])
    assert np.array_equal(om, ref)


def test_closed_level_left_zero():
    T2 = np.arange(16.0).reshape(4, 4)
    om = oracle.level_omega(T2, [0, 2, 3, 4], n_open=3)
    assert om[2, :].tolist() == [0.0, 0.0, 0.0] and om[:, 2].tolist() == [0.0, 0.0, 0.0]
    assert om[0, 0] == 0 + 1 + 4 + 5 and om[1, 1] == 10 and om[0, 1] == 2 + 6


def _oracle_T2(c, e):
    E = c.E[e:e + 1]
    F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
    no = syn.n_open(c.eps, E)
    R, _ = oracle.R(c.w, c.Ek, c.a, E[0])
    K, _, _ = oracle.K(R, F[0], G[0], Fp[0], Gp[0], c.a)
    T2, rs, _, _, _, _ = oracle.T2(K, int(no[0]))
    return K, T2, rs, int(no[0])


def test_one_channel_per_level_is_T2():
    lev, E, cases = syn.symmetry_cases(1, 9, seed=3, max_ch=1)
    c, ls = cases[0]
    for e in range(0, len(E), 3):
        K, T2, rs, no = _oracle_T2(c, e)
        om = oracle.level_omega(T2, ls, no)
        assert np.array_equal(om[:no, :no], T2[:no, :no])


def test_single_channel_closed_form():
    # nch = 1, all open: Omega = |T|^2 = 4 sin^2(delta) = 4 K^2 / (1 + K^2)
    lev, E, cases = syn.symmetry_cases(1, 1, seed=5, max_ch=1, lev_hi=0.1)
    c, ls = cases[0]
    for e in range(len(E)):
        K, T2, rs, no = _oracle_T2(c, e)
        om = oracle.level_omega(T2, ls, no)
        k = K[0, 0]
        assert math.isclose(om[0, 0], 4 * k * k / (1 + k * k), rel_tol=1e-13)


def test_symmetry_and_row_sum_identity():
    lev, E, cases = syn.symmetry_cases(2, 6, seed=11)
    for c, ls in cases:
        for e in (0, len(E) // 2, len(E) - 1):
            K, T2, rs, no = _oracle_T2(c, e)
            om = oracle.level_omega(T2, ls, no)
            assert nrel(om, om.T) < 1e-13
            Ko = K[:no, :no]
            y = np.diag(np.linalg.inv(np.eye(no) + Ko @ Ko))
            nlo = int(np.searchsorted(ls[1:], no, side="right"))
            for la in range(nlo):
                i0, i1 = ls[la], ls[la + 1]
                assert math.isclose(om[la].sum(), 4.0 * np.sum(1.0 - y[i0:i1]), rel_tol=1e-11)
                assert om[la].sum() <= 4.0 * (i1 - i0) * (1 + 1e-12)


def test_weights_are_linear():
    lev, E, cases = syn.symmetry_cases(1, 4, seed=2)
    c, ls = cases[0]
    K, T2, rs, no = _oracle_T2(c, 2)
    assert np.allclose(oracle.level_omega(T2, ls, no, g=2.5), 2.5 * oracle.level_omega(T2, ls, no),
                       rtol=1e-15, atol=0)


def test_level_start_groups_equal_thresholds():
    c = syn.make_case("darc", ne=4)
    ls = syn.level_start(c.eps)
    assert len(ls) == 301 and ls[0] == 0 and ls[-1] == 2000
    sizes = np.diff(ls)
    assert sorted(set(sizes.tolist())) == [6, 7] and (sizes == 7).sum() == 200
    for a in range(300):
        assert np.all(c.eps[ls[a]:ls[a + 1]] == c.eps[ls[a]])


# ----------------------------------------------------------------------------- GPU parity
@pytest.fixture(scope="module")
def ctx():
    import paper_1403_5524_b200 as rmx
    return rmx.Context()


def _oracle_omega(cases, E, weights):
    nlevel = len(cases[0][1]) - 1
    out = np.zeros((len(E), nlevel, nlevel))
    for (c, ls), g in zip(cases, weights):
        F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
        no = syn.n_open(c.eps, E)
        ref = oracle.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, np.arange(len(E)), want=("T2",))
        for e in range(len(E)):
            out[e] += oracle.level_omega(ref["T2"][e], ls, int(no[e]), g)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("nlevel,max_ch,nlev", [(7, 3, 300), (60, 4, 700)])
def test_gpu_levels_multi_symmetry(ctx, nlevel, max_ch, nlev):
    import torch
    lev, E, cases = syn.symmetry_cases(3, nlevel, seed=7, nlev=nlev, ne=9, max_ch=max_ch)
    weights = [1.0, 3.0, 5.0]
    ref = _oracle_omega(cases, E, weights)
    om_fused = torch.zeros(ref.shape, dtype=torch.float64, device="cuda")
    om_calls = torch.zeros_like(om_fused)
    for (c, ls), g in zip(cases, weights):
        F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
        no = syn.n_open(c.eps, E)
        ctx.sweep_levels(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, ls, g=g, omega=om_fused, batch=4)
        R, st = ctx.build_R(c.w, c.Ek, c.a, E)
        K, st = ctx.match_K(R, F, G, Fp, Gp, c.a, no, status=st)
        ctx.collision_strength_levels(K, ls, g=g, n_open=no, omega=om_calls, status=st)
        assert int((st != 0).sum()) == 0
    torch.cuda.synchronize()
    for om in (om_fused.cpu().numpy(), om_calls.cpu().numpy()):
        for e in range(len(E)):
            assert nrel(om[e], ref[e]) < TOL, (e, nrel(om[e], ref[e]))
            assert np.all(om[e][ref[e] == 0] == 0)  # closed levels untouched


@pytest.mark.gpu
def test_gpu_levels_darc_sample(ctx):
    """darc shapes (2000 channels in 300 levels): fused sweep_levels at two mesh energies against
    the oracle's level sums of its own |T|^2."""
    import torch
    c = syn.make_case("darc")
    idx = np.array([30000, 90000])
    E = c.E[idx]
    ls = syn.level_start(c.eps)
    F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
    no = syn.n_open(c.eps, E)
    out = ctx.sweep_levels(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, ls, g=1.0)
    torch.cuda.synchronize()
    om = out["omega"].cpu().numpy()
    ref = oracle.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, np.arange(2), want=("T2",))
    for e in range(2):
        r = oracle.level_omega(ref["T2"][e], ls, int(no[e]))
        assert nrel(om[e], r) < TOL, (e, nrel(om[e], r))
