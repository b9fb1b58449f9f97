"""Degenerate and error cases of the C ABI on the GPU (include/rmx.h error model):
empty and invalid sizes are synchronous RMX_EINVAL; an exact zero pivot is RMX_E_SINGULAR and a
non-finite input RMX_E_NONFINITE for that energy only (the batch is never aborted); one channel and
one pole reduce to the single-channel closed form K = -(G - aRG')^{-1}(F - aRF') with
R = w^2 / (2a (E_1 - E)) (Eq. 1-2 under reading R1); both R formations agree on
the INT8 path's size boundary nch = 256 with a single pole."""
import numpy as np
import pytest

import rmx_synth as syn

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_1403_5524_b200 as rmx
    return rmx.Context()


def test_empty_and_invalid_sizes_are_einval(ctx):
    import paper_1403_5524_b200 as rmx
    c = syn.brute_force_case(8, 20, 1, ne=3, lo=0.5, hi=5.0)
    F, G, Fp, Gp = syn.asymptotic(c.eps, c.E, c.a)
    with pytest.raises(rmx.RmxError):
        ctx.build_R(c.w, c.Ek, c.a, np.zeros(0))                      # ne = 0
    with pytest.raises(rmx.RmxError):
        ctx.build_R(c.w, c.Ek, -1.0, c.E)                             # a <= 0
    with pytest.raises(rmx.RmxError):
        ctx.build_R(np.zeros((0, 20)), c.Ek, c.a, c.E)                # nch = 0
    R, st = ctx.build_R(c.w, c.Ek, c.a, c.E)
    with pytest.raises(rmx.RmxError):
        ctx.match_K(R, F, G, Fp, Gp, 0.0)                             # a <= 0
    with pytest.raises(rmx.RmxError):
        ctx.sweep(c.w, c.Ek, c.a, np.zeros(0), F[:0], G[:0], Fp[:0], Gp[:0])  # ne = 0
    # the context stays usable after the argument errors
    R2, st2 = ctx.build_R(c.w, c.Ek, c.a, c.E)
    assert np.array_equal(R2.cpu().numpy(), R.cpu().numpy())


def test_singular_and_nonfinite_status_per_energy(ctx):
    """w = 0 makes R = 0 and A = diag(G): a zero G_j is an exact zero pivot (RMX_E_SINGULAR) at that
    energy only; a NaN in F' reaches K (RMX_E_NONFINITE); the other energies are untouched."""
    import torch
    nch, nlev, ne = 12, 30, 4
    rng = np.random.default_rng(3)
    w = np.zeros((nch, nlev))
    Ek = np.sort(rng.uniform(10.0, 20.0, nlev))
    E = np.array([1.0, 2.0, 3.0, 4.0])
    F = rng.uniform(0.5, 1.5, (ne, nch))
    G = rng.uniform(0.5, 1.5, (ne, nch))
    Fp = rng.uniform(-1.0, 1.0, (ne, nch))
    Gp = rng.uniform(-1.0, 1.0, (ne, nch))
    G[1, 5] = 0.0          # energy 1: zero pivot
    Fp[2, 3] = np.nan      # energy 2: NaN through aRF' (R = 0 but 0 * NaN = NaN)
    no = np.full(ne, nch, dtype=np.int32)
    R, st = ctx.build_R(w, Ek, 7.0, E)
    K, st = ctx.match_K(R, F, G, Fp, Gp, 7.0, no, status=st)
    T2, rs, st = ctx.collision_strength(K, no, status=st)
    torch.cuda.synchronize()
    s = st.cpu().numpy()
    assert s[1] == 2 and s[2] == 3, s
    assert s[0] == 0 and s[3] == 0, s
    # R = 0: K = -G^{-1} F exactly (diagonal); row sums of |T|^2 = 4k^2/(1+k^2) per channel
    Kn = K.cpu().numpy()
    for e in (0, 3):
        assert np.allclose(np.diag(Kn[e]), -F[e] / G[e], rtol=1e-15, atol=0)
        off = Kn[e] - np.diag(np.diag(Kn[e]))
        assert np.all(off == 0.0)
        k = -F[e] / G[e]
        assert np.allclose(rs.cpu().numpy()[e], 4 * k * k / (1 + k * k), rtol=1e-13, atol=0)


def test_single_channel_single_pole_closed_form(ctx):
    """nch = 1, nlev = 1: R = w^2/(2a(E_1 - E)) and K = -(G - aRG')^{-1}(F - aRF') as scalars; |T|^2 =
    4K^2/(1+K^2) (T = 2iK/(1 - iK))."""
    import torch
    w = np.array([[0.7]])
    Ek = np.array([3.0])
    a = 5.0
    E = np.array([0.5, 1.25, 2.9, 3.1, 4.0])
    rng = np.random.default_rng(5)
    F, G = rng.uniform(0.2, 1.0, (5, 1)), rng.uniform(0.2, 1.0, (5, 1))
    Fp, Gp = rng.uniform(-1.0, 1.0, (5, 1)), rng.uniform(-1.0, 1.0, (5, 1))
    no = np.ones(5, dtype=np.int32)
    R, st = ctx.build_R(w, Ek, a, E)
    K, st = ctx.match_K(R, F, G, Fp, Gp, a, no, status=st)
    T2, rs, st = ctx.collision_strength(K, no, status=st)
    torch.cuda.synchronize()
    Rr = 0.7 ** 2 / (2 * a * (3.0 - E))
    Kr = -(F[:, 0] - a * Rr * Fp[:, 0]) / (G[:, 0] - a * Rr * Gp[:, 0])
    assert np.allclose(R.cpu().numpy()[:, 0, 0], Rr, rtol=1e-14, atol=0)
    assert np.allclose(K.cpu().numpy()[:, 0, 0], Kr, rtol=1e-12, atol=0)
    assert np.allclose(rs.cpu().numpy()[:, 0], 4 * Kr ** 2 / (1 + Kr ** 2), rtol=1e-12, atol=0)
    assert np.all(st.cpu().numpy() == 0)


def test_int8_and_dmma_agree_at_the_boundary_single_pole(ctx):
    """nch = 256 (the smallest INT8-CRT size) and nlev = 1: R = w w^T / (2a(E_1 - E)) exactly up to the
    fixed-point rounding; both R formations against the closed form."""
    import paper_1403_5524_b200 as rmx
    import torch
    rng = np.random.default_rng(8)
    w = rng.normal(0.0, 0.3, (256, 1))
    Ek = np.array([2.0])
    E = np.array([0.5, 1.999, 2.5])
    ref = np.einsum("i,j->ij", w[:, 0], w[:, 0])[None] / (2 * 4.0 * (2.0 - E))[:, None, None]
    c8 = rmx.Context()
    c8.set_r_algo(rmx.R_INT8)
    for cx in (ctx, c8):
        R, st = cx.build_R(w, Ek, 4.0, E)
        torch.cuda.synchronize()
        Rn = R.cpu().numpy()
        for e in range(len(E)):
            assert np.max(np.abs(Rn[e] - ref[e])) / np.max(np.abs(ref[e])) < 1e-13
        assert np.all(st.cpu().numpy() == 0)
