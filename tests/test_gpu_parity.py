"""GPU parity: the CUDA path (through the C ABI, librmx.so) against the CPU oracle on the same
seeded inputs. Tolerances are BASELINE.json:5's, read normwise per energy (reading T1):
    R: 1e-10, K (open-open block K_oo): 1e-10, |T|^2: 1e-8,
excluding energies within 1e-6 Ry of a pole (BASELINE.json:5) or of a threshold (reading T3).
Sizes span several tiles and ragged tails (R tiles 64/128, LU/Cholesky panels 32, k-slabs 32).
"""
import numpy as np
import pytest

import oracle
import rmx_synth as syn

pytestmark = pytest.mark.gpu

TOL_R, TOL_K, TOL_T2 = 1e-10, 1e-10, 1e-8


@pytest.fixture(scope="module")
def ctx():
    import paper_1403_5524_b200 as rmx
    return rmx.Context()


def nrel(x, ref):
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (den if den > 0 else 1.0))


def excluded(c, E):
    dp = np.min(np.abs(E - c.Ek))
    dt = np.min(np.abs(E - c.eps))
    return dp < 1e-6 or dt < 1e-6


def run_three_calls(ctx, c, idx):
    import torch
    E = c.E[idx]
    F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
    no = syn.n_open(c.eps, E)
    R, st = ctx.build_R(c.w, c.Ek, c.a, E)
    K, st = ctx.match_K(R, F, G, Fp, Gp, c.a, no, status=st)
    T2, rs, st = ctx.collision_strength(K, no, status=st)
    torch.cuda.synchronize()
    return dict(R=R.cpu().numpy(), K=K.cpu().numpy(), T2=T2.cpu().numpy(), rowsum=rs.cpu().numpy(),
                status=st.cpu().numpy(), n_open=no, F=F, G=G, Fp=Fp, Gp=Gp)


KAPPA_MAX = 1e7  # scaled cond_1(A) above which K's 1e-10 bar is a conditioning exclusion (reading T4)


def scaled_cond(R, G, Gp, a):
    """cond_1 of A = diag(G) - aR diag(G') with unit-max columns (closed-channel columns carry
    e^{-kappa a}; column scaling does not change K_oo, so this is the conditioning that matters)."""
    A = np.diag(G) - a * R * Gp[None, :]
    As = A / np.max(np.abs(A), axis=0)[None, :]
    return float(np.linalg.cond(As, 1))


def compare(c, idx, gpu, threads=None):
    E = c.E[idx]
    ref = oracle.sweep(c.w, c.Ek, c.a, E, gpu["F"], gpu["G"], gpu["Fp"], gpu["Gp"], gpu["n_open"],
                       np.arange(len(idx)), threads=threads)
    worst = dict(R=0.0, K=0.0, T2=0.0, rowsum=0.0)
    n_checked, cond_excl = 0, []
    for p in range(len(idx)):
        if excluded(c, E[p]):
            continue
        assert gpu["status"][p] == 0 and ref["status"][p] == 0, (p, gpu["status"][p], ref["status"][p])
        o = gpu["n_open"][p]
        worst["R"] = max(worst["R"], nrel(gpu["R"][p], ref["R"][p]))
        if o:
            ek = nrel(gpu["K"][p][:o, :o], ref["K"][p][:o, :o])
            if ek >= TOL_K:
                kap = scaled_cond(ref["R"][p], gpu["G"][p], gpu["Gp"][p], c.a)
                assert kap > KAPPA_MAX and ek < 1e-15 * kap, (p, E[p], ek, kap)
                cond_excl.append((int(idx[p]), ek, kap))
            else:
                worst["K"] = max(worst["K"], ek)
        worst["T2"] = max(worst["T2"], nrel(gpu["T2"][p], ref["T2"][p]))
        worst["rowsum"] = max(worst["rowsum"], nrel(gpu["rowsum"][p], ref["rowsum"][p]))
        n_checked += 1
    assert n_checked > 0
    assert worst["R"] < TOL_R, worst
    assert worst["K"] < TOL_K, worst
    assert worst["T2"] < TOL_T2, worst
    assert worst["rowsum"] < TOL_T2, worst
    assert len(cond_excl) <= max(1, n_checked // 4), cond_excl
    if cond_excl:
        print(f"conditioning exclusions (index, errK, scaled cond): {cond_excl}")
    return worst, ref


def stagewise(ctx, c, idx, ref, gpu, threads=None):
    """Stage-isolated parity: the GPU matching fed with the oracle's R, and the GPU T epilogue fed
    with the oracle's K, must each meet the bar with no conditioning exclusions (this isolates the
    kernels' own rounding from the R rounding propagated through an ill-conditioned matching)."""
    import torch
    F, G, Fp, Gp, no = gpu["F"], gpu["G"], gpu["Fp"], gpu["Gp"], gpu["n_open"]
    K, st = ctx.match_K(torch.from_numpy(ref["R"]), F, G, Fp, Gp, c.a, no)
    T2, rs, st = ctx.collision_strength(torch.from_numpy(ref["K"]), no, status=st)
    torch.cuda.synchronize()
    K, T2, rs = K.cpu().numpy(), T2.cpu().numpy(), rs.cpu().numpy()
    E = c.E[idx]
    for p in range(len(idx)):
        if excluded(c, E[p]):
            continue
        o = no[p]
        if o:
            assert nrel(K[p][:o, :o], ref["K"][p][:o, :o]) < TOL_K, p
        assert nrel(T2[p], ref["T2"][p]) < TOL_T2, p
        assert nrel(rs[p], ref["rowsum"][p]) < TOL_T2, p


def test_tiny_config_all_energies(ctx):
    """BASELINE.json:7 at full size (1000 energies, nch = 8: small-channel R path)."""
    c = syn.make_case("tiny")
    idx = np.arange(c.ne)
    gpu = run_three_calls(ctx, c, idx)
    compare(c, idx, gpu)
    # R bitwise symmetric (upper triangle mirrored), closed columns exactly -e_j
    assert np.array_equal(gpu["R"], np.swapaxes(gpu["R"], 1, 2))
    for p in range(3):
        o = gpu["n_open"][p]
        for j in range(o, 8):
            e = np.zeros(8)
            e[j] = -1.0
            assert np.array_equal(gpu["K"][p][:, j], e)


def test_small_config_sampled(ctx):
    """BASELINE.json:8 (nch = 64 -> 64-tile DMMA path, nlev = 3000), 96 energies incl. poles/thresholds."""
    c = syn.make_case("small")
    idx = syn.parity_sample(c, 80)
    gpu = run_three_calls(ctx, c, idx)
    _, ref = compare(c, idx, gpu)
    stagewise(ctx, c, idx, ref, gpu)


@pytest.mark.parametrize("nch,nlev,seed", [(150, 1000, 1), (203, 517, 2), (37, 77, 3), (1, 5, 4),
                                           (33, 64, 5), (129, 257, 6)])
def test_ragged_shapes(ctx, nch, nlev, seed):
    """Several R tiles with ragged tails (nch mod 128/64 != 0), odd nlev (ldw padding, TMA zero
    fill), LU panels with ragged last panel, closed channels (eps_hi > 0)."""
    c = syn.brute_force_case(nch, nlev, seed, ne=12, lo=0.5, hi=9.0, a=12.0, eps_hi=4.0)
    idx = np.arange(c.ne)
    gpu = run_three_calls(ctx, c, idx)
    _, ref = compare(c, idx, gpu)
    stagewise(ctx, c, idx, ref, gpu)
    assert np.array_equal(gpu["R"], np.swapaxes(gpu["R"], 1, 2))


def test_bp_config_sampled(ctx):
    """BASELINE.json:9 shape (nch = 500, nlev = 15000, closed channels) on 10 sampled energies."""
    c = syn.make_case("bp", ne=2000)
    idx = syn.parity_sample(c, 6, n_pole=2, n_thresh=2)
    gpu = run_three_calls(ctx, c, idx)
    _, ref = compare(c, idx, gpu, threads=oracle.default_threads())
    stagewise(ctx, c, idx, ref, gpu)


def test_pole_and_edge_status(ctx):
    """E on a pole (|E - E_k| < 1e-10) -> RMX_E_POLE and NaN R; n_open = 0 -> |T|^2 = 0."""
    import torch
    c = syn.brute_force_case(40, 100, 9, ne=4, lo=1.0, hi=5.0)
    E = np.array([c.Ek[50], c.Ek[50] + 5e-11, 2.5, 3.0])
    F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
    no = np.array([40, 40, 0, 40], dtype=np.int32)
    R, st = ctx.build_R(c.w, c.Ek, c.a, E)
    K, st = ctx.match_K(R, F, G, Fp, Gp, c.a, no, status=st)
    T2, rs, st = ctx.collision_strength(K, no, status=st)
    torch.cuda.synchronize()
    st = st.cpu().numpy()
    assert st[0] == 1 and st[1] == 1 and st[2] == 0 and st[3] == 0
    assert torch.isnan(R[0]).all() and torch.isnan(R[1]).all()
    assert (T2[2] == 0).all() and (rs[2] == 0).all()


def test_sweep_matches_three_calls_and_is_batch_invariant(ctx):
    """rmx_sweep (fused driver, K computed in place of R) gives bitwise the same row sums as the
    three-call pipeline, for any batch size (per-energy arithmetic independent of batching)."""
    import torch
    c = syn.brute_force_case(70, 300, 11, ne=40, lo=0.5, hi=9.0, a=12.0, eps_hi=3.0)
    idx = np.arange(c.ne)
    gpu = run_three_calls(ctx, c, idx)
    F, G, Fp, Gp = syn.asymptotic(c.eps, c.E, c.a)
    no = syn.n_open(c.eps, c.E)
    outs = []
    dump = [0, c.ne // 2, c.ne - 1]
    for batch in (0, 1, 7):
        out = ctx.sweep(c.w, c.Ek, c.a, c.E, F, G, Fp, Gp, no, batch=batch, dump_idx=dump)
        torch.cuda.synchronize()
        outs.append({k: v.cpu().numpy() for k, v in out.items()})
    for o in outs:
        assert np.array_equal(o["rowsum"], gpu["rowsum"])
        assert np.array_equal(o["status"], gpu["status"])
        assert np.array_equal(o["R"], gpu["R"][dump])
        assert np.array_equal(o["T2"], gpu["T2"][dump])
        for d, e in enumerate(dump):
            on = no[e]
            assert np.array_equal(o["K"][d][:, :on], gpu["K"][e][:, :on])


def test_sweep_host_e2e(ctx):
    """rmx_sweep_host: host buffers in/out, same row sums as the device sweep."""
    import paper_1403_5524_b200 as rmx
    import torch
    c = syn.brute_force_case(64, 200, 12, ne=20, lo=0.5, hi=9.0, a=12.0, eps_hi=3.0)
    F, G, Fp, Gp = syn.asymptotic(c.eps, c.E, c.a)
    no = syn.n_open(c.eps, c.E)
    dev = ctx.sweep(c.w, c.Ek, c.a, c.E, F, G, Fp, Gp, no)
    torch.cuda.synchronize()
    rs, st, h2d, d2h = ctx.sweep_host(c.w, c.Ek, c.a, c.E, F, G, Fp, Gp, no)
    assert np.array_equal(rs, dev["rowsum"].cpu().numpy())
    assert np.array_equal(st, dev["status"].cpu().numpy())
    assert h2d > 0 and d2h == rs.nbytes + st.nbytes
    assert rmx.load_library().rmx_sm_target() == 100
