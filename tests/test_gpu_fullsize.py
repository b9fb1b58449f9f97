"""GPU parity at BASELINE.json's full sizes in the launch configuration bench.py times (SURVEY.md
§8(d)): the fused rmx_sweep over one bench block of 296 energies of config 'darc' (nch = 2000,
nlev = 40000; BASELINE.json:10) and of config 'fine' (nch = 1200, nlev = 30000, the 200 narrow
resonance poles inside the window; BASELINE.json:11).

Sampled outputs the oracle can compute one by one: full R, K_oo, |T|^2 and row sums of dumped
energies (oracle sweep, long double), plus R entries sampled at further dumped energies
(oracle_R_entries). Properties that hold at any size, checked on every energy of the block:
status OK, 0 <= sum_j |T_ij|^2 <= 4 (unitarity), and bitwise-symmetric dumped R.
Tolerances as tests/test_gpu_parity.py (BASELINE.json:5 read normwise per energy, reading T1; the
conditioning exclusion of reading T4 for K).
"""
import numpy as np
import pytest

import oracle
import rmx_synth as syn

pytestmark = pytest.mark.gpu

TOL_R, TOL_K, TOL_T2 = 1e-10, 1e-10, 1e-8
BATCH = 296  # = 2 x 148 SMs, bench.py's energies per step


def nrel(x, ref):
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (den if den > 0 else 1.0))


@pytest.fixture(scope="module")
def ctx():
    import paper_1403_5524_b200 as rmx
    return rmx.Context()


def _run_block(ctx, c, lo, dump_local):
    import torch
    E = c.E[lo:lo + BATCH]
    F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
    no = syn.n_open(c.eps, E)
    out = ctx.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, batch=BATCH, dump_idx=dump_local)
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    return E, F, G, Fp, Gp, no, res


def _check_block(c, E, F, G, Fp, Gp, no, res, full_local, entry_local):
    assert np.all(res["status"] == 0)
    rs = res["rowsum"]
    assert np.all(rs >= 0) and np.all(rs <= 4.0 * (1 + 1e-10)), rs.max()
    assert np.array_equal(res["R"], np.swapaxes(res["R"], 1, 2))
    dump = list(full_local) + list(entry_local)
    ref = oracle.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, np.array(full_local),
                       threads=oracle.default_threads())
    def excluded(x):  # BASELINE.json:5 pole exclusion + reading T3 (thresholds)
        return np.min(np.abs(x - c.Ek)) < 1e-6 or np.min(np.abs(x - c.eps)) < 1e-6

    for q, l in enumerate(full_local):
        if excluded(E[l]):
            continue
        d = dump.index(l)
        o = int(no[l])
        assert nrel(res["R"][d], ref["R"][q]) < TOL_R
        ek = nrel(res["K"][d][:o, :o], ref["K"][q][:o, :o])
        if ek >= TOL_K:  # reading T4: allowed only where the matching is ill-conditioned
            A = np.diag(G[l]) - c.a * ref["R"][q] * Gp[l][None, :]
            kap = float(np.linalg.cond(A / np.max(np.abs(A), axis=0)[None, :], 1))
            assert kap > 1e7 and ek < 1e-15 * kap, (l, ek, kap)
        assert nrel(res["T2"][d], ref["T2"][q]) < TOL_T2
        assert nrel(rs[l], ref["rowsum"][q]) < TOL_T2
    rng = np.random.default_rng(0)
    for l in entry_local:
        if excluded(E[l]):
            continue
        d = dump.index(l)
        ii = rng.integers(0, c.nch, 48)
        jj = rng.integers(0, c.nch, 48)
        vals, st = oracle.R_entries(c.w, c.Ek, c.a, E[l], ii, jj)
        assert st == 0
        scale = np.max(np.abs(res["R"][d]))
        assert np.max(np.abs(res["R"][d][ii, jj] - vals)) / scale < TOL_R


def test_darc_bench_block(ctx):
    c = syn.make_case("darc")
    full, entries = [0, 151], [37, 295]
    E, F, G, Fp, Gp, no, res = _run_block(ctx, c, 50000, full + entries)
    _check_block(c, E, F, G, Fp, Gp, no, res, full, entries)


def test_fine_bench_block(ctx):
    c = syn.make_case("fine")
    # a block inside the resonance window where the narrow poles sit
    lo = 200000
    full, entries = [5], [100, 250]
    E, F, G, Fp, Gp, no, res = _run_block(ctx, c, lo, full + entries)
    _check_block(c, E, F, G, Fp, Gp, no, res, full, entries)
