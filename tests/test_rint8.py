"""R formation on the INT8 tensor cores by exact CRT (rmx_set_r_algo(RMX_R_INT8), rint8.cu) against
the long-double oracle: R to the BASELINE.json:5 bar (1e-10 normwise; the fixed-point rounding of
X = W diag(d) and W leaves ~1e-14), bitwise symmetry, pole energies, ragged shapes; then the whole
R -> K -> |T|^2 sweep with INT8 R at the same bars as the DMMA path; and a full darc bench block
sampled against the oracle."""
import numpy as np
import pytest

import oracle
import rmx_synth as syn

pytestmark = pytest.mark.gpu


def nrel(x, ref):
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (den if den > 0 else 1.0))


@pytest.fixture(scope="module")
def ctx():
    import paper_1403_5524_b200 as rmx
    c = rmx.Context()
    c.set_r_algo(rmx.R_INT8)
    return c


@pytest.mark.parametrize("nch,nlev,seed", [(300, 1000, 1), (403, 517, 2), (257, 77, 3), (256, 5, 4),
                                           (529, 257, 6), (300, 2100, 7), (512, 300, 8), (784, 129, 9)])
def test_int8_R_matches_oracle(ctx, nch, nlev, seed):
    import torch
    c = syn.brute_force_case(nch, nlev, seed, ne=11, lo=0.5, hi=9.0, a=12.0, eps_hi=4.0)
    R, st = ctx.build_R(c.w, c.Ek, c.a, c.E)
    torch.cuda.synchronize()
    R = R.cpu().numpy()
    assert np.all(st.cpu().numpy() == 0)
    assert np.array_equal(R, np.swapaxes(R, 1, 2))
    worst = 0.0
    for p, E in enumerate(c.E):
        ref, _ = oracle.R(c.w, c.Ek, c.a, E)
        worst = max(worst, nrel(R[p], ref))
    assert worst < 1e-12, worst


_NOPAIR_SCRIPT = r"""
import numpy as np, torch, oracle, rmx_synth as syn, paper_1403_5524_b200 as rmx
ctx = rmx.Context(); ctx.set_r_algo(rmx.R_INT8)
c = syn.brute_force_case(529, 300, 9, ne=5, lo=0.5, hi=9.0, a=12.0, eps_hi=4.0)
R, st = ctx.build_R(c.w, c.Ek, c.a, c.E); torch.cuda.synchronize(); R = R.cpu().numpy()
assert np.all(st.cpu().numpy() == 0) and np.array_equal(R, np.swapaxes(R, 1, 2))
w = 0.0
for p, E in enumerate(c.E):
    ref, _ = oracle.R(c.w, c.Ek, c.a, E)
    w = max(w, float(np.max(np.abs(R[p] - ref)) / np.max(np.abs(ref))))
print("WORST", w)
"""


def test_int8_one_sm_kernel_layout():
    """The 1-SM GEMM layout (128 x 256 tiles, half tiles below the diagonal) that RMX_I8_NOPAIR selects
    for nch > 256 (the default there is the CTA-pair kernel; nch = 256 above runs the 1-SM kernel by
    default) - in a subprocess, since the switch is read once per process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RMX_I8_NOPAIR="1")
    out = subprocess.run([sys.executable, "-c", _NOPAIR_SCRIPT], cwd=root, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    worst = float(out.stdout.split("WORST")[-1])
    assert worst < 1e-12, worst


def test_int8_pole_status(ctx):
    import torch
    c = syn.brute_force_case(260, 300, 9, ne=4, lo=1.0, hi=5.0)
    E = np.array([c.Ek[50], 2.5])
    R, st = ctx.build_R(c.w, c.Ek, c.a, E)
    torch.cuda.synchronize()
    assert st.cpu().numpy().tolist() == [1, 0]
    assert torch.isnan(R[0]).all() and torch.isfinite(R[1]).all()


def test_int8_sweep_parity(ctx):
    """The fused sweep with INT8 R: K_oo and |T|^2 / row sums to the 1e-10 / 1e-8 bars."""
    import torch
    c = syn.brute_force_case(300, 900, 13, ne=10, lo=0.5, hi=9.0, a=12.0, eps_hi=3.0)
    F, G, Fp, Gp = syn.asymptotic(c.eps, c.E, c.a)
    no = syn.n_open(c.eps, c.E)
    out = ctx.sweep(c.w, c.Ek, c.a, c.E, F, G, Fp, Gp, no, batch=4, dump_idx=list(range(c.ne)))
    torch.cuda.synchronize()
    ref = oracle.sweep(c.w, c.Ek, c.a, c.E, F, G, Fp, Gp, no, np.arange(c.ne))
    for p in range(c.ne):
        o = int(no[p])
        assert nrel(out["R"][p].cpu().numpy(), ref["R"][p]) < 1e-12
        if o:
            assert nrel(out["K"][p].cpu().numpy()[:o, :o], ref["K"][p][:o, :o]) < 1e-10
        assert nrel(out["T2"][p].cpu().numpy(), ref["T2"][p]) < 1e-8
        assert nrel(out["rowsum"][p].cpu().numpy(), ref["rowsum"][p]) < 1e-8


def test_int8_darc_block(ctx):
    """darc (nch 2000, nlev 40000) in the bench launch configuration: INT8 R of 296 energies against the
    DMMA R (both fp64-accurate) and sampled oracle entries."""
    import torch
    import paper_1403_5524_b200 as rmx
    c = syn.make_case("darc")
    E = c.E[50000:50000 + 296]
    dump = [0, 100, 295]
    F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
    no = syn.n_open(c.eps, E)
    out8 = ctx.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, batch=296, dump_idx=dump)
    ctx64 = rmx.Context()
    out64 = ctx64.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, batch=296, dump_idx=dump)
    torch.cuda.synchronize()
    assert int((out8["status"] != 0).sum()) == 0
    rng = np.random.default_rng(0)
    for d, l in enumerate(dump):
        R8, R64 = out8["R"][d].cpu().numpy(), out64["R"][d].cpu().numpy()
        assert nrel(R8, R64) < 1e-12, nrel(R8, R64)
        ii, jj = rng.integers(0, c.nch, 40), rng.integers(0, c.nch, 40)
        vals, st = oracle.R_entries(c.w, c.Ek, c.a, E[l], ii, jj)
        assert np.max(np.abs(R8[ii, jj] - vals)) / np.max(np.abs(R8)) < 1e-12
        o = int(no[l])
        assert nrel(out8["T2"][d].cpu().numpy(), out64["T2"][d].cpu().numpy()) < 1e-8
    # row sums of all 296 energies: INT8 and DMMA R give the same |T|^2 row sums to the 1e-8 bar; the
    # three energies where they differ most are compared with the oracle, hard 1e-8 bar, both paths
    rs8, rs64 = out8["rowsum"].cpu().numpy(), out64["rowsum"].cpu().numpy()
    per = np.max(np.abs(rs8 - rs64), axis=1) / np.max(np.abs(rs64), axis=1)
    assert np.max(per) < 1e-8, np.sort(per)[-5:]
    worst = [int(x) for x in np.argsort(per)[-3:]]
    ref = oracle.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, np.array(worst), want=("rowsum",),
                       threads=oracle.default_threads())["rowsum"]
    for q, l in enumerate(worst):
        e8, e64 = nrel(rs8[l], ref[q]), nrel(rs64[l], ref[q])
        assert e8 < 1e-8 and e64 < 1e-8, (l, e8, e64)


def test_int8_many_poles_signed_residues(ctx):
    """nlev > 65000 switches the X residues to balanced int8 (the u8 x s8 accumulator bound): R still
    matches the oracle."""
    import torch
    rng = np.random.default_rng(5)
    nch, nlev = 260, 70001
    Ek = np.sort(rng.uniform(-5.0, 300.0, nlev))
    w = rng.normal(0.0, 0.05, (nch, nlev))
    E = np.array([0.7, 13.3, 57.9])
    R, st = ctx.build_R(w, Ek, 12.0, E)
    torch.cuda.synchronize()
    R = R.cpu().numpy()
    for p, x in enumerate(E):
        ref, _ = oracle.R(w, Ek, 12.0, x)
        assert nrel(R[p], ref) < 1e-12, (x, nrel(R[p], ref))


def test_int8_fine_block(ctx):
    """fine (nch 1200, nlev 30000; 200 narrow resonance poles |w| ~ 1e-3 inside the window, which the
    row-bound fixed-point rounding must not wash out): INT8 R against sampled oracle entries and the
    DMMA R on dumped energies, |T|^2 against the DMMA path."""
    import torch
    import paper_1403_5524_b200 as rmx
    c = syn.make_case("fine")
    E = c.E[200000:200000 + 296]
    dump = [0, 5, 250]
    F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
    no = syn.n_open(c.eps, E)
    out8 = ctx.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, batch=296, dump_idx=dump)
    ctx64 = rmx.Context()
    out64 = ctx64.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, batch=296, dump_idx=dump)
    torch.cuda.synchronize()
    assert int((out8["status"] != 0).sum()) == 0
    rng = np.random.default_rng(1)
    for d, l in enumerate(dump):
        R8, R64 = out8["R"][d].cpu().numpy(), out64["R"][d].cpu().numpy()
        assert nrel(R8, R64) < 1e-12, nrel(R8, R64)
        ii, jj = rng.integers(0, c.nch, 40), rng.integers(0, c.nch, 40)
        vals, st = oracle.R_entries(c.w, c.Ek, c.a, E[l], ii, jj)
        assert np.max(np.abs(R8[ii, jj] - vals)) / np.max(np.abs(R8)) < 1e-12
        assert nrel(out8["T2"][d].cpu().numpy(), out64["T2"][d].cpu().numpy()) < 1e-8


def test_int8_crt_worst_case_magnitude(ctx):
    """The CRT's exactness bound at its limit (rint8.cu: |P| <= nlev 2^106 < M/2, 0.23 M at the maximum
    nlev 131071): constant-sign amplitudes w > 0 and E below every pole (all d_k > 0), so every product
    w_ik d_k w_jk is positive and |P| reaches its maximum; nch = 300 runs the CTA-pair GEMM, nlev > 65000
    the balanced int8 residues. R against the long-double oracle."""
    import torch
    rng = np.random.default_rng(17)
    nch, nlev = 300, 131071
    Ek = np.sort(rng.uniform(1.0, 200.0, nlev))
    w = rng.uniform(0.01, 0.05, (nch, nlev))
    E = np.array([0.25, 0.9])
    R, st = ctx.build_R(w, Ek, 12.0, E)
    torch.cuda.synchronize()
    R = R.cpu().numpy()
    assert np.all(st.cpu().numpy() == 0)
    assert np.all(R > 0)
    for p, x in enumerate(E):
        ref, _ = oracle.R(w, Ek, 12.0, x, threads=oracle.default_threads())
        assert nrel(R[p], ref) < 1e-12, (x, nrel(R[p], ref))


@pytest.mark.parametrize("nch,nlev,seed", [(300, 1000, 11), (529, 2100, 12), (257, 77, 13), (640, 4096, 14),
                                           (384, 1023, 15)])
def test_int8_tc_conversion_bitwise(ctx, nch, nlev, seed, monkeypatch):
    """The X-residue conversion with the byte-weight sums on the tensor cores (oz_convert_tc_kernel, the
    default) and the dp4a conversion (oz_convert_kernel, RMX_I8_CONV_ALU) compute the same exact
    residues of X' = rint(w d 2^s) (DESIGN.md §5.5 step 2), so R must be bitwise equal; both are held
    to the oracle too. nlev spans one and several 1024-k work items, ragged tails included."""
    import torch
    c = syn.brute_force_case(nch, nlev, seed, ne=9, lo=0.5, hi=9.0, a=12.0, eps_hi=4.0)
    monkeypatch.delenv("RMX_I8_CONV_ALU", raising=False)
    monkeypatch.delenv("RMX_I8_CONV_EL", raising=False)
    R_tc, st1 = ctx.build_R(c.w, c.Ek, c.a, c.E)
    torch.cuda.synchronize()
    R_tc = R_tc.cpu().numpy()
    monkeypatch.setenv("RMX_I8_CONV_EL", "4")  # 4 elements per thread, one K-slice per MMA
    R_tc4, st3 = ctx.build_R(c.w, c.Ek, c.a, c.E)
    torch.cuda.synchronize()
    R_tc4 = R_tc4.cpu().numpy()
    monkeypatch.delenv("RMX_I8_CONV_EL")
    monkeypatch.setenv("RMX_I8_CONV_ALU", "1")
    R_alu, st2 = ctx.build_R(c.w, c.Ek, c.a, c.E)
    torch.cuda.synchronize()
    R_alu = R_alu.cpu().numpy()
    assert all(np.all(x.cpu().numpy() == 0) for x in (st1, st2, st3))
    assert np.array_equal(R_tc, R_alu)
    assert np.array_equal(R_tc4, R_alu)
    for p in (0, c.ne // 2, c.ne - 1):
        ref, _ = oracle.R(c.w, c.Ek, c.a, c.E[p])
        assert nrel(R_tc[p], ref) < 1e-12


@pytest.mark.parametrize("stages", ["6", "5"])
def test_int8_ring_depth_bitwise(ctx, stages, monkeypatch):
    """The pair GEMM's ring depth (RMX_I8_STAGES: 7 by default, 6 / 5 leave shared memory for a
    conversion CTA beside it - DESIGN.md §9) changes only the pipelining, never the exact int32
    products: R bitwise equal to the default ring's, nch > 256 so the CTA-pair kernel runs (ragged
    last column block, several 128-byte K boxes)."""
    import torch
    c = syn.brute_force_case(529, 1300, 21, ne=5, lo=0.5, hi=9.0, a=12.0, eps_hi=4.0)
    monkeypatch.delenv("RMX_I8_STAGES", raising=False)
    R7, _ = ctx.build_R(c.w, c.Ek, c.a, c.E)
    torch.cuda.synchronize()
    monkeypatch.setenv("RMX_I8_STAGES", stages)
    Rs, st = ctx.build_R(c.w, c.Ek, c.a, c.E)
    torch.cuda.synchronize()
    assert np.all(st.cpu().numpy() == 0)
    assert np.array_equal(R7.cpu().numpy(), Rs.cpu().numpy())
