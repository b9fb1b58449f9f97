"""GPU parity on SURVEY.md §8(d)'s darc and fine parity samples (the energies where the method is
hardest: near isolated R poles at +-1e-5 and +-1e-3, next to poles of K, just above thresholds, and
the narrow window resonances of fine at +1.5e-6 .. +1e-4; rmx_synth.survey_sample), at full size
(darc nch 2000, nlev 40000; fine nch 1200, nlev 30000; BASELINE.json:10-11), through the fused
rmx_sweep in both R formations - the bench default (exact INT8-CRT on tcgen05) and the FP64 DMMA
kernel - and stage by stage (GPU K from the oracle's R, GPU |T|^2 from the oracle's K).

Bars (BASELINE.json:5, normwise per energy, reading T1): R 1e-10, K_oo 1e-10, |T|^2 and row sums
1e-8. The only exclusion is reading T4's fp64 floor for K_oo: next to an R pole or a pole of K the
matching is so ill-conditioned (scaled cond_1(A) up to 1e9) that an fp64-accurate R (normwise error
~1e-15 .. 1e-14) already costs ~1e-10 in K_oo. There the GPU K_oo may exceed 1e-10 only if an fp64
LAPACK solve (numpy) fed the same R misses the oracle's K_oo by a comparable amount (within 10x, and
that miss itself above 1e-11), while the GPU R stays within 1e-13 of the oracle's. Every exclusion is
printed and counted. |T|^2 and the row sums have no exclusion. PAPER.md:128-130, 152-153 (§3: the fine
mesh exists to resolve narrow resonances, so near-pole energies are the workload).
"""
import time

import numpy as np
import pytest

import oracle
import rmx_synth as syn

pytestmark = pytest.mark.gpu

TOL_R, TOL_K, TOL_T2 = 1e-10, 1e-10, 1e-8


def nrel(x, ref):
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(x - ref)) / (den if den > 0 else 1.0))


def scaled_cond(R, G, Gp, a):
    A = np.diag(G) - a * R * Gp[None, :]
    return float(np.linalg.cond(A / np.max(np.abs(A), axis=0)[None, :], 1))


def lapack_floor(s, p, R):
    """Normwise K_oo error against the oracle of an fp64 LAPACK solve (numpy) fed the fp64 R `R`: what
    any fp64 matching of this R can be expected to reach (reading T4)."""
    c, o = s["c"], int(s["no"][p])
    A = np.diag(s["G"][p]) - c.a * R * s["Gp"][p][None, :]
    B = np.diag(s["F"][p]) - c.a * R * s["Fp"][p][None, :]
    return nrel(-np.linalg.solve(A, B[:, :o])[:o], s["ref"]["K"][p][:o, :o])


def check_K(s, p, ek, R, excl):
    """K_oo bar with reading T4's fp64-floor exclusion (printed and counted by the caller); R = the fp64
    R the GPU matching was fed (its own R end to end, the oracle's rounded R stage by stage)."""
    if ek < TOL_K:
        return
    er = nrel(R, s["ref"]["R"][p])
    enp = lapack_floor(s, p, R)
    assert er < 1e-13 and enp > 0.1 * TOL_K and ek < 10.0 * enp, (s["lab"][p], ek, enp, er)
    excl.append((s["lab"][p], f"{ek:.2e}", f"lapack(same R) {enp:.2e}"))


@pytest.fixture(scope="module", params=["darc", "fine"])
def sample(request):
    c = syn.make_case(request.param)
    E, lab = syn.survey_sample(c)
    F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
    no = syn.n_open(c.eps, E)
    t0 = time.perf_counter()
    ref = oracle.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, np.arange(len(E)),
                       threads=oracle.default_threads())
    print(f"\n[{c.name}] oracle on {len(E)} energies: {time.perf_counter() - t0:.1f} s "
          f"({oracle.default_threads()} threads)")
    assert np.all(ref["status"] == 0)
    return dict(c=c, E=E, lab=lab, F=F, G=G, Fp=Fp, Gp=Gp, no=no, ref=ref)


def _sweep(s, algo):
    import torch
    import paper_1403_5524_b200 as rmx
    c = s["c"]
    ctx = rmx.Context()
    ctx.set_r_algo(algo)
    n = len(s["E"])
    out = ctx.sweep(c.w, c.Ek, c.a, s["E"], s["F"], s["G"], s["Fp"], s["Gp"], s["no"], batch=n,
                    dump_idx=list(range(n)))
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    ctx.close()
    return res


def _check_end_to_end(s, res, what):
    c, ref, no = s["c"], s["ref"], s["no"]
    assert np.all(res["status"] == 0), res["status"]
    excl = []
    rows = []
    for p in range(len(s["E"])):
        o = int(no[p])
        er = nrel(res["R"][p], ref["R"][p])
        ek = nrel(res["K"][p][:o, :o], ref["K"][p][:o, :o]) if o else 0.0
        et = nrel(res["T2"][p], ref["T2"][p])
        es = nrel(res["rowsum"][p], ref["rowsum"][p])
        kap = scaled_cond(ref["R"][p], s["G"][p], s["Gp"][p], c.a) if o else 0.0
        rows.append((s["lab"][p], o, er, ek, et, es, kap))
        assert er < TOL_R, (s["lab"][p], er)
        check_K(s, p, ek, res["R"][p], excl)
        assert et < TOL_T2 and es < TOL_T2, (s["lab"][p], et, es)
    print(f"\n[{c.name} {what}] label, n_open, err R, err K_oo, err |T|^2, err rowsum, scaled cond(A)")
    for r in rows:
        print(f"  {r[0]:<36s} {r[1]:5d} {r[2]:.1e} {r[3]:.1e} {r[4]:.1e} {r[5]:.1e} {r[6]:.1e}")
    print(f"[{c.name} {what}] K_oo fp64-floor exclusions: {len(excl)} of {len(rows)}: {excl}")
    assert len(excl) <= len(rows) // 2


def test_sample_int8_sweep(sample):
    """Bench-default R formation (exact INT8-CRT, tcgen05) -> K -> |T|^2 against the oracle."""
    import paper_1403_5524_b200 as rmx
    _check_end_to_end(sample, _sweep(sample, rmx.R_INT8), "int8-crt sweep")


def test_sample_dmma_sweep(sample):
    """The FP64 DMMA R formation -> K -> |T|^2 against the oracle."""
    import paper_1403_5524_b200 as rmx
    _check_end_to_end(sample, _sweep(sample, rmx.R_DMMA), "fp64-dmma sweep")


def test_sample_stagewise(sample):
    """Stage isolation: the GPU matching fed with the oracle's R and the GPU T epilogue fed with the
    oracle's K meet the bars at every sample energy - |T|^2 with no exclusion, K_oo up to the fp64
    floor of the same R (so a miss end to end is the R rounding propagated, not a kernel's own error)."""
    import torch
    import paper_1403_5524_b200 as rmx
    c, ref, no = sample["c"], sample["ref"], sample["no"]
    ctx = rmx.Context()
    K, st = ctx.match_K(torch.from_numpy(ref["R"]), sample["F"], sample["G"], sample["Fp"], sample["Gp"], c.a, no)
    T2, rs, st = ctx.collision_strength(torch.from_numpy(ref["K"]), no, status=st)
    torch.cuda.synchronize()
    K, T2, rs, st = K.cpu().numpy(), T2.cpu().numpy(), rs.cpu().numpy(), st.cpu().numpy()
    assert np.all(st == 0)
    worst = [0.0, 0.0, 0.0]
    excl = []
    for p in range(len(sample["E"])):
        o = int(no[p])
        ek = nrel(K[p][:o, :o], ref["K"][p][:o, :o]) if o else 0.0
        et, es = nrel(T2[p], ref["T2"][p]), nrel(rs[p], ref["rowsum"][p])
        check_K(sample, p, ek, ref["R"][p], excl)
        assert et < TOL_T2 and es < TOL_T2, (sample["lab"][p], et, es)
        worst = [max(worst[0], ek), max(worst[1], et), max(worst[2], es)]
    print(f"\n[{c.name} stagewise] worst K_oo {worst[0]:.1e}  |T|^2 {worst[1]:.1e}  rowsum {worst[2]:.1e}; "
          f"K_oo fp64-floor exclusions {len(excl)} of {len(sample['E'])}: {excl}")
    assert len(excl) <= len(sample["E"]) // 2
