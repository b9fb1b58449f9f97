"""Measurement of the SURVEY.md §8(f) 'next' rows on one B200 (one JSON line per row, CUDA-event
timing on the launching stream after warm-up, inputs resident in HBM):

  levels  NEXT-2  fused level-pair collision strengths: darc sweep (296 energies) with and without
                  rmx_sweep_levels' Omega epilogue (300 levels) - the overhead of the fusion
  photo   NEXT-1  fused photoionisation sweep (rmx_sweep_photo) on darc shapes, and the dipole
                  amplitude contraction alone (FP64 FMA roofline)
  inner   NEXT-3  rmx_inner_region (cuSOLVER syevd + DGEMM) at nlev = 3000 (config 'small') and 8000
  conv    NEXT-4  rmx_convolve_gaussian on the 'fine' mesh (400000 points, FWHM 4 meV = PAPER.md:132's
                  ALS resolution), 3 spectra mixed 2:1:1 (FP64 FMA roofline)
  maxwell NEXT-4  rmx_maxwell_average of 300 ground-level pairs over the darc mesh (100000 points),
                  16 temperatures (HBM roofline: Omega read once)

    python tools/bench_next.py [--rows levels,photo,inner,conv,maxwell] [--out FILE]
The oracle (CPU, host cores) is timed beside each row on a bounded sample.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import rmx_synth as syn  # noqa: E402

FP64_DFMA_PEAK = 34.2   # TFLOP/s, measured on this pool (profiles/r01_fp64_peak.jsonl)
FP64_DMMA_PEAK = 37.1


def hbm_peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


def timed(fn, reps=3, warm=2):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def row_levels(ctx, out):
    import torch
    c = syn.make_case("darc")
    ls = syn.level_start(c.eps)
    idx = np.arange(50000, 50000 + 296)
    E = c.E[idx]
    F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
    no = syn.n_open(c.eps, E)
    dev = "cuda"
    w, nlev, ldw = ctx.prepare_w(c.w)
    t = {k: torch.from_numpy(v).to(dev) for k, v in dict(Ek=c.Ek, E=E, F=F, G=G, Fp=Fp, Gp=Gp).items()}
    nod = torch.from_numpy(no).to(dev)
    lsd = torch.from_numpy(ls).to(dev)
    om = torch.zeros((len(E), 300, 300), dtype=torch.float64, device=dev)
    base = timed(lambda: ctx.sweep(w, t["Ek"], c.a, t["E"], t["F"], t["G"], t["Fp"], t["Gp"], nod,
                                   batch=296, prepared=(nlev, ldw)), reps=2, warm=1)
    lev = timed(lambda: ctx.sweep_levels(w[:, :nlev], t["Ek"], c.a, t["E"], t["F"], t["G"], t["Fp"],
                                         t["Gp"], nod, lsd, omega=om, batch=296), reps=2, warm=1)
    out.append({"row": "NEXT-2 level-pair collision strengths (fused)", "workload": "darc, 296 energies at mesh 50000.., 300 levels",
                "ms_sweep": base, "ms_sweep_levels": lev, "overhead_frac": lev / base - 1.0,
                "energies_per_s": len(E) / (lev / 1e3)})


def row_photo(ctx, out):
    import torch
    import oracle
    c = syn.make_case("darc")
    rng = np.random.default_rng(0)
    d = rng.normal(0.0, 1.0, c.nlev)  # synthetic inner-region dipoles d_k ~ N(0,1) (P1)
    idx = np.arange(50000, 50000 + 296)
    E = c.E[idx]
    F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
    no = syn.n_open(c.eps, E)
    dev = "cuda"
    w, nlev, ldw = ctx.prepare_w(c.w)
    t = {k: torch.from_numpy(v).to(dev) for k, v in dict(Ek=c.Ek, E=E, F=F, G=G, Fp=Fp, Gp=Gp, d=d).items()}
    nod = torch.from_numpy(no).to(dev)
    base = timed(lambda: ctx.sweep(w, t["Ek"], c.a, t["E"], t["F"], t["G"], t["Fp"], t["Gp"], nod,
                                   batch=296, prepared=(nlev, ldw)), reps=2, warm=1)
    ph = timed(lambda: ctx.sweep_photo(w[:, :nlev], t["Ek"], t["d"], c.a, t["E"], t["F"], t["G"], t["Fp"],
                                       t["Gp"], nod, -2.0, batch=296), reps=2, warm=1)
    gms = timed(lambda: ctx.dipole_amplitude(w[:, :nlev], t["Ek"], t["d"], t["E"]), reps=5, warm=2)
    gfl = 2.0 * c.nch * c.nlev * len(E)
    # oracle: the dipole contraction + amplitudes at one energy (the K of that energy from the oracle)
    t0 = time.perf_counter()
    oracle.photo_sweep(c.w, c.Ek, d, c.a, E[:1], F[:1], G[:1], Fp[:1], Gp[:1], no[:1], E0=-2.0)
    cpu_s = time.perf_counter() - t0
    out.append({"row": "NEXT-1 photoionisation sweep (fused)", "workload": "darc shapes, 296 energies, d_k ~ N(0,1)",
                "ms_sweep": base, "ms_sweep_photo": ph, "overhead_frac": ph / base - 1.0,
                "energies_per_s": len(E) / (ph / 1e3),
                "dipole_g": {"ms": gms, "achieved_tflops": gfl / (gms / 1e3) / 1e12,
                             "peak": FP64_DFMA_PEAK, "bound": "alu (FP64 FMA)",
                             "frac": gfl / (gms / 1e3) / 1e12 / FP64_DFMA_PEAK},
                "cpu_baseline": {"value": 1.0 / cpu_s, "unit": "energies/s", "cores": os.cpu_count(),
                                 "kind": "oracle", "sample": "1 darc energy, R -> K -> g -> M"}})


def row_inner(ctx, out):
    import torch
    import oracle
    for nlev, nch in ((3000, 64), (8000, 500)):
        rng = np.random.default_rng(nlev)
        H = np.diag(rng.uniform(0.0, 50.0, nlev))
        iu = np.triu_indices(nlev, 1)
        H[iu] = rng.normal(0.0, 0.05, len(iu[0]))
        H = np.triu(H) + np.triu(H, 1).T
        P = rng.normal(0.0, 1.0, (nlev, nch))
        Hd, Pd = torch.from_numpy(H).cuda(), torch.from_numpy(P).cuda()
        ms = timed(lambda: ctx.inner_region(Hd, Pd), reps=2, warm=1)
        t0 = time.perf_counter()
        if nlev <= 3000:
            oracle.inner_region(H, P)
        cpu = time.perf_counter() - t0
        out.append({"row": "NEXT-3 inner-region eigensolve", "workload": f"nlev={nlev}, nch={nch} (syevd + w = P^T V)",
                    "ms": ms, "bound": "library (cuSOLVER syevd)",
                    "cpu_baseline": {"value": cpu if nlev <= 3000 else None, "unit": "s", "cores": os.cpu_count(),
                                     "kind": "oracle (numpy eigh)"}})


def row_conv(ctx, out):
    import torch
    import oracle
    ne, dE = 400000, 5e-7
    fwhm = 4e-3 / 13.605693122994  # 4 meV in Ry
    rng = np.random.default_rng(1)
    nspec = 32  # 32 spectra per call (e.g. Omega(0 -> b) for 32 transitions): the kernel, not the
    x = rng.uniform(0.0, 1.0, (nspec, ne))  # Python call overhead, dominates the timed region
    xd = torch.from_numpy(x).cuda()
    ms = timed(lambda: ctx.convolve_gaussian(xd, dE, fwhm), reps=5, warm=2) / nspec
    s = fwhm / (2 * np.sqrt(2 * np.log(2)))
    M = int(np.floor(5 * s / dE))
    flops = 2.0 * (2 * M + 1) * ne  # algorithmic: one multiply-add per window point per output
    instr = (2.0 * M + 1) * ne       # executed FP64 instructions (interior: one DADD + one DFMA per pair)
    t0 = time.perf_counter()
    oracle.convolve_gaussian(x[:1, :4000], dE, fwhm)
    cpu = time.perf_counter() - t0
    out.append({"row": "NEXT-4 Gaussian convolution", "workload": f"fine mesh ne={ne}, FWHM 4 meV (M={M}), 32 spectra per call, ms per spectrum",
                "ms": ms, "points_per_s": ne / (ms / 1e3), "achieved_tflops": flops / (ms / 1e3) / 1e12,
                "bound": "alu (FP64 pipe)", "peak": FP64_DFMA_PEAK,
                "frac_fp64_issue": instr / (ms / 1e3) / (FP64_DFMA_PEAK * 1e12 / 2),
                "note": "symmetric window: 2M+1 FP64 instructions per output for 2(2M+1) algorithmic flops",
                "cpu_baseline": {"value": 4000 / cpu, "unit": "points/s", "cores": 1, "kind": "oracle",
                                 "sample": "first 4000 mesh points"}})


def row_maxwell(ctx, out):
    import torch
    import oracle
    c = syn.make_case("darc", ne=4)
    ne, npair = 100000, 4096
    E = syn.mesh(0.5, 60.0, ne)
    ls = syn.level_start(c.eps)
    rng = np.random.default_rng(3)
    # 4096 level pairs (a < b) of the 300 darc levels; E_th = energy of the upper level b
    lev = c.eps[ls[:-1]]
    Eth = np.sort(rng.choice(lev, npair))
    om = rng.uniform(0.0, 2.0, (ne, npair)) * (E[:, None] > Eth[None, :])
    kT = list(np.geomspace(0.05, 20.0, 16))
    omd, Ed, Ethd = (torch.from_numpy(v).cuda() for v in (om, E, Eth))
    ms = timed(lambda: ctx.maxwell_average(omd, Ed, Ethd, kT), reps=5, warm=2)
    byts = om.nbytes + E.nbytes * 2
    t0 = time.perf_counter()
    oracle.maxwell_average(om[:, :10], E, Eth[:10], kT)
    cpu = time.perf_counter() - t0
    out.append({"row": "NEXT-4 Maxwellian average", "workload": "darc mesh ne=100000, 4096 level pairs, 16 temperatures",
                "ms": ms, "achieved_gbs": byts / (ms / 1e3) / 1e9, "bound": "hbm", "peak": hbm_peak(),
                "frac": byts / (ms / 1e3) / 1e9 / hbm_peak(),
                "note": "Omega [ne][npair] read once; Boltzmann factors shared per (E_i, T) within a chunk",
                "exp_per_s": ne * npair * 16 / (ms / 1e3),
                "cpu_baseline": {"value": 10 / cpu, "unit": "pairs/s", "cores": 1, "kind": "oracle",
                                 "sample": "10 pairs x 16 temperatures"}})


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", default="levels,photo,inner,conv,maxwell")
    p.add_argument("--out", default=None)
    args = p.parse_args()
    import torch
    import paper_1403_5524_b200 as rmx
    torch.cuda.set_device(0)
    ctx = rmx.Context(0)
    out = []
    for r in args.rows.split(","):
        globals()[f"row_{r}"](ctx, out)
        print(json.dumps(out[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            for o in out:
                f.write(json.dumps(o) + "\n")


if __name__ == "__main__":
    main()
