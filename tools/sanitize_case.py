"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck): one fused sweep per R
formation on ragged shapes - FP64 DMMA R (nch 150, 2 tiles), INT8-CRT R with the CTA-pair GEMM and a
ragged last column block (nch 529) - through matching and the T epilogue, plus the three-call API and
the NEXT-1/NEXT-2 epilogue options. Exits non-zero on a bad status.

    compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_5524_b200 as rmx  # noqa: E402
import rmx_synth as syn  # noqa: E402

for algo, nch, nlev in ((rmx.R_DMMA, 150, 517), (rmx.R_INT8, 529, 300)):
    ctx = rmx.Context(0)
    ctx.set_r_algo(algo)
    c = syn.brute_force_case(nch, nlev, 3, ne=3, lo=0.5, hi=9.0, a=12.0, eps_hi=4.0)
    F, G, Fp, Gp = syn.asymptotic(c.eps, c.E, c.a)
    no = syn.n_open(c.eps, c.E)
    out = ctx.sweep(c.w, c.Ek, c.a, c.E, F, G, Fp, Gp, no, batch=2, dump_idx=[0, 2])
    R, st = ctx.build_R(c.w, c.Ek, c.a, c.E)
    K, st = ctx.match_K(R, F, G, Fp, Gp, c.a, no, status=st)
    T2, rs, st = ctx.collision_strength(K, no, status=st)
    ls = syn.level_start(np.repeat(np.arange(nch // 3 + 1), 3)[:nch].astype(np.float64))
    om = ctx.collision_strength_levels(K, ls, g=1.0, n_open=no)
    d = np.random.default_rng(0).normal(size=nlev)
    ph = ctx.sweep_photo(c.w, c.Ek, d, c.a, c.E, F, G, Fp, Gp, no, E0=-1.0)
    torch.cuda.synchronize()
    bad = int((out["status"] != 0).sum()) + int((st != 0).sum())
    print(f"algo {algo} nch {nch}: bad status {bad}", flush=True)
    assert bad == 0
    ctx.close()
print("SANITIZE_CASE_OK")
