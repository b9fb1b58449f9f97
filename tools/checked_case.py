"""Bounds-checked workload (the stand-in for compute-sanitizer, which is closed on the GPU pool):
run with the checked build,

    RMX_LIB=paper_1403_5524_b200/librmx_checked.so python tools/checked_case.py

librmx_checked.so (-DRMX_CHECKS) traps on any workspace / output index outside its matrix
(rmx_common.cuh RMX_CHECK: MatView::at, GEMM C tiles, LU row interchanges). On top of that every
output buffer here is surrounded by NaN-free guard bands of a sentinel value that must survive, and
the results are compared with the oracle. Shapes: ragged tiles and panels, odd nlev, closed channels;
FP64 DMMA R (nch 150 / 33) and INT8-CRT R with the CTA-pair GEMM and ragged last block (nch 529);
three-call API, fused sweep with dumps, NEXT-1 / NEXT-2 epilogue options. Prints CHECKED_CASE_OK."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (test infrastructure: the comparison)
import paper_1403_5524_b200 as rmx  # noqa: E402
import rmx_synth as syn  # noqa: E402

SENT = -12345.678
G = 4096  # guard doubles on each side


def guarded(shape, dtype=torch.float64):
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * G,), SENT if dtype == torch.float64 else -7, dtype=dtype, device="cuda")
    return buf, buf[G:G + n].view(*shape)


def guards_ok(buf, dtype=torch.float64):
    s = SENT if dtype == torch.float64 else -7
    return bool((buf[:G] == s).all()) and bool((buf[-G:] == s).all())


def nrel(x, r):
    return float(np.max(np.abs(x - r)) / max(np.max(np.abs(r)), 1e-300))


lib = rmx.load_library()
print("library:", os.environ.get("RMX_LIB", "default"), flush=True)
for algo, nch, nlev in ((rmx.R_DMMA, 150, 517), (rmx.R_DMMA, 33, 64), (rmx.R_INT8, 529, 300)):
    ctx = rmx.Context(0)
    ctx.set_r_algo(algo)
    c = syn.brute_force_case(nch, nlev, 3, ne=3, lo=0.5, hi=9.0, a=12.0, eps_hi=4.0)
    F, Gs, Fp, Gp = syn.asymptotic(c.eps, c.E, c.a)
    no = syn.n_open(c.eps, c.E)
    ne = c.ne
    bR, R = guarded((ne, nch, nch))
    bK, K = guarded((ne, nch, nch))
    bT, T2 = guarded((ne, nch, nch))
    bS, rs = guarded((ne, nch))
    bst, st = guarded((ne,), torch.int32)
    st.zero_()
    ctx.build_R(c.w, c.Ek, c.a, c.E, status=st, out=R)
    ctx.match_K(R, F, Gs, Fp, Gp, c.a, no, status=st, out=K)
    nod = torch.from_numpy(no).cuda()
    rc = lib.rmx_collision_strength(ctx._h, ctypes.c_void_p(K.data_ptr()), nch, ne,
                                    ctypes.c_void_p(nod.data_ptr()), ctypes.c_void_p(T2.data_ptr()),
                                    ctypes.c_void_p(rs.data_ptr()), ctypes.c_void_p(st.data_ptr()))
    assert rc == 0, ctx.lib.rmx_last_error(ctx._h)
    bS2, rs2 = guarded((ne, nch))
    out = ctx.sweep(c.w, c.Ek, c.a, c.E, F, Gs, Fp, Gp, no, batch=2, dump_idx=[0, 2], rowsum=rs2)
    ls = syn.level_start(np.repeat(np.arange(nch // 3 + 1), 3)[:nch].astype(np.float64))
    om, _ = ctx.collision_strength_levels(K, ls, g=1.0, n_open=no)
    d = np.random.default_rng(0).normal(size=nlev)
    ph = ctx.sweep_photo(c.w, c.Ek, d, c.a, c.E, F, Gs, Fp, Gp, no, E0=-1.0)
    torch.cuda.synchronize()
    for b, dt in ((bR, torch.float64), (bK, torch.float64), (bT, torch.float64), (bS, torch.float64),
                  (bS2, torch.float64), (bst, torch.int32)):
        assert guards_ok(b, dt), "guard band overwritten"
    assert int((st != 0).sum()) == 0 and int((out["status"] != 0).sum()) == 0
    ref = oracle.sweep(c.w, c.Ek, c.a, c.E, F, Gs, Fp, Gp, no, np.arange(ne))
    Rh, Kh, T2h, rsh = R.cpu().numpy(), K.cpu().numpy(), T2.cpu().numpy(), rs.cpu().numpy()
    for p in range(ne):
        o = int(no[p])
        assert nrel(Rh[p], ref["R"][p]) < 1e-10
        assert o == 0 or nrel(Kh[p][:o, :o], ref["K"][p][:o, :o]) < 1e-10
        assert nrel(T2h[p], ref["T2"][p]) < 1e-8 and nrel(rsh[p], ref["rowsum"][p]) < 1e-8
    assert np.array_equal(rs2.cpu().numpy(), rsh)
    print(f"algo {algo} nch {nch} nlev {nlev}: checks, guard bands and oracle parity ok", flush=True)
    ctx.close()
print("CHECKED_CASE_OK")
