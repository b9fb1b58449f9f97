"""Per-phase clock64 breakdown of the matching kernel (block 0, summed over its energies) on darc
bench batches, from the diagnostic build:  python -m paper_1403_5524_b200.build --phases;
RMX_LIB=paper_1403_5524_b200/librmx_phases.so python tools/phases.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1403_5524_b200 as rmx  # noqa: E402
import rmx_synth as syn  # noqa: E402

c = syn.make_case("darc")
ctx = rmx.Context(0)
ctx.set_r_algo(rmx.R_INT8)
for lo in (20000, 50000, 90000):
    E = c.E[lo:lo + 296]
    F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
    no = syn.n_open(c.eps, E)
    ctx.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, batch=296)
    torch.cuda.synchronize()
out = (ctypes.c_ulonglong * 8)()
ctx.lib.rmx_debug_match_phases(out)
names = ["formation", "panels (panel_lu + K=32 updates)", "U12 + K=128 trailing", "back substitution GEMMs",
         "output", "tri_inv128 (L11, LU)", "tri_inv128 (U_pp, back sub)"]
tot = sum(out[k] for k in range(7))
for k, n in enumerate(names):
    print(f"{n:36s} {out[k] / 1e6:10.1f} Mcycles {100 * out[k] / tot:5.1f} %")
if hasattr(ctx.lib, "rmx_debug_panel_phases"):
    ctx.lib.rmx_debug_panel_phases(out)
    for k, n in enumerate(["staging", "factor (smem)", "write-back + interchanges", "rank-w update"]):
        print(f"  panel {n:30s} {out[k] / 1e6:10.1f} Mcycles")
# T epilogue (tepi.cu, complex LDL^T route)
ctx.lib.rmx_debug_tepi_phases(out)
names = ["copy (+ photo v)", "diagonal LDL^T + inverse (smem)", "W21 = A21 Tinv^T", "L21 scaling",
         "trailing updates (K = 2 x 64)", "Z = L^-1", "Y = D^-1 Z, A^-1 = Z^T Y", "mirror + epilogue"]
tot = sum(out[k] for k in range(8))
print()
for k, n in enumerate(names):
    print(f"tepi {n:36s} {out[k] / 1e6:10.1f} Mcycles {100 * out[k] / tot:5.1f} %")
