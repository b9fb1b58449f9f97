"""One launch of each librmx kernel on a darc-shaped batch at a representative energy (for ncu)."""
import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import rmx_synth as syn, paper_1403_5524_b200 as rmx
cfg = sys.argv[1] if len(sys.argv) > 1 else "darc"
ne = int(sys.argv[2]) if len(sys.argv) > 2 else 148
frac = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
c = syn.make_case(cfg)
i0 = int(frac * (c.ne - ne))
E = c.E[i0:i0 + ne]
F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
no = syn.n_open(c.eps, E)
print("n_open mean", no.mean(), flush=True)
ctx = rmx.Context()
R, st = ctx.build_R(c.w, c.Ek, c.a, E)
K, st = ctx.match_K(R, F, G, Fp, Gp, c.a, no, status=st)
T2, rs, st = ctx.collision_strength(K, no, status=st)
torch.cuda.synchronize()
ctx.set_timing(True); ctx.reset_stats()
R, st = ctx.build_R(c.w, c.Ek, c.a, E)
K, st = ctx.match_K(R, F, G, Fp, Gp, c.a, no, status=st)
T2, rs, st = ctx.collision_strength(K, no, status=st)
print(ctx.stats(), "bad", int((st != 0).sum()), flush=True)
