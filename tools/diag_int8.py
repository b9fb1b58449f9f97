import numpy as np, torch, sys
sys.path.insert(0, "/root/repo")
import rmx_synth as syn, oracle, paper_1403_5524_b200 as rmx
c = syn.make_case("darc")
E = c.E[50000:50000 + 296]
F, G, Fp, Gp = syn.asymptotic(c.eps, E, c.a)
no = syn.n_open(c.eps, E)
ctx8 = rmx.Context(); ctx8.set_r_algo(rmx.R_INT8)
ctx64 = rmx.Context()
o8 = ctx8.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, batch=296)
o64 = ctx64.sweep(c.w, c.Ek, c.a, E, F, G, Fp, Gp, no, batch=296)
torch.cuda.synchronize()
rs8, rs64 = o8["rowsum"].cpu().numpy(), o64["rowsum"].cpu().numpy()
per = np.max(np.abs(rs8 - rs64), axis=1) / np.max(np.abs(rs64), axis=1)
order = np.argsort(per)[::-1][:3]
for l in order:
    dt = np.min(np.abs(E[l] - c.eps)); dp = np.min(np.abs(E[l] - c.Ek))
    ref = oracle.sweep(c.w, c.Ek, c.a, E[l:l+1], F[l:l+1], G[l:l+1], Fp[l:l+1], Gp[l:l+1], no[l:l+1], np.arange(1), want=("rowsum",), diag=True)
    r = ref["rowsum"][0]
    e8 = np.max(np.abs(rs8[l]-r))/np.max(np.abs(r)); e64 = np.max(np.abs(rs64[l]-r))/np.max(np.abs(r))
    print(l, f"8vs64 {per[l]:.2e} int8-oracle {e8:.2e} dmma-oracle {e64:.2e} dthresh {dt:.2e} dpole {dp:.2e} cond {ref['diag'][0][2]:.2e}")
print("median per-energy diff", np.median(per))
